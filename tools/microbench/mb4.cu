// Contraction kernel variants (design exploration): W[r][i] = sum_k P[r][k] V[k][i], canonical chain.
#include <cstdio>
#include <vector>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)
__device__ __forceinline__ void cpa16(void* d, const void* s){ unsigned a=(unsigned)__cvta_generic_to_shared(d); asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n"::"r"(a),"l"(s)); }
__device__ __forceinline__ void cpa8(void* d, const void* s){ unsigned a=(unsigned)__cvta_generic_to_shared(d); asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n"::"r"(a),"l"(s)); }

// RM rows x CM cols per thread; TR x TC tile; P tile [TR][Kp]; V tile [Kp][TC]
template<int RM,int CM,int TR,int TC,bool PSMEM>
__global__ void __launch_bounds__((TR/RM)*(TC/CM)) cv(const double* __restrict__ P, const double* __restrict__ V, double* __restrict__ W, int rows, int K, int S, int ld){
  constexpr int NT=(TR/RM)*(TC/CM);
  extern __shared__ __align__(16) double sm[];
  const int Kp=(K+3)&~3;
  double* vs=sm; double* ps=sm+Kp*TC;
  const int i0=blockIdx.x*TC, r0=blockIdx.y*TR, tid=threadIdx.x;
  { constexpr int CH=TC/2; const int c=2*(tid%CH); const bool in=i0+c<ld;
    for(int kp=tid/CH; kp<Kp; kp+=NT/CH){ double* d=vs+kp*TC+c; if(kp<K&&in) cpa16(d,V+(size_t)kp*ld+i0+c); else {d[0]=0;d[1]=0;} } }
  if (PSMEM) for(int r=0;r<TR;r++){ const bool rin=r0+r<rows; for(int kp=tid;kp<Kp;kp+=NT){ if(rin&&kp<K) cpa8(ps+r*Kp+kp,P+(size_t)(r0+r)*K+kp); else ps[r*Kp+kp]=0; } }
  asm volatile("cp.async.wait_all;\n"::); __syncthreads();
  const int rr=(tid/(TC/CM))*RM, cc=(tid%(TC/CM))*CM;
  double acc[RM][CM];
  #pragma unroll
  for(int a=0;a<RM;a++)
  #pragma unroll
  for(int b=0;b<CM;b++) acc[a][b]=0;
  const double* prow[RM];
  #pragma unroll
  for(int a=0;a<RM;a++) prow[a]= PSMEM ? ps+(size_t)(rr+a)*Kp : P+(size_t)min(r0+rr+a,rows-1)*K;
  #pragma unroll 4
  for(int kp=0;kp<K;kp++){
    double pr[RM], vc[CM];
    #pragma unroll
    for(int a=0;a<RM;a++) pr[a]= PSMEM ? prow[a][kp] : __ldg(prow[a]+kp);
    #pragma unroll
    for(int b=0;b<CM;b++) vc[b]=vs[kp*TC+cc+b];
    #pragma unroll
    for(int a=0;a<RM;a++)
    #pragma unroll
    for(int b=0;b<CM;b++) acc[a][b]=__fma_rn(pr[a],vc[b],acc[a][b]);
  }
  #pragma unroll
  for(int a=0;a<RM;a++)
  #pragma unroll
  for(int b=0;b<CM;b++) if(r0+rr+a<rows && i0+cc+b<S) W[(size_t)(r0+rr+a)*ld+i0+cc+b]=acc[a][b];
}
template<int RM,int CM,int TR,int TC,bool PSMEM>
int run(const char* name,const double* P,const double* V,double* W,int K,int S,int ld,int reps){
  constexpr int NT=(TR/RM)*(TC/CM);
  int Kp=(K+3)&~3; size_t sm=sizeof(double)*Kp*(TC+(PSMEM?TR:0));
  cudaFuncSetAttribute(cv<RM,CM,TR,TC,PSMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize,(int)sm);
  dim3 g((S+TC-1)/TC,(K+TR-1)/TR);
  cudaStream_t s; cudaStreamCreate(&s); cudaGraph_t gr; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s,cudaStreamCaptureModeGlobal);
  for(int r=0;r<reps;r++) cv<RM,CM,TR,TC,PSMEM><<<g,NT,sm,s>>>(P,V,W,K,K,S,ld);
  cudaStreamEndCapture(s,&gr); CK(cudaGraphInstantiate(&ge,gr,0));
  cudaGraphLaunch(ge,s); CK(cudaStreamSynchronize(s));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0,s); cudaGraphLaunch(ge,s); cudaEventRecord(e1,s); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  printf("%-4s RM=%d CM=%d TR=%2d TC=%2d P%s blocks=%4d thr=%3d K=%3d : %7.3f us\n",name,RM,CM,TR,TC,PSMEM?"smem":"ldg ",g.x*g.y,NT,K,ms*1e3/reps);
  return 0;
}
int main(){
  int S=1001, ld=1004;
  std::vector<double> hP(200*200,0.01), hV(200*ld,1.0);
  double *P,*V,*W; CK(cudaMalloc(&P,8*200*200)); CK(cudaMalloc(&V,8*200*ld)); CK(cudaMalloc(&W,8*200*ld));
  cudaMemcpy(P,hP.data(),8*200*200,cudaMemcpyHostToDevice); cudaMemcpy(V,hV.data(),8*200*ld,cudaMemcpyHostToDevice);
  for (int K : {4, 100}) {
    run<2,2,16,32,true>("A",P,V,W,K,S,ld,200);
    run<2,2,16,32,false>("B",P,V,W,K,S,ld,200);
    run<1,2,8,32,true>("C",P,V,W,K,S,ld,200);
    run<4,1,16,32,true>("D",P,V,W,K,S,ld,200);
    run<4,1,16,32,false>("D2",P,V,W,K,S,ld,200);
    run<2,1,8,32,true>("E",P,V,W,K,S,ld,200);
    run<2,1,8,32,false>("E2",P,V,W,K,S,ld,200);
    run<1,1,4,32,false>("F",P,V,W,K,S,ld,200);
    run<4,2,16,64,true>("G",P,V,W,K,S,ld,200);
    run<2,2,8,64,true>("H",P,V,W,K,S,ld,200);
  }
  return 0;
}
