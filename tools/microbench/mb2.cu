// Latency + contraction-variant micro-benchmarks (design exploration, not product code).
#include <cstdio>
#include <cstdint>
#include <vector>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void lat_dfma(double* out, long long* cyc, int n){
  double a = out[0], b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i=0;i<n;i++){ a = __fma_rn(a,b,c); }
  long long t1 = clock64();
  out[1]=a; cyc[0]=t1-t0;
}
__global__ void lat_dadd(double* out, long long* cyc, int n){
  double a = out[0], c = 1e-9;
  long long t0 = clock64();
  for (int i=0;i<n;i++){ a = __dadd_rn(a,c); }
  long long t1 = clock64();
  out[1]=a; cyc[0]=t1-t0;
}
__global__ void lat_lds(double* out, long long* cyc, int n){
  __shared__ int idx[1024];
  for(int i=threadIdx.x;i<1024;i+=blockDim.x) idx[i]=(i*37+11)&1023;
  __syncthreads();
  int j=0;
  long long t0 = clock64();
  for (int i=0;i<n;i++){ j = idx[j]; }
  long long t1 = clock64();
  out[1]=j; cyc[0]=t1-t0;
}

// contraction variants: W[r][i] = sum_k P[r][k] V[k][i], canonical fma chain
template<int RM, int CM, int TR, int TC>
__global__ void __launch_bounds__((TR/RM)*(TC/CM)) contract_v(const double* __restrict__ P, const double* __restrict__ V, double* __restrict__ W, int rows, int K, int S){
  extern __shared__ __align__(16) double sm[];
  double* vs = sm;                 // [K][TC]
  double* ps = sm + K*TC;          // [K][TR] transposed
  constexpr int NT=(TR/RM)*(TC/CM);
  const int i0=blockIdx.x*TC, r0=blockIdx.y*TR, tid=threadIdx.x;
  for(int e=tid;e<K*TC;e+=NT){int kp=e/TC,c=e%TC; vs[e]=(i0+c<S)?V[(size_t)kp*S+i0+c]:0.0;}
  for(int e=tid;e<K*TR;e+=NT){int r=e/K,kp=e%K; ps[kp*TR+r]=(r0+r<rows)?P[(size_t)(r0+r)*K+kp]:0.0;}
  __syncthreads();
  const int rr=(tid/(TC/CM))*RM, cc=(tid%(TC/CM))*CM;
  double acc[RM][CM];
  #pragma unroll
  for(int a=0;a<RM;a++) 
  #pragma unroll
  for(int b=0;b<CM;b++) acc[a][b]=0.0;
  #pragma unroll 2
  for(int kp=0;kp<K;kp++){
    double pr[RM], vc[CM];
    #pragma unroll
    for(int a=0;a<RM;a++) pr[a]=ps[kp*TR+rr+a];
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
  for(int b=0;b<CM;b++) if(r0+rr+a<rows && i0+cc+b<S) W[(size_t)(r0+rr+a)*S+i0+cc+b]=acc[a][b];
}

// diagnostics: MODE 0 = stage+compute (plain loads), 1 = staging only, 2 = compute only,
// 3 = cp.async 8B staging + compute, 4 = no smem for V (global __ldg in loop, P in smem)
__device__ __forceinline__ void cpa8(void* d, const void* s){ unsigned a=(unsigned)__cvta_generic_to_shared(d); asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n"::"r"(a),"l"(s)); }
template<int MODE>
__global__ void __launch_bounds__(128) contract_diag(const double* __restrict__ P, const double* __restrict__ V, double* __restrict__ W, int rows, int K, int S){
  constexpr int TR=16, TC=32, RM=2, CM=2, NT=128;
  extern __shared__ __align__(16) double sm[];
  double* vs = sm; double* ps = sm + K*TC;
  const int i0=blockIdx.x*TC, r0=blockIdx.y*TR, tid=threadIdx.x;
  if (MODE==0 || MODE==1) {
    for(int e=tid;e<K*TC;e+=NT){int kp=e/TC,c=e%TC; vs[e]=(i0+c<S)?V[(size_t)kp*S+i0+c]:0.0;}
    for(int e=tid;e<K*TR;e+=NT){int r=e/K,kp=e%K; ps[kp*TR+r]=(r0+r<rows)?P[(size_t)(r0+r)*K+kp]:0.0;}
  } else if (MODE==3) {
    for(int e=tid;e<K*TC;e+=NT){int kp=e/TC,c=e%TC; if(i0+c<S) cpa8(vs+e, V+(size_t)kp*S+i0+c); else vs[e]=0.0;}
    for(int e=tid;e<K*TR;e+=NT){int r=e/K,kp=e%K; if(r0+r<rows) cpa8(ps+kp*TR+r, P+(size_t)(r0+r)*K+kp); else ps[kp*TR+r]=0.0;}
    asm volatile("cp.async.wait_all;\n"::);
  } else if (MODE==4) {
    for(int e=tid;e<K*TR;e+=NT){int r=e/K,kp=e%K; ps[kp*TR+r]=(r0+r<rows)?P[(size_t)(r0+r)*K+kp]:0.0;}
  } else {
    for(int e=tid;e<K*(TC+TR);e+=NT) sm[e]=0.5;
  }
  __syncthreads();
  if (MODE==1) { if(tid==0) W[blockIdx.x]=vs[5]+ps[3]; return; }
  const int rr=(tid/(TC/CM))*RM, cc=(tid%(TC/CM))*CM;
  double a00=0,a01=0,a10=0,a11=0;
  #pragma unroll 4
  for(int kp=0;kp<K;kp++){
    double p0=ps[kp*TR+rr], p1=ps[kp*TR+rr+1];
    double v0,v1;
    if (MODE==4) { v0=__ldg(V+(size_t)kp*S+min(i0+cc,S-1)); v1=__ldg(V+(size_t)kp*S+min(i0+cc+1,S-1)); }
    else { v0=vs[kp*TC+cc]; v1=vs[kp*TC+cc+1]; }
    a00=__fma_rn(p0,v0,a00); a01=__fma_rn(p0,v1,a01); a10=__fma_rn(p1,v0,a10); a11=__fma_rn(p1,v1,a11);
  }
  if(r0+rr+1<rows && i0+cc+1<S){ W[(size_t)(r0+rr)*S+i0+cc]=a00; W[(size_t)(r0+rr)*S+i0+cc+1]=a01; W[(size_t)(r0+rr+1)*S+i0+cc]=a10; W[(size_t)(r0+rr+1)*S+i0+cc+1]=a11; }
}
template<int MODE>
int run_diag(const double* P, const double* V, double* W, int K, int S, int reps){
  size_t sm=sizeof(double)*K*(16+32);
  cudaFuncSetAttribute(contract_diag<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,(int)sm);
  dim3 g((S+31)/32,(K+15)/16);
  cudaStream_t s; cudaStreamCreate(&s); cudaGraph_t gr; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s,cudaStreamCaptureModeGlobal);
  for(int r=0;r<reps;r++) contract_diag<MODE><<<g,128,sm,s>>>(P,V,W,K,K,S);
  cudaStreamEndCapture(s,&gr); CK(cudaGraphInstantiate(&ge,gr,0));
  cudaGraphLaunch(ge,s); CK(cudaStreamSynchronize(s));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0,s); cudaGraphLaunch(ge,s); cudaEventRecord(e1,s); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  printf("{\"test\":\"contract_diag\",\"mode\":%d,\"us_per_launch\":%.3f}\n",MODE,ms*1e3/reps);
  return 0;
}

template<int RM,int CM,int TR,int TC>
int run_variant(const char* name, const double* P, const double* V, double* W, int K, int S, int reps){
  constexpr int NT=(TR/RM)*(TC/CM);
  size_t sm=sizeof(double)*K*(TR+TC);
  if(sm>48*1024) cudaFuncSetAttribute(contract_v<RM,CM,TR,TC>, cudaFuncAttributeMaxDynamicSharedMemorySize,(int)sm);
  dim3 g((S+TC-1)/TC,(K+TR-1)/TR);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaGraph_t gr; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s,cudaStreamCaptureModeGlobal);
  for(int r=0;r<reps;r++) contract_v<RM,CM,TR,TC><<<g,NT,sm,s>>>(P,V,W,K,K,S);
  cudaStreamEndCapture(s,&gr); CK(cudaGraphInstantiate(&ge,gr,0));
  cudaGraphLaunch(ge,s); CK(cudaStreamSynchronize(s));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0,s); cudaGraphLaunch(ge,s); cudaEventRecord(e1,s); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  printf("{\"test\":\"contract_%s\",\"RM\":%d,\"CM\":%d,\"TR\":%d,\"TC\":%d,\"blocks\":%d,\"threads\":%d,\"us_per_launch\":%.3f}\n",name,RM,CM,TR,TC,g.x*g.y,NT,ms*1e3/reps);
  return 0;
}

__global__ void k_empty(){}

int main(){
  double* d; long long* c; CK(cudaMalloc(&d,64)); CK(cudaMalloc(&c,64)); CK(cudaMemset(d,0,64));
  long long h; int n=4096;
  lat_dfma<<<1,1>>>(d,c,n); lat_dfma<<<1,1>>>(d,c,n); CK(cudaMemcpy(&h,c,8,cudaMemcpyDeviceToHost)); printf("{\"test\":\"lat_dfma_cycles\",\"v\":%.2f}\n",(double)h/n);
  lat_dadd<<<1,1>>>(d,c,n); lat_dadd<<<1,1>>>(d,c,n); CK(cudaMemcpy(&h,c,8,cudaMemcpyDeviceToHost)); printf("{\"test\":\"lat_dadd_cycles\",\"v\":%.2f}\n",(double)h/n);
  lat_lds<<<1,32>>>(d,c,n); lat_lds<<<1,32>>>(d,c,n); CK(cudaMemcpy(&h,c,8,cudaMemcpyDeviceToHost)); printf("{\"test\":\"lat_lds_cycles\",\"v\":%.2f}\n",(double)h/n);
  int K=100,S=1001;
  std::vector<double> hP(200*200,0.01), hV(200*S,1.0);
  double *P,*V,*W; CK(cudaMalloc(&P,8*200*200)); CK(cudaMalloc(&V,8*200*S)); CK(cudaMalloc(&W,8*200*S));
  cudaMemcpy(P,hP.data(),8*200*200,cudaMemcpyHostToDevice); cudaMemcpy(V,hV.data(),8*200*S,cudaMemcpyHostToDevice);
  int reps=200;

  for (int kk : {4, 25, 50, 100, 200}) { printf("K=%d ", kk); run_diag<2>(P,V,W,kk,S,reps); }
  for (int kk : {4, 25, 50, 100}) { printf("K=%d ", kk); run_diag<3>(P,V,W,kk,S,reps); }
  // empty-kernel graph cost for reference
  { cudaStream_t s; cudaStreamCreate(&s); cudaGraph_t gr; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s,cudaStreamCaptureModeGlobal);
    for(int r=0;r<reps;r++) k_empty<<<400,256,0,s>>>();
    cudaStreamEndCapture(s,&gr); cudaGraphInstantiate(&ge,gr,0); cudaGraphLaunch(ge,s); cudaStreamSynchronize(s);
    cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0,s); cudaGraphLaunch(ge,s); cudaEventRecord(e1,s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1); printf("{\"test\":\"graph_empty_400x256\",\"us_per_launch\":%.3f}\n",ms*1e3/reps); }
  return 0;
}
