// Phase timestamps inside the contraction kernel (which phase costs the microseconds?).
#include <cstdio>
#include <vector>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)
__device__ __forceinline__ unsigned long long gt(){ return (unsigned long long)clock64(); }
__device__ __forceinline__ void cpa16(void* d, const void* s){ unsigned a=(unsigned)__cvta_generic_to_shared(d); asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n"::"r"(a),"l"(s)); }
__device__ __forceinline__ void cpa8(void* d, const void* s){ unsigned a=(unsigned)__cvta_generic_to_shared(d); asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n"::"r"(a),"l"(s)); }
__global__ void __launch_bounds__(128) ck(const double* __restrict__ Pt, const double* __restrict__ Vn, double* __restrict__ Wt, int rows, int K, int S, int ld, unsigned long long* ts){
  unsigned long long t0=gt();
  extern __shared__ __align__(16) double csm[];
  const int Kp=(K+3)&~3; double* vs=csm; double* ps=csm+(size_t)Kp*32;
  const int i0=blockIdx.x*32, r0=blockIdx.y*16, tid=threadIdx.x;
  for(int r=0;r<16;++r){ const bool rin=r0+r<rows; const double* src=Pt+(size_t)(r0+r)*K; for(int kp=tid;kp<Kp;kp+=128){ if(rin&&kp<K) cpa8(ps+r*Kp+kp,src+kp); else ps[r*Kp+kp]=0.0; } }
  unsigned long long t1=gt();
  { const int c=2*(tid&15); const bool in=i0+c<ld; const double* src=Vn+i0+c;
    for(int kp=tid>>4;kp<Kp;kp+=8){ double* dst=vs+kp*32+c; if(kp<K&&in) cpa16(dst,src+(size_t)kp*ld); else {dst[0]=0;dst[1]=0;} } }
  unsigned long long t2=gt();
  asm volatile("cp.async.wait_all;\n"::); __syncthreads();
  unsigned long long t3=gt();
  const int rr=(tid/16)*2, cc=(tid%16)*2; const double* p0=ps+(size_t)rr*Kp; const double* p1=p0+Kp;
  double a00=0,a01=0,a10=0,a11=0;
  for(int kp=0;kp<Kp;kp+=4){
    #pragma unroll
    for(int q=0;q<4;q++){ double x0=p0[kp+q], x1=p1[kp+q]; double2 v=*reinterpret_cast<const double2*>(vs+(kp+q)*32+cc);
      a00=__fma_rn(x0,v.x,a00); a01=__fma_rn(x0,v.y,a01); a10=__fma_rn(x1,v.x,a10); a11=__fma_rn(x1,v.y,a11); }
  }
  unsigned long long t4=gt();
  const int i=i0+cc;
  if(r0+rr+1<rows && i+1<S){ Wt[(size_t)(r0+rr)*ld+i]=a00; Wt[(size_t)(r0+rr)*ld+i+1]=a01; Wt[(size_t)(r0+rr+1)*ld+i]=a10; Wt[(size_t)(r0+rr+1)*ld+i+1]=a11; }
  unsigned long long t5=gt();
  if(tid==0){ unsigned long long* o=ts+8*(blockIdx.y*gridDim.x+blockIdx.x); o[0]=t0;o[1]=t1;o[2]=t2;o[3]=t3;o[4]=t4;o[5]=t5; }
}
int main(){
  int S=1001, ld=1004, K=100;
  std::vector<double> hP(K*K,0.01), hV(K*ld,1.0);
  double *P,*V,*W; CK(cudaMalloc(&P,8*K*K)); CK(cudaMalloc(&V,8*K*ld)); CK(cudaMalloc(&W,8*K*ld));
  cudaMemcpy(P,hP.data(),8*K*K,cudaMemcpyHostToDevice); cudaMemcpy(V,hV.data(),8*K*ld,cudaMemcpyHostToDevice);
  dim3 g((S+31)/32,(K+15)/16); int nb=g.x*g.y;
  unsigned long long* ts; CK(cudaMalloc(&ts,8*8*nb));
  size_t sm=8*((K+3)&~3)*48; cudaFuncSetAttribute(ck,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)sm);
  for(int rep=0;rep<5;rep++){ ck<<<g,128,sm>>>(P,V,W,K,K,S,ld,ts); }
  CK(cudaDeviceSynchronize());
  std::vector<unsigned long long> h(8*nb); cudaMemcpy(h.data(),ts,8*8*nb,cudaMemcpyDeviceToHost);
  unsigned long long mn=~0ull, mx=0; for(int b=0;b<nb;b++){ mn=std::min(mn,h[8*b]); mx=std::max(mx,h[8*b+5]); }
  double ph[5]={0}; for(int b=0;b<nb;b++) for(int j=0;j<5;j++) ph[j]+=(double)(h[8*b+j+1]-h[8*b+j]);
  printf("blocks %d; (cycles) \n", nb);
  const char* nm[5]={"P issue","V issue","cp.async wait+sync","compute","store"};
  for(int j=0;j<5;j++) printf("  %-20s avg %.0f cycles\n", nm[j], ph[j]/nb);
  unsigned long long last_start=0; for(int b=0;b<nb;b++) last_start=std::max(last_start,h[8*b]);
  printf("done\n");
  return 0;
}
