// DFMA throughput vs (warps per SM, chains per thread) -- design exploration.
#include <cstdio>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s: %s\n",#x,cudaGetErrorString(e)); return 1;}}while(0)
template<int C>
__global__ void dfma_chains(double* out, int iters){
  double a[C];
  #pragma unroll
  for(int c=0;c<C;c++) a[c]=threadIdx.x*1e-3+c;
  const double m=0.999999, d=1e-9;
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int c=0;c<C;c++) a[c]=__fma_rn(a[c],m,d);
  }
  double s=0;
  #pragma unroll
  for(int c=0;c<C;c++) s+=a[c];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
template<int C>
int run(int warps_per_sm, int sms, double* out){
  int iters=4000;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  dfma_chains<C><<<sms, 32*warps_per_sm>>>(out, 10);
  cudaEventRecord(e0); dfma_chains<C><<<sms, 32*warps_per_sm>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  double dfma_per_sm = (double)32*warps_per_sm*C*iters;
  double cycles = ms*1e-3*1.965e9;
  printf("{\"warps_per_sm\":%d,\"chains\":%d,\"dfma_per_sm_per_cycle\":%.2f}\n", warps_per_sm, C, dfma_per_sm/cycles);
  return 0;
}
int main(){
  double* out; CK(cudaMalloc(&out, 8*148*1024));
  int sms=148;
  for (int w : {1,2,4,6,8,16,32}) { run<1>(w,sms,out); run<2>(w,sms,out); run<4>(w,sms,out); run<8>(w,sms,out); }
  return 0;
}
