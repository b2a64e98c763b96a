// DMMA m8n8k4.f64 dependent-chain latency and throughput per SM.
#include <cstdio>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s: %s\n",#x,cudaGetErrorString(e)); return 1;}}while(0)
template<int C>
__global__ void chain(double* out, long long* cyc, int n){
  double a=threadIdx.x*1e-3, b=0.5; double d0[C], d1[C];
  #pragma unroll
  for(int c=0;c<C;c++){d0[c]=c; d1[c]=c;}
  long long t0=clock64();
  for(int i=0;i<n;i++){
    #pragma unroll
    for(int c=0;c<C;c++) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0[c]),"+d"(d1[c]) : "d"(a),"d"(b));
  }
  long long t1=clock64();
  double s=0;
  #pragma unroll
  for(int c=0;c<C;c++) s+=d0[c]+d1[c];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s; if(threadIdx.x==0&&blockIdx.x==0) cyc[0]=t1-t0;
}
int main(){
  double* o; long long* c; CK(cudaMalloc(&o,8*148*2048)); CK(cudaMalloc(&c,8));
  long long h; int n=2000;
  chain<1><<<1,32>>>(o,c,n); CK(cudaDeviceSynchronize()); chain<1><<<1,32>>>(o,c,n); cudaMemcpy(&h,c,8,cudaMemcpyDeviceToHost);
  printf("dmma dependent latency: %.1f cycles\n",(double)h/n);
  chain<4><<<1,32>>>(o,c,n); chain<4><<<1,32>>>(o,c,n); cudaMemcpy(&h,c,8,cudaMemcpyDeviceToHost);
  printf("1 warp, 4 chains: %.1f cycles per dmma\n",(double)h/n/4);
  for (int w : {4, 8, 16}) { chain<4><<<148,32*w>>>(o,c,n); CK(cudaDeviceSynchronize()); cudaMemcpy(&h,c,8,cudaMemcpyDeviceToHost);
    printf("%d warps/SM x 4 chains: %.2f cycles per dmma per SM (%.1f FMA/SM/clk)\n", w, (double)h/(n*4.0*w), 256.0/((double)h/(n*4.0*w))); }
  return 0;
}
