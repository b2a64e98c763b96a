// FP64 / sync micro-benchmarks for sm_100a design decisions (not product code).
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void k_dadd(double* out, int iters){
  double a0=threadIdx.x*1e-3,a1=a0+1,a2=a0+2,a3=a0+3,a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
  double d=1e-9;
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int u=0;u<16;u++){a0=__dadd_rn(a0,d);a1=__dadd_rn(a1,d);a2=__dadd_rn(a2,d);a3=__dadd_rn(a3,d);a4=__dadd_rn(a4,d);a5=__dadd_rn(a5,d);a6=__dadd_rn(a6,d);a7=__dadd_rn(a7,d);}
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=a0+a1+a2+a3+a4+a5+a6+a7;
}
__global__ void k_dfma(double* out, int iters){
  double a0=threadIdx.x*1e-3,a1=a0+1,a2=a0+2,a3=a0+3,a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
  double d=1e-9,m=0.999;
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int u=0;u<16;u++){a0=__fma_rn(a0,m,d);a1=__fma_rn(a1,m,d);a2=__fma_rn(a2,m,d);a3=__fma_rn(a3,m,d);a4=__fma_rn(a4,m,d);a5=__fma_rn(a5,m,d);a6=__fma_rn(a6,m,d);a7=__fma_rn(a7,m,d);}
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=a0+a1+a2+a3+a4+a5+a6+a7;
}
// max-plus with argmax from registers: 8 rows per thread, window shifting
template<int R>
__global__ void k_maxplus(const double* __restrict__ W, double* out, int* arg_out, int A, int iters){
  double best[R]; int arg[R];
  #pragma unroll
  for(int r=0;r<R;r++){best[r]=-1e300;arg[r]=-1;}
  double w[R];
  #pragma unroll
  for(int r=0;r<R;r++) w[r]=W[(threadIdx.x+r)&1023];
  for(int it=0;it<iters;it++){
    for(int a=0;a<A;a++){
      double pay = __dmul_rn(0.37, (double)a);
      #pragma unroll
      for(int r=0;r<R;r++){
        double c=__dadd_rn(pay,w[r]);
        if(c>best[r]){best[r]=c;arg[r]=a;}
      }
      #pragma unroll
      for(int r=0;r<R-1;r++) w[r]=w[r+1];
      w[R-1]=__dadd_rn(w[0],1e-12);
    }
  }
  double s=0; int ai=0;
  #pragma unroll
  for(int r=0;r<R;r++){s+=best[r]; ai+=arg[r];}
  out[blockIdx.x*blockDim.x+threadIdx.x]=s; arg_out[blockIdx.x*blockDim.x+threadIdx.x]=ai;
}
// max only (fmax) for comparison
template<int R>
__global__ void k_maxonly(const double* __restrict__ W, double* out, int A, int iters){
  double best[R];
  #pragma unroll
  for(int r=0;r<R;r++){best[r]=-1e300;}
  double w[R];
  #pragma unroll
  for(int r=0;r<R;r++) w[r]=W[(threadIdx.x+r)&1023];
  for(int it=0;it<iters;it++){
    for(int a=0;a<A;a++){
      double pay = __dmul_rn(0.37, (double)a);
      #pragma unroll
      for(int r=0;r<R;r++){ best[r]=fmax(best[r],__dadd_rn(pay,w[r])); }
      #pragma unroll
      for(int r=0;r<R-1;r++) w[r]=w[r+1];
      w[R-1]=__dadd_rn(w[0],1e-12);
    }
  }
  double s=0;
  #pragma unroll
  for(int r=0;r<R;r++){s+=best[r];}
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_gridsync(int n, unsigned* dummy){
  cg::grid_group g=cg::this_grid();
  for(int i=0;i<n;i++){ if(threadIdx.x==0 && blockIdx.x==0) dummy[0]+=1; g.sync(); }
}
__global__ void k_empty(double* p){ if(threadIdx.x==0&&blockIdx.x==0&&p) p[0]+=1.0; }
__global__ void k_dmma(double* out, int iters){
  double a=threadIdx.x*1e-3, b=0.5, c0=0,c1=0,c2=0,c3=0,c4=0,c5=0,c6=0,c7=0,c8=0,c9=0,c10=0,c11=0,c12=0,c13=0,c14=0,c15=0;
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int u=0;u<4;u++){
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0),"+d"(c1) : "d"(a),"d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c2),"+d"(c3) : "d"(a),"d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c4),"+d"(c5) : "d"(a),"d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c6),"+d"(c7) : "d"(a),"d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c8),"+d"(c9) : "d"(a),"d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c10),"+d"(c11) : "d"(a),"d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c12),"+d"(c13) : "d"(a),"d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c14),"+d"(c15) : "d"(a),"d"(b));
    }
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=c0+c1+c2+c3+c4+c5+c6+c7+c8+c9+c10+c11+c12+c13+c14+c15;
}

int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  int clk=0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"clock_khz\":%d}\n", p.name, p.multiProcessorCount, clk);
  int SM=p.multiProcessorCount;
  double *out, *W; int* ia; unsigned* du;
  CK(cudaMalloc(&out, sizeof(double)*SM*8*1024)); CK(cudaMalloc(&W, 8*4096)); CK(cudaMemset(W,0,8*4096));
  CK(cudaMalloc(&ia, sizeof(int)*SM*8*1024)); CK(cudaMalloc(&du, 64)); CK(cudaMemset(du,0,64));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  // DADD/DFMA
  for(int rep=0;rep<2;rep++){
    int iters=2000, blocks=SM*4, thr=256;
    cudaEventRecord(e0); k_dadd<<<blocks,thr>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    double ops=(double)blocks*thr*iters*16*8; if(rep) printf("{\"test\":\"dadd\",\"Gop_s\":%.1f,\"per_sm_clk_at_max\":%.2f}\n", ops/ms/1e6, ops/(ms*1e-3)/SM/(clk*1e3));
    cudaEventRecord(e0); k_dfma<<<blocks,thr>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    if(rep) printf("{\"test\":\"dfma\",\"Gop_s\":%.1f,\"TFLOPs\":%.2f}\n", ops/ms/1e6, 2*ops/ms/1e9);
    cudaEventRecord(e0); k_dmma<<<blocks,thr>>>(out,iters/2); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    double fl=(double)blocks*(thr/32)*(iters/2)*4*8*(8*8*4*2);
    if(rep) printf("{\"test\":\"dmma_m8n8k4\",\"TFLOPs\":%.2f}\n", fl/ms/1e9);
  }
  for(int occ=1; occ<=8; occ*=2) for(int rep=0;rep<2;rep++){
    int iters=20, A=201, blocks=SM*occ, thr=256;
    cudaEventRecord(e0); k_maxplus<8><<<blocks,thr>>>(W,out,ia,A,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    double cells=(double)blocks*thr*8*iters*A;
    if(rep) printf("{\"test\":\"maxplus_argmax_R8\",\"occ\":%d,\"Gcell_s\":%.1f,\"cells_per_sm_clk\":%.2f}\n", occ, cells/ms/1e6, cells/(ms*1e-3)/SM/(clk*1e3));
    cudaEventRecord(e0); k_maxonly<8><<<blocks,thr>>>(W,out,A,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    if(rep) printf("{\"test\":\"maxonly_R8\",\"occ\":%d,\"Gcell_s\":%.1f,\"cells_per_sm_clk\":%.2f}\n", occ, cells/ms/1e6, cells/(ms*1e-3)/SM/(clk*1e3));
  }
  // grid sync
  for(int thr=128; thr<=512; thr*=2){
    int n=2000; void* args[]={&n,&du};
    int blocks=SM;
    CK(cudaLaunchCooperativeKernel((void*)k_gridsync, blocks, thr, args, 0, 0)); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); CK(cudaLaunchCooperativeKernel((void*)k_gridsync, blocks, thr, args, 0, 0)); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("{\"test\":\"grid_sync\",\"blocks\":%d,\"thr\":%d,\"us_per_sync\":%.3f}\n", blocks, thr, ms*1e3/n);
  }
  // graph of empty kernels
  {
    cudaStream_t s; cudaStreamCreate(&s); cudaGraph_t g; cudaGraphExec_t ge;
    int n=576;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for(int i=0;i<n;i++) k_empty<<<SM,256,0,s>>>(out);
    cudaStreamEndCapture(s,&g); CK(cudaGraphInstantiate(&ge,g,0));
    cudaGraphLaunch(ge,s); cudaStreamSynchronize(s);
    cudaEventRecord(e0,s); cudaGraphLaunch(ge,s); cudaEventRecord(e1,s); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("{\"test\":\"graph_empty_kernels\",\"n\":%d,\"us_per_kernel\":%.3f}\n", n, ms*1e3/n);
    cudaEventRecord(e0,s); for(int i=0;i<n;i++) k_empty<<<SM,256,0,s>>>(out); cudaEventRecord(e1,s); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("{\"test\":\"stream_empty_kernels\",\"n\":%d,\"us_per_kernel\":%.3f}\n", n, ms*1e3/n);
  }
  return 0;
}
