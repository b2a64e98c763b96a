// (1) Is FP64 DMMA (mma.sync m8n8k4 f64) bit-identical to a sequential fma chain over k?
// (2) How fast is a K=100 accumulation chain with DMMA vs DFMA?
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

// one warp: C[8x8] = A[8xK] * B[Kx8], K multiple of 4, via K/4 DMMA (row.col), accumulating in order
__global__ void dmma_tile(const double* A, const double* B, double* C, int K){
  int lane=threadIdx.x;
  // fragment layout for m8n8k4.f64: A row-major 8x4: lane holds A[lane/4][lane%4]; B col 4x8: lane holds B[lane%4][lane/4]
  // C/D 8x8: lane holds d0 = C[lane/4][2*(lane%4)], d1 = C[lane/4][2*(lane%4)+1]
  double d0=0.0, d1=0.0;
  for(int k0=0;k0<K;k0+=4){
    double a = A[(lane/4)*K + k0 + lane%4];
    double b = B[(k0 + lane%4)*8 + lane/4];
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0),"+d"(d1) : "d"(a),"d"(b));
  }
  C[(lane/4)*8 + 2*(lane%4)] = d0;
  C[(lane/4)*8 + 2*(lane%4)+1] = d1;
}
__global__ void fma_tile(const double* A, const double* B, double* C, int K){
  int lane=threadIdx.x;
  for(int e=lane;e<64;e+=32){ int r=e/8,c=e%8; double acc=0.0; for(int k=0;k<K;k++) acc=__fma_rn(A[r*K+k],B[k*8+c],acc); C[e]=acc; }
}
int main(){
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-1,1);
  int trials=2000, K=100; long long mism=0, tot=0; double maxrel=0;
  double *dA,*dB,*dC1,*dC2; CK(cudaMalloc(&dA,8*8*K)); CK(cudaMalloc(&dB,8*8*K)); CK(cudaMalloc(&dC1,8*64)); CK(cudaMalloc(&dC2,8*64));
  std::vector<double> A(8*K),B(8*K),C1(64),C2(64);
  for(int tr=0;tr<trials;tr++){
    int mode=tr%4;
    for(auto& x:A){ x=U(rng); if(mode==1) x=std::ldexp(x, (int)(rng()%60)-30); }
    for(auto& x:B){ x=U(rng); if(mode==2) x=std::ldexp(x, (int)(rng()%60)-30); if(mode==3) x = x*1e5 + 1.0/3.0; }
    cudaMemcpy(dA,A.data(),8*8*K,cudaMemcpyHostToDevice); cudaMemcpy(dB,B.data(),8*8*K,cudaMemcpyHostToDevice);
    dmma_tile<<<1,32>>>(dA,dB,dC1,K); fma_tile<<<1,32>>>(dA,dB,dC2,K);
    cudaMemcpy(C1.data(),dC1,8*64,cudaMemcpyDeviceToHost); cudaMemcpy(C2.data(),dC2,8*64,cudaMemcpyDeviceToHost);
    for(int e=0;e<64;e++){ tot++; if(C1[e]!=C2[e]){ mism++; maxrel=std::max(maxrel, std::fabs(C1[e]-C2[e])/std::max(1e-300,std::fabs(C2[e]))); } }
  }
  printf("{\"test\":\"dmma_vs_fma_chain\",\"K\":%d,\"outputs\":%lld,\"mismatches\":%lld,\"max_rel\":%.3e}\n",K,tot,mism,maxrel);
  return 0;
}
