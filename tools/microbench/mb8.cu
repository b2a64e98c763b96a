// DMMA (mma.sync.m8n8k4.f64) latency and throughput vs independent chains per SM sub-partition.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb8 mb8.cu && ./mb8
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters, long long* cyc) {
  double c[CH][2];
  for (int j = 0; j < CH; ++j) c[j][0] = c[j][1] = threadIdx.x * 1e-3 + j;
  double a = 1.0000001, b = 0.9999999;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int CH>
void run(int warps, double* out, long long* cyc) {
  const int iters = 2000;
  k<CH><<<148, 32 * warps>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / iters;   // cycles per loop iteration (CH DMMAs per warp)
  printf("chains/warp %2d warps/SM %2d (chains/SP %5.1f): %.1f cycles per iteration, %.2f cycles per DMMA per SP\n", CH,
         warps, CH * warps / 4.0, per, per / (CH * warps / 4.0));
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 8);
  for (int w : {1, 4, 8, 16, 32}) { run<1>(w, out, cyc); run<2>(w, out, cyc); run<4>(w, out, cyc); run<8>(w, out, cyc); }
  return 0;
}
