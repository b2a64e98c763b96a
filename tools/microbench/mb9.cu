// Thread-block clusters on B200 for a fused expectation + stencil stage: how many clusters
// of 8 / 16 CTAs can be resident, where their CTAs land, and what one "write own W tile -> cluster barrier ->
// read the halo" exchange costs, through L2 (st.global + barrier.cluster release/acquire + ld.global.cg) or
// through distributed shared memory (ld.shared::cluster).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb9 mb9.cu && ./mb9
#include <cstdio>
#include <vector>
#include <set>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
__device__ __forceinline__ unsigned ctarank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync_rel_acq() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__global__ void where(unsigned* out) {
  if (threadIdx.x == 0) out[blockIdx.y * gridDim.x + blockIdx.x] = smid();
}

// ROWS x TW own tile per CTA, halo of HL columns left and HR right; iters exchanges
template <int MODE>
__global__ void exch(double* buf, int ld, int TW, int HL, int HR, int iters, long long* cyc, double* sink) {
  extern __shared__ double sm[];
  constexpr int ROWS = 8;
  const int c = ctarank(), cs = gridDim.x, tid = threadIdx.x;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double* b = buf + (size_t)(it & 1) * ROWS * ld + (size_t)blockIdx.y * 2 * ROWS * ld;
    for (int e = tid; e < ROWS * TW; e += blockDim.x) {
      const int r = e / TW, x = e - r * TW;
      const double v = acc + r + x;
      if (MODE == 0) __stcg(b + (size_t)r * ld + c * TW + x, v);
      else sm[(it & 1) * ROWS * TW + e] = v;
    }
    cluster_sync_rel_acq();
    const int lo = c * TW - HL, n = TW + HL + HR;
    if (MODE < 2) {
      constexpr int NL = 12;   // loads per thread issued before any use (ROWS * n <= NL * blockDim)
      double v[NL];
#pragma unroll
      for (int u = 0; u < NL; ++u) {
        const int e = tid + u * blockDim.x;
        const int r = e / n, col = lo + e - r * n;
        v[u] = 0.0;
        if (e < ROWS * n && col >= 0 && col < cs * TW) {
          if (MODE == 0) v[u] = __ldcg(b + (size_t)r * ld + col);
          else {
            const int owner = col / TW, x = col - owner * TW;
            const double* p = sm + (it & 1) * ROWS * TW + r * TW + x;
            unsigned la = (unsigned)__cvta_generic_to_shared(p), ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(owner));
            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v[u]) : "r"(ra));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < NL; ++u) acc += v[u];
    }
  }
  cluster_sync_rel_acq();
  long long t1 = clock64();
  if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) *cyc = t1 - t0;
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  printf("%s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  CK(cudaFuncSetAttribute(where, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(exch<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(exch<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(exch<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(exch<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(exch<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(exch<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int cs : {2, 4, 8, 16}) {
    for (int smem : {32, 64, 96, 160}) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(cs, 64); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem * 1024;
      cfg.attrs = at; cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)exch<0>, &cfg);
      printf("cluster %2d smem %3d KB: max active clusters %d (%s) = %d CTAs\n", cs, smem, n,
             e == cudaSuccess ? "ok" : cudaGetErrorString(e), n * cs);
    }
  }
  // placement of a (16 x 13) grid in clusters of 16 and of (8 x 13) in clusters of 8
  unsigned* d_out;
  CK(cudaMalloc(&d_out, 4096 * 4));
  for (int cs : {8, 16}) {
    for (int ny : {13, 26}) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(cs, ny); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 0;
      cfg.attrs = at; cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, where, d_out));
      CK(cudaDeviceSynchronize());
      std::vector<unsigned> h(cs * ny);
      CK(cudaMemcpy(h.data(), d_out, h.size() * 4, cudaMemcpyDeviceToHost));
      std::set<unsigned> sms(h.begin(), h.end());
      int lo = 0;
      for (unsigned s : sms) lo += s < 74;
      printf("cluster %d grid %dx%d: %zu distinct SMs (%d below 74), cluster 0 SMs:", cs, cs, ny, sms.size(), lo);
      for (int i = 0; i < cs; ++i) printf(" %u", h[i]);
      printf("\n");
    }
  }
  // exchange cost
  double *buf, *sink;
  long long* cyc;
  const int ld = 1024;
  CK(cudaMalloc(&buf, (size_t)64 * 2 * 8 * ld * sizeof(double)));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMalloc(&cyc, 8));
  for (int mode = 0; mode < 3; ++mode) {
    for (int cs : {8, 16}) {
      for (int ny : {13, 26}) {
        const int TW = 1024 / cs, iters = 1000;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(cs, ny); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 2 * 8 * TW * sizeof(double) + 32 * 1024;
        cfg.attrs = at; cfg.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep) {
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0); cudaEventCreate(&e1);
          cudaEventRecord(e0);
          cudaError_t e = mode == 0 ? cudaLaunchKernelEx(&cfg, exch<0>, buf, ld, TW, 105, 96, iters, cyc, sink)
                                    : mode == 1 ? cudaLaunchKernelEx(&cfg, exch<1>, buf, ld, TW, 105, 96, iters, cyc, sink) : cudaLaunchKernelEx(&cfg, exch<2>, buf, ld, TW, 105, 96, iters, cyc, sink);
          cudaEventRecord(e1);
          CK(e);
          CK(cudaDeviceSynchronize());
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          long long hc;
          cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
          if (rep) printf("exchange %s cluster %2d x %2d groups (TW %d): %.3f us / iteration, %lld cycles\n",
                          mode == 2 ? "BARONLY" : mode ? "DSMEM" : "L2   ", cs, ny, TW, ms * 1e3 / iters, hc / iters);
        }
      }
    }
  }
  // barrier only
  return 0;
}
