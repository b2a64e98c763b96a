// batch.cuh -- kernels of a batch context (esdp_create_batch; SURVEY §8(b) esdp_create_batch, cfg5): n
// storage configurations that share T, K, S, lambda, P and pi but each have their own pbar / eta / s0
// and so their own action grid.  Per stage the batch runs ONE expectation launch over all instances --
// V_{t+1} is laid out [K][n][ld], so W_t = P_t V_{t+1} is a single [K] x [n ld] product (the kernel of
// kernels.cuh, unchanged) -- and ONE window-stencil launch over (tile, k, instance).  The per-instance
// stage-invariant parameters live in device memory (BatchInst); everything else is the single-instance
// device code, so every instance is bit-identical to a context of its own.
#pragma once
#include "kernels.cuh"
#include "window.cuh"

namespace esdp {

struct BatchInst {
  WinParams wp;          // window plan (stage-invariant fields; ld = the batch's row stride)
  StencilParams sp;      // brute-force plan (stage-invariant fields)
  SimParams sim;         // simulation tables of this instance (pol = its [T][K][S] slab)
  int f0, on_grid;       // s0 on the grid (objective, Eq. 6 at t = 0)
  double w0;
};

// Block-cooperative copy of a trivially copyable struct from global to shared memory.
template <int NT, class T>
__device__ __forceinline__ void copy_struct(T& dst, const T& src) {   // NT = blockDim.x
  static_assert(sizeof(T) % 4 == 0, "word copy");
  const int* s = reinterpret_cast<const int*>(&src);
  int* d = reinterpret_cast<int*>(&dst);
#pragma unroll
  for (int j = threadIdx.x; j < (int)(sizeof(T) / 4); j += NT) d[j] = __ldg(s + j);
}

// grid (tiles, K, number of window instances); idx maps blockIdx.z to the instance.  W_t / V_t rows are
// [K][n][ld]: instance m's row k starts at base + k * row_stride + m * ld.
// throughput regime (one launch of many instances per stage): 5 blocks per SM (48 registers) measured
// 4.5 % faster than the latency-tuned 4 of window_stencil_kernel on cfg5 (65.1 -> 62.1 ms, 64 instances)
#ifndef ESDP_WIN_MINB_BATCH
#define ESDP_WIN_MINB_BATCH 5
#endif
template <int OPT, bool kLevels>
__global__ void __launch_bounds__(kWinThreads, ESDP_WIN_MINB_BATCH) window_batch_kernel(const BatchInst* __restrict__ bi,
                                                                      const int* __restrict__ idx,
                                                                      const double* Wt, double* Vt,
                                                                      int16_t* pol_base, size_t pol_inst,
                                                                      size_t pol_stage, const double* lam_t,
                                                                      int ld, int row_stride, int rank1) {
  extern __shared__ __align__(16) double wsm[];
  __shared__ WinParams p;
  const int m = __ldg(idx + blockIdx.z);
  copy_struct<kWinThreads>(p, bi[m].wp);
  __syncthreads();
  if (threadIdx.x == 0) {
    p.W = Wt + (size_t)m * ld;
    p.V = Vt + (size_t)m * ld;
    p.pol = pol_base + (size_t)m * pol_inst + pol_stage;
    p.lambda_t = lam_t;
    p.ld = row_stride;
    p.rank1 = rank1;
  }
  __syncthreads();
  window_item<true, OPT, kLevels>(p, blockIdx.y, blockIdx.x * (kWinThreads * OPT), wsm);   // waits for W_t inside
  pdl_trigger();
}
typedef void (*WindowBatchKernel)(const BatchInst*, const int*, const double*, double*, int16_t*, size_t, size_t,
                                  const double*, int, int, int);
inline WindowBatchKernel window_batch_kernel_of(int opt, int levels) {
  if (levels) return window_batch_kernel<1, true>;
  return opt == 4 ? window_batch_kernel<4, false> : opt == 2 ? window_batch_kernel<2, false> : window_batch_kernel<1, false>;
}

// grid (tiles, K, number of brute-force instances): the brute-force stencil of kernels.cuh per instance.
__global__ void __launch_bounds__(kStencilWarps * 32) stencil_batch_kernel(const BatchInst* __restrict__ bi,
                                                                           const int* __restrict__ idx,
                                                                           const double* Wt, double* Vt,
                                                                           int16_t* pol_base, size_t pol_inst,
                                                                           size_t pol_stage, const double* lam_t,
                                                                           int ld, int row_stride, int rank1) {
  extern __shared__ double smem[];
  __shared__ StencilParams p;
  const int m = __ldg(idx + blockIdx.z);
  copy_struct<kStencilWarps * 32>(p, bi[m].sp);
  __syncthreads();
  if (threadIdx.x == 0) {
    p.W = Wt + (size_t)m * ld;
    p.V = Vt + (size_t)m * ld;
    p.pol = pol_base + (size_t)m * pol_inst + pol_stage;
    p.lambda_t = lam_t;
    p.ld = row_stride;
    p.rank1 = rank1;
  }
  pdl_wait();                          // W_t is the previous contraction's output
  __syncthreads();
  stencil_item(p, blockIdx.y, blockIdx.x * kTile, smem);
  pdl_trigger();
}

// J of every instance: one block per instance.
__global__ void objective_batch_kernel(const BatchInst* __restrict__ bi, const double* __restrict__ V1,
                                       const double* __restrict__ pi1, int K, int ld, int row_stride,
                                       double* __restrict__ J) {
  extern __shared__ double vk[];  // [2][K]
  pdl_wait();
  const int m = blockIdx.x;
  objective_block(V1 + (size_t)m * ld, pi1, K, row_stride, __ldg(&bi[m].f0), __ldg(&bi[m].w0), __ldg(&bi[m].on_grid),
                  J + m, vk);
}

// Forward simulation of every instance: grid (path blocks, n); instance m draws with key seed + m and
// writes out[m * n_paths + path] -- the same paths as esdp_simulate(seed + m) on a context of its own.
__global__ void __launch_bounds__(128) simulate_batch_kernel(const BatchInst* __restrict__ bi, int64_t n_paths,
                                                             uint64_t seed, double* __restrict__ out) {
  extern __shared__ __align__(16) double ssm[];
  __shared__ SimParams sp;
  const int m = blockIdx.y;
  copy_struct<128>(sp, bi[m].sim);
  __syncthreads();
  simulate_block(sp, n_paths, seed + (uint64_t)m, out + (size_t)m * n_paths, ssm);
}

}  // namespace esdp
