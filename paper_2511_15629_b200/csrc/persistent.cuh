// persistent.cuh -- the whole backward induction as ONE cooperative kernel (one CTA set resident on
// every SM for all T stages).  Per stage t = T..1:
//   phase E: W_t = P_t V_{t+1} (warp tiles on the FP64 tensor cores, or the rank-1 GEMV), W_T = 0
//   grid barrier
//   phase S: V_t, pol_t from W_t (one 256-thread block per (k, 256-column) item; window or brute force)
//   grid barrier
// then J (Eq. 6 at t = 0) in block 0.  It replaces the 2T kernel launches of the graph path (measured
// ~1.5-2 us of fixed cost each on B200) by 2T grid barriers.  The per-item device code
// is exactly the graph path's (stencil_item / window_item / dmma_tile), so results are bit-identical.
// Data written inside the kernel is read through L2 (__ldcg); grid.sync() fences at GPU scope.
#pragma once
#include <cooperative_groups.h>

#include "kernels.cuh"
#include "window.cuh"

namespace esdp {

constexpr int kPersistThreads = 256;

struct PersistParams {
  StencilParams sp;         // stage-invariant fields; W/V/pol/lambda/g set per stage
  WinParams wp;
  int use_window;
  int T, K, S, A, ld, rows, rank1, kind, keep;
  const double* P;          // [T-1][K][K] (Markov)
  const double* pi;         // rank-1: [T][K]; Markov: [K] (pi_1)
  const double* lambda;     // [T][K]
  const double* g;          // TABLE: [T][K][A]
  double* V;                // keep: [T][K][ld], else [2][K][ld]
  double* W;                // keep: [T][rows][ld], else [rows][ld]
  int16_t* pol;             // [T][K][S]
  double* J;
  int f0, on_grid;
  double w0;
  unsigned long long* stamps;   // nullable: [T][3] globaltimer at stage start / after E / after S (block 0)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kPersistThreads, 2) backward_persistent_kernel(PersistParams pp) {
  extern __shared__ __align__(16) double psm[];
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, gwarp = b * (kPersistThreads / 32) + (tid >> 5), nwarps = G * (kPersistThreads / 32);
  const size_t RS = (size_t)pp.rows * pp.ld, KS = (size_t)pp.K * pp.ld;
  const int ntc = (pp.S + kTile - 1) / kTile;     // stencil column tiles (kTile == kWinTile == 256)
  const int nct = (pp.S + 15) / 16;               // DMMA column tiles
  const int etiles = ((pp.rows + 7) / 8) * nct;
  for (int t = pp.T; t >= 1; --t) {
    if (pp.stamps && b == 0 && tid == 0) pp.stamps[(size_t)(t - 1) * 3 + 0] = gtimer();
    double* Wt = pp.keep ? pp.W + (size_t)(t - 1) * RS : pp.W;
    double* Vt = pp.keep ? pp.V + (size_t)(t - 1) * KS : pp.V + (size_t)((t - 1) & 1) * KS;
    // ---- phase E: expectation ----
    if (t == pp.T) {
      for (size_t e = (size_t)b * kPersistThreads + tid; e < RS; e += (size_t)G * kPersistThreads) Wt[e] = 0.0;
    } else {
      const double* Vn = pp.keep ? pp.V + (size_t)t * KS : pp.V + (size_t)(t & 1) * KS;
      if (pp.rank1) {
        const double* pit = pp.pi + (size_t)t * pp.K;       // pi_{t+1}
        for (int i = b * kPersistThreads + tid; i < pp.S; i += G * kPersistThreads) gemv_cols(pit, Vn, Wt, pp.K, pp.S, pp.ld, i);
      } else {
        const double* Pt = pp.P + (size_t)(t - 1) * pp.K * pp.K;
        for (int tile = gwarp; tile < etiles; tile += nwarps)
          dmma_tile(Pt, Vn, Wt, pp.rows, pp.K, pp.S, pp.ld, nct, tile, lane);
      }
    }
    grid.sync();
    if (pp.stamps && b == 0 && tid == 0) pp.stamps[(size_t)(t - 1) * 3 + 1] = gtimer();
    // ---- phase S: max-plus stencil ----
    int16_t* polt = pp.pol + (size_t)(t - 1) * pp.K * pp.S;
    const double* lamt = pp.lambda + (size_t)(t - 1) * pp.K;
    if (pp.use_window) {
      WinParams wp = pp.wp;
      wp.W = Wt; wp.V = Vt; wp.pol = polt; wp.lambda_t = lamt;
      for (int item = b; item < pp.K * ntc; item += G) {
        window_item(wp, item / ntc, (item % ntc) * kWinTile, psm);
        __syncthreads();
      }
    } else {
      StencilParams sp = pp.sp;
      sp.W = Wt; sp.V = Vt; sp.pol = polt; sp.lambda_t = lamt;
      sp.g = pp.kind == 2 ? pp.g + (size_t)(t - 1) * pp.K * pp.A : pp.g;
      for (int item = b; item < pp.K * ntc; item += G) {
        stencil_item(sp, item / ntc, (item % ntc) * kTile, psm);
        __syncthreads();
      }
    }
    grid.sync();
    if (pp.stamps && b == 0 && tid == 0) pp.stamps[(size_t)(t - 1) * 3 + 2] = gtimer();
  }
  if (b == 0) {
    const double* V1 = pp.V;   // stage 1 lives at offset 0 in both layouts
    objective_block(V1, pp.pi, pp.K, pp.ld, pp.f0, pp.w0, pp.on_grid, pp.J, psm);
  }
}

}  // namespace esdp
