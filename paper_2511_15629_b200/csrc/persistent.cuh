// persistent.cuh -- the whole backward induction (Alg. 1 lines 3-12; its Markov-price form,
// SURVEY.md §8(a) a2-a4) as ONE persistent dataflow kernel: a device-side task scheduler instead of
// 2T kernel boundaries.
//
// Tasks (one 256-thread CTA each):
//   S(t, k, c)   the max-plus stencil of row k, column tile c (256 columns) of stage t (window_item or
//                stencil_item -- the graph path's device code, so results are bit-identical);
//   E(t, rg, cb) W_t rows [16 rg, 16 rg + 16) x columns [64 cb, 64 cb + 64) = P_t V_{t+1} on the FP64
//                tensor cores (dmma2_tile), or, rank-1, 256 columns of the GEMV pi_{t+1} . V_{t+1};
//   OBJ          J (Eq. 6 at t = 0) once V_1 is complete.
// Dependencies are column-local: E(t, ., cb) needs V_{t+1} on its columns (all rows), S(t, k, c) needs
// W_t row k on c's columns plus the action halo [o_min - 1, o_max + 1].  With a single W buffer (no
// keep-values) an E task also waits for every S task of stage t+1 that reads the columns it overwrites.
//
// Scheduling: a ready queue in global memory.  A task is pushed when its last input completes (counters
// s_done[t][c] = finished rows of tile c, e_ready[t][cb] = finished input tiles of E block cb,
// e_cnt[t][rg][c] = finished E blocks of row group rg that tile c reads); idle CTAs pop queue slots in
// order and spin on an empty slot until it is filled.  A popped task is always ready, so every CTA that
// holds a task makes progress and the kernel cannot deadlock whatever the number of resident CTAs; stage
// t-1 starts on the columns stage t has finished while stage t completes the others -- no grid-wide
// barrier, no launch gap.  Producers: __syncthreads, __threadfence, atomics, st.release of the queue
// slot.  Consumers: ld.acquire of the slot, __syncthreads; data produced inside the kernel is read
// through L2 (__ldcg / cp.async.cg).  Task ids: s * period + pos, where pos indexes the host-built
// per-stage pattern (kind, a, b); S entries belong to stage T - s, E entries to stage T - s - 1.
#pragma once
#include "kernels.cuh"
#include "window.cuh"

namespace esdp {

constexpr int kPersistThreads = 256;
constexpr int kDfDR = 2, kDfDC = 4;     // E tile: 16 rows x 64 columns, 8 warps
constexpr int kDfRows = kDfDR * 8, kDfCols = kDfDC * 16;
static_assert(kDfDR * kDfDC * 32 == kPersistThreads, "E tile uses every warp");

enum DfKind : int { kTaskS = 0, kTaskE = 1 };

struct PersistParams {
  StencilParams sp;         // stage-invariant fields; W/V/pol/lambda/g set per task
  WinParams wp;
  int use_window;
  int T, K, S, A, ld, Kp, rows, rank1, kind, keep;
  const double* P;          // [T-1][K][K] (Markov)
  const double* pi;         // rank-1: [T][K]; Markov: [K] (pi_1)
  const double* lambda;     // [T][K]
  const double* g;          // TABLE: [T][K][A]
  double* V;                // keep: [T][Kp][ld], else [2][Kp][ld]
  double* W;                // keep: [T][rows][ld], else [rows][ld]
  int16_t* pol;             // [T][Kp][S]
  double* J;
  int f0, on_grid;
  double w0;
  // schedule (host-built, see esdp.cu build_schedule)
  int ntc, ecw, ncb, nrg, period, ntasks;
  const int* pat;           // [period]: kind | a << 1 | b << 16  (S: a = k, b = c; E: a = rg, b = cb)
  const int* pos_s;         // [K][ntc]: pattern position of S(k, c)
  const int* pos_e;         // [nrg][ncb]: pattern position of E(rg, cb)
  const int* e_need;        // [ntc]: E column blocks (per row group) tile c reads
  const int* e_dep;         // [ncb][2]: S tiles [lo, hi] of stage t+1 an E block waits for
  const int* e_feed;        // [ncb][2]: tiles [lo, hi] whose reads cover the E block
  const int* c_feeds;       // [ntc][2]: E blocks [lo, hi] whose inputs include tile c
  int* ctl;                 // [0] queue head, [1] queue tail, [2] finished tiles of stage 1
  int* s_done;              // [T][ntc]
  int* e_cnt;               // [T][nrg][ntc]
  int* e_ready;             // [T][ncb]
  int* queue;               // [ntasks] task id + 1 (0 = not yet pushed)
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void wait_geq(const int* p, int need) {
  if (ld_acquire(p) >= need) return;
  unsigned ns = 32;
  while (ld_acquire(p) < need) {
    __nanosleep(ns);
    ns = ns < 256 ? 2 * ns : 256;
  }
}

#ifdef ESDP_DF_TRACE
// diagnostic build only: per ticket [grab, inputs ready, done] globaltimer stamps and the SM id
constexpr int kTraceMax = 1 << 18;
__device__ unsigned long long g_df_trace[kTraceMax][4];
__device__ __forceinline__ unsigned long long df_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned df_smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
#define DF_STAMP(j) do { if (tid == 0 && tk < kTraceMax) g_df_trace[tk][j] = df_now(); } while (0)
#else
#define DF_STAMP(j) do { } while (0)
#endif

// release fence for the CTA's writes before they are signalled (bar.sync makes them cumulative); a plain
// __threadfence() is fence.sc.gpu, much slower under load
__device__ __forceinline__ void fence_release() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(kPersistThreads, 4) backward_persistent_kernel(PersistParams pp) {
  extern __shared__ __align__(16) double psm[];
  __shared__ int s_task;
  const int tid = threadIdx.x;
  const size_t RS = (size_t)pp.rows * pp.ld, KS = (size_t)pp.Kp * pp.ld;
  const int obj_id = pp.T * pp.period;
  for (;;) {
    int tk = 0;
    if (tid == 0) {
      const int slot = atomicAdd(pp.ctl, 1);
      int id = -1;
      if (slot < pp.ntasks) {
        const int* q = pp.queue + slot;
        unsigned ns = 32;
        while ((id = ld_acquire(q)) == 0) { __nanosleep(ns); ns = ns < 256 ? 2 * ns : 256; }
        --id;
      }
      s_task = id;
#ifdef ESDP_DF_TRACE
      if (id >= 0 && id < kTraceMax) g_df_trace[id][0] = df_now();
#endif
    }
    __syncthreads();
    tk = s_task;
    if (tk < 0) break;
    DF_STAMP(1);
    if (tk == obj_id) {                                     // OBJ: V_1 complete
      objective_block(pp.V, pp.pi, pp.K, pp.ld, pp.f0, pp.w0, pp.on_grid, pp.J, psm);
      break;                                                // the last task
    }
    const int s = tk / pp.period, pe = __ldg(pp.pat + (tk - s * pp.period));
    const int kind = pe & 1, a = (pe >> 1) & 0x7fff, b = pe >> 16;
    const int t = pp.T - s - kind;                          // S tasks: stage T-s; E tasks: stage T-s-1
    double* Wt = pp.keep ? pp.W + (size_t)(t - 1) * RS : pp.W;
    double* Vt = pp.keep ? pp.V + (size_t)(t - 1) * KS : pp.V + (size_t)((t - 1) & 1) * KS;
    if (kind == kTaskS) {
      int16_t* polt = pp.pol + (size_t)(t - 1) * pp.Kp * pp.S;
      const double* lamt = pp.lambda + (size_t)(t - 1) * pp.K;
      if (pp.use_window) {
        const WinStage st{Wt, Vt, polt, lamt};
        window_item(pp.wp, st, a, b * kWinTile, psm);
      } else {
        StencilParams sp = pp.sp;
        sp.W = Wt; sp.V = Vt; sp.pol = polt; sp.lambda_t = lamt;
        sp.g = pp.kind == 2 ? pp.g + (size_t)(t - 1) * pp.K * pp.A : pp.g;
        stencil_item(sp, a, b * kTile, psm);
      }
    } else {
      const double* Vn = pp.keep ? pp.V + (size_t)t * KS : pp.V + (size_t)(t & 1) * KS;
      if (pp.rank1) {
        gemv_cols(pp.pi + (size_t)t * pp.K, Vn, Wt, pp.K, pp.S, pp.ld, b * pp.ecw + tid);
      } else {
        dmma2_tile<kDfDR, kDfDC, false>(pp.P + (size_t)(t - 1) * pp.K * pp.K, Vn, Wt, pp.rows, pp.K, pp.S, pp.ld,
                                 a * kDfRows, b * kDfCols, psm);
      }
    }
    __syncthreads();
    // completion (warp 0): count, and push every task this one made ready.  The counter updates of one
    // completion go out from different lanes at once, so a push costs ~3 atomic round trips.
    DF_STAMP(3);
    if (tid < 32) {
      const int lane = tid;
      if (lane == 0) fence_release();
      __syncwarp();
      int done = 0;
      if (kind == kTaskS) {
        if (lane == 0) done = atomicAdd(pp.s_done + (size_t)(t - 1) * pp.ntc + b, 1) + 1;
        done = __shfl_sync(0xffffffffu, done, 0);
        if (done == pp.K && t == 1) {
          if (lane == 0 && atomicAdd(pp.ctl + 2, 1) + 1 == pp.ntc)                  // V_1 complete: OBJ
            st_release(pp.queue + atomicAdd(pp.ctl + 1, 1), obj_id + 1);
        }
      }
      // candidates: S -> E blocks of stage t-1 fed by tile b (each needs all its input tiles);
      //             E -> tiles c of stage t whose reads cover block b (each needs e_need[c] blocks)
      const bool fromS = kind == kTaskS;
      if (!fromS || (done == pp.K && t > 1)) {
        const int lo = __ldg((fromS ? pp.c_feeds : pp.e_feed) + 2 * b);
        const int hi = __ldg((fromS ? pp.c_feeds : pp.e_feed) + 2 * b + 1);
        const int per = fromS ? pp.nrg : (pp.rank1 ? pp.K : min(pp.K, (a + 1) * kDfRows) - a * kDfRows);
        for (int c0 = lo; c0 <= hi; c0 += 32) {
          const int x = c0 + lane;
          bool ready = false;
          if (x <= hi) {
            if (fromS) {
              const int need = __ldg(pp.e_dep + 2 * x + 1) - __ldg(pp.e_dep + 2 * x) + 1;
              ready = atomicAdd(pp.e_ready + (size_t)(t - 2) * pp.ncb + x, 1) + 1 == need;
            } else {
              ready = atomicAdd(pp.e_cnt + ((size_t)(t - 1) * pp.nrg + a) * pp.ntc + x, 1) + 1 == __ldg(pp.e_need + x);
            }
          }
          const unsigned m = __ballot_sync(0xffffffffu, ready);
          if (m == 0u) continue;
          const int n = __popc(m) * per;
          int base = 0;
          if (lane == 0) base = atomicAdd(pp.ctl + 1, n);
          base = __shfl_sync(0xffffffffu, base, 0);
          for (int j = lane; j < n; j += 32) {
            const int r = j / per, q = j - r * per;
            const int y = c0 + (__fns(m, 0, r + 1));           // the r-th ready candidate
            int id;
            if (fromS) id = s * pp.period + __ldg(pp.pos_e + q * pp.ncb + y);            // E(t-1, q, y): period T-t
            else id = (pp.T - t) * pp.period + __ldg(pp.pos_s + (size_t)((pp.rank1 ? 0 : a * kDfRows) + q) * pp.ntc + y);
            st_release(pp.queue + base + j, id + 1);
          }
        }
      }
    }
#ifdef ESDP_DF_TRACE
    if (tid == 0 && tk < kTraceMax) g_df_trace[tk][2] = df_now();
#endif
  }
}

}  // namespace esdp
