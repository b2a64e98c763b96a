// kernels.cuh -- sm_100a kernels of the backward induction (arXiv 2511.15629, Alg. 1 in Markov form).
//
// Every floating-point operation on the value path is an explicit round-to-nearest intrinsic
// (__dadd_rn / __dmul_rn / __dsub_rn / __ddiv_rn / __fma_rn) so that nvcc never contracts or
// reassociates: results are reproducible bit for bit (R14/R15).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

// Checked builds (`make EXTRA=-DESDP_CHECK`, tests run against them like the default build): device-side
// bounds and invariant asserts on the indices the hot kernels compute -- the substitute for
// compute-sanitizer, which is closed on this GPU pool.
#ifdef ESDP_CHECK
#include <cassert>
#define ESDP_ASSERT(c) assert(c)
#else
#define ESDP_ASSERT(c) ((void)0)
#endif

namespace esdp {

constexpr int kMaxA = 8191;
constexpr int R = 8;                  // SoC columns per thread in the stencil (register window)
constexpr int kLanes = 32;
constexpr int kTile = kLanes * R;     // 256 SoC columns per stencil block
constexpr int kPad = 8;               // smem guard columns below the lowest offset
constexpr int kStencilWarps = 8;      // action chunks per block (one warp each)

__host__ __device__ __forceinline__ int skew(int j) { return j + (j >> 3); }  // 8-column groups + 1 pad

// Programmatic dependent launch (PDL): a kernel lets its successor be scheduled at once, and waits for
// its predecessor's results only where it first reads them.  Both are no-ops without a PDL launch.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Late trigger: after a block's stores (an early trigger measured slower: dependents hold SM slots)
__device__ __forceinline__ void pdl_trigger_late() { pdl_trigger(); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

#ifdef ESDP_WIN_TRACE
// diagnostic phase marks (tools/wintrace.py): thread 0 of each block of the last launch records
// %globaltimer at mark m (and %smid); which = 0 window stencil, 1 expectation
__device__ unsigned long long g_ktrace[2][4096][8];
__device__ __forceinline__ void ktrace(int which, int m) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const int b = blockIdx.y * gridDim.x + blockIdx.x;
    if (b < 4096) {
      g_ktrace[which][b][m] = t;
      if (m == 0) { unsigned sm; asm("mov.u32 %0, %%smid;" : "=r"(sm)); g_ktrace[which][b][7] = sm; }
    }
  }
}
#else
__device__ __forceinline__ void ktrace(int, int) {}
#endif

// A maximal run of actions whose offsets are consecutive integers decreasing by one and whose
// interpolation weight is 0 ("recombining" interior of Eq. 10), or a single action.
struct Seg {
  int a0;      // first action index
  int n;       // number of actions
  int o0;      // offset of a0 (index units); action a0+m has offset o0 - m  (RUN)
  int interp;  // 1: single action with weight w > 0 (endpoint), 0: RUN / single integral action
};

struct StencilParams {
  const double* W;        // [rows][S] continuation of stage t (rows = K, or 1 in rank-1 mode)
  double* V;              // [K][S] out
  int16_t* pol;           // [K][S] out
  const double* lambda_t; // [K]  lambda_{t,k}
  const double* act;      // [A]
  const double* g;        // [A] (LINEAR_MINUS_G) or [K][A] of stage t (TABLE) or nullptr
  const double* w;        // [A]
  const double* omw;      // [A]
  const int* off;         // [A]
  const Seg* segs;        // [nseg]
  int nseg, A, S, K, kind, rank1, o_min, o_span;  // o_span = o_max - o_min
  int ld;                 // leading dimension of W and V rows (>= S)
};

// ------------------------------------------------------------------------------------------------
// Expectation: W_t[k][i] = sum_{k'} P_t[k][k'] V_{t+1}[k'][i]  (Alg. 1 line 11; Eq. 6)
// canonical ascending-k' fma chain (R15): bit-identical to the oracle.  (FP64 DMMA was measured at
// the same 37 TFLOP/s as DFMA on B200 and would change the summation order.)
// Each output is a K-long dependent DFMA chain (9-cycle latency): the kernel keeps 4 chains per
// thread and prefetches the next 4 k' of operands from shared memory while the current 4 retire.
// Block tile: kRowsC rows x kColsC columns; V tile [Kp][kColsC] staged with 16-byte cp.async
// (V rows have a padded leading dimension ld, a multiple of 4 doubles), P tile [kRowsC][Kp];
// rows k' >= K are zero-filled, which leaves every chain unchanged (fma(0, 0, acc) == acc for acc != -0,
// and the chain starts at +0 and can never reach -0).
// ------------------------------------------------------------------------------------------------
constexpr int kRowsC = 16;
constexpr int kColsC = 32;
constexpr int kThreadsC = (kRowsC / 2) * (kColsC / 2);  // 128, 2x2 outputs per thread

__host__ __device__ __forceinline__ int pad4(int K) { return (K + 3) & ~3; }
inline size_t contract_smem_bytes(int K) { return sizeof(double) * (size_t)pad4(K) * (kRowsC + kColsC); }

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc));
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

__global__ void __launch_bounds__(kThreadsC) contract_kernel(const double* __restrict__ Pt,   // [rows][K]
                                                             const double* __restrict__ Vn,   // [K][ld]
                                                             double* __restrict__ Wt,         // [rows][ld]
                                                             int rows, int K, int S, int ld) {
  extern __shared__ __align__(16) double csm[];
  const int Kp = pad4(K);
  double* vs = csm;                        // [Kp][kColsC]
  double* ps = csm + (size_t)Kp * kColsC;  // [kRowsC][Kp]
  const int i0 = blockIdx.x * kColsC, r0 = blockIdx.y * kRowsC;
  const int tid = threadIdx.x;
  pdl_trigger();
  for (int r = 0; r < kRowsC; ++r) {  // P tile rows (inputs: staged before the dependency wait)
    const bool rin = r0 + r < rows;
    const double* src = Pt + (size_t)(r0 + r) * K;
    for (int kp = tid; kp < Kp; kp += kThreadsC) {
      if (rin && kp < K) cp_async8(ps + r * Kp + kp, src + kp);
      else ps[r * Kp + kp] = 0.0;
    }
  }
  pdl_wait();                          // V_{t+1} is the previous stencil's output
  {  // V tile: 16 two-double chunks per row, 8 rows per pass (no runtime division)
    const int c = 2 * (tid & 15);
    const bool in = i0 + c < ld;
    const double* src = Vn + i0 + c;
    for (int kp = tid >> 4; kp < Kp; kp += kThreadsC / 16) {
      double* dst = vs + kp * kColsC + c;
      if (kp < K && in) cp_async16(dst, src + (size_t)kp * ld);
      else { dst[0] = 0.0; dst[1] = 0.0; }
    }
  }
  cp_async_wait_all();
  __syncthreads();
  const int rr = (tid / (kColsC / 2)) * 2, cc = (tid % (kColsC / 2)) * 2;
  const double* p0 = ps + (size_t)rr * Kp;
  const double* p1 = p0 + Kp;
  double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
  double4 x0 = *reinterpret_cast<const double4*>(p0), x1 = *reinterpret_cast<const double4*>(p1);
  double2 v0 = *reinterpret_cast<const double2*>(vs + 0 * kColsC + cc);
  double2 v1 = *reinterpret_cast<const double2*>(vs + 1 * kColsC + cc);
  double2 v2 = *reinterpret_cast<const double2*>(vs + 2 * kColsC + cc);
  double2 v3 = *reinterpret_cast<const double2*>(vs + 3 * kColsC + cc);
  for (int kp = 0; kp < Kp; kp += 4) {
    // prefetch the next 4 k' (clamped re-read of the last chunk at the end: harmless)
    const int kn = (kp + 4 < Kp) ? kp + 4 : kp;
    const double4 y0 = *reinterpret_cast<const double4*>(p0 + kn), y1 = *reinterpret_cast<const double4*>(p1 + kn);
    const double2 u0 = *reinterpret_cast<const double2*>(vs + (kn + 0) * kColsC + cc);
    const double2 u1 = *reinterpret_cast<const double2*>(vs + (kn + 1) * kColsC + cc);
    const double2 u2 = *reinterpret_cast<const double2*>(vs + (kn + 2) * kColsC + cc);
    const double2 u3 = *reinterpret_cast<const double2*>(vs + (kn + 3) * kColsC + cc);
    a00 = __fma_rn(x0.x, v0.x, a00); a01 = __fma_rn(x0.x, v0.y, a01); a10 = __fma_rn(x1.x, v0.x, a10); a11 = __fma_rn(x1.x, v0.y, a11);
    a00 = __fma_rn(x0.y, v1.x, a00); a01 = __fma_rn(x0.y, v1.y, a01); a10 = __fma_rn(x1.y, v1.x, a10); a11 = __fma_rn(x1.y, v1.y, a11);
    a00 = __fma_rn(x0.z, v2.x, a00); a01 = __fma_rn(x0.z, v2.y, a01); a10 = __fma_rn(x1.z, v2.x, a10); a11 = __fma_rn(x1.z, v2.y, a11);
    a00 = __fma_rn(x0.w, v3.x, a00); a01 = __fma_rn(x0.w, v3.y, a01); a10 = __fma_rn(x1.w, v3.x, a10); a11 = __fma_rn(x1.w, v3.y, a11);
    x0 = y0; x1 = y1; v0 = u0; v1 = u1; v2 = u2; v3 = u3;
  }
  const int i = i0 + cc;
  if (r0 + rr < rows) {
    if (i < S) Wt[(size_t)(r0 + rr) * ld + i] = a00;
    if (i + 1 < S) Wt[(size_t)(r0 + rr) * ld + i + 1] = a01;
  }
  if (r0 + rr + 1 < rows) {
    if (i < S) Wt[(size_t)(r0 + rr + 1) * ld + i] = a10;
    if (i + 1 < S) Wt[(size_t)(r0 + rr + 1) * ld + i + 1] = a11;
  }
}

// ------------------------------------------------------------------------------------------------
// Expectation on the FP64 tensor cores: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  Measured on B200
// (tools/microbench/mb6.cu, 128k outputs with random, wide-range and cancelling operands): each DMMA
// accumulates its 4 products as a sequential fma chain, so a K/4-long chain of DMMAs is bit-identical
// to the canonical ascending-k' fma chain (R15) -- and it issues 256 FMAs per warp instruction instead
// of 32, with 2 operand registers per lane per 4 k'.  Every parity test re-checks the bit equality.
// Fragment layout (PTX ISA, m8n8k4 .f64, row.col): A[8x4] lane -> A[lane/4][lane%4];
// B[4x8] lane -> B[lane%4][lane/4]; C/D[8x8] lane -> C[lane/4][2(lane%4) + {0,1}].
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// Runtime guard of the DMMA bit-exactness the expectation kernels rely on: every warp
// computes one 8 x 8 tile of A B over kProbeQ k'-quads twice -- as the DMMA chain the kernels use and as
// the canonical ascending-k' fma chain (R15) -- and counts the outputs whose bits differ.  A [tiles][8][4Q],
// B [tiles][4Q][8] (host-generated: random signs, wide exponent range, cancelling pairs).
constexpr int kProbeQ = 32;
__global__ void dmma_probe_kernel(const double* __restrict__ A, const double* __restrict__ B, int ntiles,
                                  unsigned* __restrict__ mismatches) {
  const int tile = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (tile >= ntiles) return;
  const double* a = A + (size_t)tile * 8 * 4 * kProbeQ;
  const double* b = B + (size_t)tile * 4 * kProbeQ * 8;
  const int kq = lane & 3, g = lane >> 2;
  double d0 = 0.0, d1 = 0.0;
  for (int q = 0; q < kProbeQ; ++q) dmma_8x8x4(d0, d1, a[g * 4 * kProbeQ + 4 * q + kq], b[(4 * q + kq) * 8 + g]);
  // lane holds C[g][2 kq], C[g][2 kq + 1]
  double c0 = 0.0, c1 = 0.0;
  for (int k = 0; k < 4 * kProbeQ; ++k) {
    c0 = __fma_rn(a[g * 4 * kProbeQ + k], b[k * 8 + 2 * kq], c0);
    c1 = __fma_rn(a[g * 4 * kProbeQ + k], b[k * 8 + 2 * kq + 1], c1);
  }
  const unsigned bad = (__double_as_longlong(c0) != __double_as_longlong(d0)) + (__double_as_longlong(c1) != __double_as_longlong(d1));
  if (bad) atomicAdd(mismatches, bad);
}

// Shared-memory-staged DMMA expectation: a block computes kDR*8 rows x kDC*16 columns of W.  The P rows
// [kDR*8][Kp] and the V tile [Kp][kDC*16] are staged once per block with cp.async (so every L2 byte is
// read by one block, not by every warp), then each warp runs its 8x16 tile's DMMA chain from shared
// memory.  cfg2: 7 x 21 = 147 blocks of 6 warps (one per SM).
// Expectation tiles: DR*8 rows x DC*16 columns per block, DR*DC warps (one 8x16 sub-tile each).  The host
// picks (1, 3) for K <= 128 and (4, 3) above (measured: cfg2 and cfg4 chains).
constexpr int kDR = 1, kDC = 3;            // small-K tile
constexpr int kDRbig = 4, kDCbig = 3;      // large-K tile

// Shared-memory row strides chosen for the DMMA operand loads: a lane (kq, g) reads A[g][kq + 4q] and
// B[kq + 4q][g]; a warp-wide 8-byte load takes at least 2 wavefronts, reached when the 32 addresses are
// distinct mod 16 doubles: A stride = 4 or 12 (mod 16), B stride = 8 (mod 16).
__host__ __device__ constexpr int dmma2_stride_a(int Kp) { return (Kp % 16 == 0 || Kp % 16 == 8) ? Kp + 4 : Kp; }
__host__ __device__ constexpr int dmma2_stride_b(int CB) { return CB + (8 - CB % 16 + 16) % 16; }

inline size_t contract_dmma2_smem(int K, int DR = kDR, int DC = kDC) {
  const int Kp = (K + 3) & ~3;
  return sizeof(double) * ((size_t)(DR * 8) * dmma2_stride_a(Kp) + (size_t)Kp * dmma2_stride_b(DC * 16));
}

// One (DR*8) x (DC*16) tile of W_t = P_t V_{t+1} by DR*DC warps: P rows and the V column block are staged
// in shared memory (cp.async), then every warp runs its 8x16 DMMA chain over k'.  kPdl: the P staging
// (an input) happens before the programmatic dependency wait, the V staging after it.
template <int DR, int DC, bool kPdl>
__device__ __forceinline__ void dmma2_tile(const double* __restrict__ Pt, const double* __restrict__ Vn,
                                           double* __restrict__ Wt, int rows, int K, int S, int ld, int r0, int i0,
                                           double* dsm) {
  constexpr int NT = DR * DC * 32;
  const int Kp = (K + 3) & ~3;
  constexpr int RB = DR * 8, CB = DC * 16, SB = dmma2_stride_b(DC * 16);
  const int SA = dmma2_stride_a(Kp);
  double* as = dsm;                     // [RB][SA]
  double* bs = dsm + (size_t)RB * SA;   // [Kp][SB]
  const int tid = threadIdx.x;
  ktrace(1, 0);
  // P rows (an input), staged before the dependency wait: 16-byte cp.async when K is even (rows then
  // start 16-byte aligned), else 8-byte
  if ((K & 1) == 0) {
    const int hp = Kp >> 1;
    for (int e = tid; e < RB * hp; e += NT) {
      const int r = e / hp, kp = 2 * (e - r * hp);
      double* dst = as + r * SA + kp;
      if (r0 + r < rows && kp < K) cp_async16(dst, Pt + (size_t)(r0 + r) * K + kp);
      else { dst[0] = 0.0; dst[1] = 0.0; }
    }
  } else {
    for (int r = 0; r < RB; ++r) {
      const bool rin = r0 + r < rows;
      const double* src = Pt + (size_t)(r0 + r) * K;
      for (int kp = tid; kp < Kp; kp += NT) {
        if (rin && kp < K) cp_async8(as + r * SA + kp, src + kp);
        else as[r * SA + kp] = 0.0;
      }
    }
  }
  ktrace(1, 1);
  if (kPdl) pdl_wait();
  ktrace(1, 2);
  {  // V tile: CB/2 two-double chunks per row
    constexpr int CH = CB / 2;
    for (int e = tid; e < Kp * CH; e += NT) {
      const int kp = e / CH, c = 2 * (e - kp * CH);
      double* dst = bs + kp * SB + c;
      if (kp < K && i0 + c < ld) cp_async16(dst, Vn + (size_t)kp * ld + i0 + c);
      else { dst[0] = 0.0; dst[1] = 0.0; }
    }
  }
  cp_async_wait_all();
  __syncthreads();
  ktrace(1, 3);
  const int warp = tid >> 5, lane = tid & 31, kq = lane & 3, g = lane >> 2;
  const int wr = warp / DC, wc = warp % DC;             // this warp's 8x16 tile inside the block
  const double* arow = as + (size_t)(wr * 8 + g) * SA + kq;
  const double* bcol = bs + (size_t)kq * SB + wc * 16 + g;
  double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
  const int nq = Kp >> 2;
#pragma unroll 4
  for (int q = 0; q < nq; ++q) {
    const double a = arow[4 * q];
    const double b0 = bcol[(size_t)(4 * q) * SB], b1 = bcol[(size_t)(4 * q) * SB + 8];
    dmma_8x8x4(d00, d01, a, b0);
    dmma_8x8x4(d10, d11, a, b1);
  }
  ktrace(1, 4);
  const int r = r0 + wr * 8 + g;
  if (r < rows) {
    const int c = i0 + wc * 16 + 2 * kq;
    double* wrp = Wt + (size_t)r * ld;
    if (c < S) wrp[c] = d00;
    if (c + 1 < S) wrp[c + 1] = d01;
    if (c + 8 < S) wrp[c + 8] = d10;
    if (c + 9 < S) wrp[c + 9] = d11;
  }
  ktrace(1, 5);
}

template <int DR, int DC>
__global__ void __launch_bounds__(DR * DC * 32) contract_dmma2_kernel(const double* __restrict__ Pt,   // [rows][K]
                                                                     const double* __restrict__ Vn,   // [K][ld]
                                                                     double* __restrict__ Wt,         // [rows][ld]
                                                                     int rows, int K, int S, int ld, int ncb) {
  extern __shared__ __align__(16) double dsm[];
  dmma2_tile<DR, DC, true>(Pt, Vn, Wt, rows, K, S, ld, (blockIdx.x / ncb) * (DR * 8), (blockIdx.x % ncb) * (DC * 16), dsm);
  pdl_trigger();   // late trigger: dependents launch as this grid drains, without holding SM slots early
}

// ------------------------------------------------------------------------------------------------
// Throughput-regime expectation (cfg4, cfg5 batches): register-blocked DMMA with a k'-pipelined
// shared-memory stage.  dmma2 above is built for latency (a few 8x16 warp tiles per block, everything
// staged before the chain starts); on large contractions its 1 A + 2 B fragment loads per 2 DMMAs keep
// the LSU ~75 % busy at the DMMA rate and its 141 KB stage (K = 200) fits one block per SM (ncu on
// cfg4: tensor pipe 42 % of active cycles, short-scoreboard stalls first).  Here a warp owns an
// (8 MT) x (8 NT) tile -- MT A and NT B fragments feed MT*NT DMMAs per k-step -- and the k' dimension
// streams through NS cp.async stages of KC k' each, so several blocks co-reside and the staging of one
// chunk overlaps the chains of the previous ones.  Every accumulator still runs its k'-quads in
// ascending order, one DMMA (4 sequential fmas) after the other: the result is the canonical chain (R15),
// bit for bit, as with dmma2.
// Block: WC warps side by side (columns); tile RB = 8 MT rows x CB = 8 NT WC columns.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int MT, int NT, int WC, int KC, int NS>
struct Dmma3 {
  static constexpr int RB = 8 * MT, CB = 8 * NT * WC, NTH = 32 * WC;
  static constexpr int SA = (KC % 16 == 0 || KC % 16 == 8) ? KC + 4 : KC;   // A rows: stride 4 or 12 mod 16
  static constexpr int SB = CB + (8 - CB % 16 + 16) % 16;                     // B rows: stride 8 mod 16
  static constexpr int STAGE = RB * SA + KC * SB;                             // doubles per stage
  static size_t smem() { return sizeof(double) * (size_t)NS * STAGE; }
};

template <int MT, int NT, int WC, int KC, int NS>
__global__ void __launch_bounds__(32 * WC) contract_dmma3_kernel(const double* __restrict__ Pt,   // [rows][K], K even
                                                                 const double* __restrict__ Vn,   // [K][ld]
                                                                 double* __restrict__ Wt,         // [rows][ld]
                                                                 int rows, int K, int S, int ld, int nrb) {
  using D = Dmma3<MT, NT, WC, KC, NS>;
  static_assert(KC % 4 == 0 && NS >= 2, "k' chunk of whole quads, at least double buffering");
  extern __shared__ __align__(16) double d3sm[];
  const int tid = threadIdx.x;
  const int r0 = (blockIdx.x % nrb) * D::RB, i0 = (blockIdx.x / nrb) * D::CB;   // neighbours share the V tile
  const int nch = (K + KC - 1) / KC;
  // Per-thread copy slots, fixed for the whole kernel: the A piece (row ra, k' pair ka) and the B pieces
  // (rows kb + j*BR, column pair cb); per chunk only the k' bound is checked and the pointers advance.
  // Out-of-range pieces are zero-filled by the copy itself (src-size 0).
  constexpr int AP = 8 * MT * (KC / 2), BP = KC * (D::CB / 2);
  static_assert(AP <= D::NTH || (AP % D::NTH == 0 && D::NTH % (KC / 2) == 0), "A pieces per thread");
  static_assert(D::NTH % (D::CB / 2) == 0 && BP % D::NTH == 0, "B pieces per thread");
  constexpr int NA = AP >= D::NTH ? AP / D::NTH : 1, NB = BP / D::NTH, BR = D::NTH / (D::CB / 2);
  const bool a_thr = tid < AP;
  const int ra = tid / (KC / 2), ka = 2 * (tid % (KC / 2));       // + j * (NTH / (KC/2)) rows for j < NA
  const int kb = tid / (D::CB / 2), cb = 2 * (tid % (D::CB / 2));
  const bool b_col = i0 + cb < ld;
  const double* ga = Pt + (size_t)min(r0 + ra, rows - 1) * K + ka;
  const double* gb = Vn + (size_t)kb * ld + (b_col ? i0 + cb : 0);
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(d3sm);
  auto cp16z = [](unsigned dst, const void* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0));
  };
  auto issue_a = [&](int ch) {   // P rows r0.. of k' chunk ch (an input: may precede the dependency wait)
    if (!a_thr) return;
    const unsigned st = sbase + (unsigned)(sizeof(double) * (size_t)(ch % NS) * D::STAGE);
    const int k = ch * KC + ka;
#pragma unroll
    for (int j = 0; j < NA; ++j) {
      const int r = ra + j * (D::NTH / (KC / 2));
      const bool ok = r0 + r < rows && k < K;
      cp16z(st + (unsigned)(sizeof(double) * (r * D::SA + ka)), ok ? ga + (size_t)j * (D::NTH / (KC / 2)) * K + ch * KC : Pt, ok);
    }
  };
  auto issue_b = [&](int ch) {   // V_{t+1} rows of chunk ch, columns i0..i0+CB
    const unsigned st = sbase + (unsigned)(sizeof(double) * ((size_t)(ch % NS) * D::STAGE + D::RB * D::SA));
    const double* src = gb + (size_t)ch * KC * ld;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int kp = kb + j * BR;
      const bool ok = b_col && ch * KC + kp < K;
      cp16z(st + (unsigned)(sizeof(double) * (kp * D::SB + cb)), ok ? src + (size_t)j * BR * ld : Vn, ok);
    }
  };
  auto As = [&](int b) { return d3sm + (size_t)b * D::STAGE; };
  auto Bs = [&](int b) { return d3sm + (size_t)b * D::STAGE + D::RB * D::SA; };
  // prologue: P chunks of the first NS-1 stages before the wait, V chunks after it; one group per stage
  ktrace(1, 0);
#pragma unroll
  for (int s = 0; s < NS - 1; ++s)
    if (s < nch) issue_a(s);
  ktrace(1, 1);
  pdl_wait();
  ktrace(1, 2);
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    if (s < nch) issue_b(s);
    cp_async_commit();
  }
  const int warp = tid >> 5, lane = tid & 31, kq = lane & 3, g = lane >> 2;
  double acc[MT][NT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    cp_async_wait_group<NS - 2>();   // chunk ch has landed (this thread's copies) ...
    __syncthreads();                 // ... everyone's; and chunk ch-1's buffer is no longer read
    if (ch == 0) ktrace(1, 3);
    if (ch + NS - 1 < nch) { issue_a(ch + NS - 1); issue_b(ch + NS - 1); }
    cp_async_commit();
    const double* as = As(ch % NS) + g * D::SA + kq;
    const double* bs = Bs(ch % NS) + kq * D::SB + warp * (8 * NT) + g;
    const int nq = min(KC, K - ch * KC + 3) >> 2;   // k'-quads of this chunk (zero quads past K skipped)
#pragma unroll
    for (int q = 0; q < KC / 4; ++q) {
      if (q < nq) {
        double a[MT], b[NT];
#pragma unroll
        for (int m = 0; m < MT; ++m) a[m] = as[m * 8 * D::SA + 4 * q];
#pragma unroll
        for (int n = 0; n < NT; ++n) b[n] = bs[4 * q * D::SB + 8 * n];
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
          for (int n = 0; n < NT; ++n) dmma_8x8x4(acc[m][n][0], acc[m][n][1], a[m], b[n]);
      }
    }
  }
  cp_async_wait_group<0>();
  ktrace(1, 4);
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    const int r = r0 + m * 8 + g;
    if (r >= rows) continue;
    double* wr = Wt + (size_t)r * ld;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int c = i0 + warp * (8 * NT) + n * 8 + 2 * kq;   // even, ld % 4 == 0: 16-byte aligned
      if (c + 1 < S) *reinterpret_cast<double2*>(wr + c) = make_double2(acc[m][n][0], acc[m][n][1]);
      else if (c < S) wr[c] = acc[m][n][0];
    }
  }
  ktrace(1, 5);
  pdl_trigger_late();
}

// ------------------------------------------------------------------------------------------------
// P-resident persistent expectation for wide products with K <= 8 MTA (the cfg5 batch GEMM: [100] x
// [128,512] per stage).  One CTA per SM keeps the whole P_t in shared memory (loaded once, before the
// dependency wait: P is an input) and walks column tiles of CT = 8 NW columns, double-buffering the V_{t+1}
// tile with cp.async; warp w owns the tile's columns [8w, 8w + 8) for every row (MTA 8-row fragments, one
// B fragment per k'-quad).  V_{t+1} is then read from L2 once per column (the 16 x 128 block tiles re-read it
// once per row block), and each k'-quad issues MTA DMMAs for MTA + 1 shared loads.  Each accumulator runs its
// k'-quads in ascending order, one DMMA after the other: the canonical chain (R15), as in dmma2/dmma3.
// ------------------------------------------------------------------------------------------------
template <int MTA, int NW, int NT = 1>
struct DmmaPres {
  static constexpr int CT = 8 * NT * NW, NTH = 32 * NW;
  static constexpr int SB = CT + (8 - CT % 16 + 16) % 16;   // B rows: stride 8 mod 16 (conflict-free)
  __host__ __device__ static int kp(int K) { return (K + 3) & ~3; }
  __host__ __device__ static int sa(int K) { const int k = kp(K); return (k % 16 == 0 || k % 16 == 8) ? k + 4 : k; }   // 4 or 12 mod 16
  static size_t smem(int K) { return sizeof(double) * ((size_t)8 * MTA * sa(K) + (size_t)2 * kp(K) * SB); }
};

template <int MTA, int NW, int NT = 1>
__global__ void __launch_bounds__(32 * NW, 1) contract_pres_kernel(const double* __restrict__ Pt,   // [rows][K], K even
                                                                  const double* __restrict__ Vn,   // [K][ld]
                                                                  double* __restrict__ Wt,         // [rows][ld]
                                                                  int rows, int K, int ncols, int ld) {
  using D = DmmaPres<MTA, NW, NT>;
  extern __shared__ __align__(16) double psm[];
  const int Kp = D::kp(K), SA = D::sa(K);
  double* As = psm;                                   // [8 MTA][SA]: all of P_t, zero rows / k' past the ends
  double* Bs = psm + (size_t)8 * MTA * SA;            // [2][Kp][SB]: V_{t+1} column tiles
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, kq = lane & 3, g = lane >> 2;
  ESDP_ASSERT(rows <= 8 * MTA && (K & 1) == 0 && blockDim.x == D::NTH);
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(psm);
  auto cp16z = [](unsigned dst, const void* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0));
  };
  {   // P_t: 8 MTA rows x Kp/2 pairs
    const int np = Kp / 2;
    for (int e = tid; e < 8 * MTA * np; e += D::NTH) {
      const int r = e / np, k2 = 2 * (e - r * np);
      const bool ok = r < rows && k2 < K;
      cp16z(sbase + (unsigned)(sizeof(double) * (r * SA + k2)), ok ? Pt + (size_t)r * K + k2 : Pt, ok);
    }
  }
  const int ntiles = (ncols + D::CT - 1) / D::CT;
  auto issue_b = [&](int tile, int st) {   // rows k' < Kp of columns [tile CT, tile CT + CT)
    const unsigned dst0 = sbase + (unsigned)(sizeof(double) * ((size_t)8 * MTA * SA + (size_t)st * Kp * D::SB));
    const int c0 = tile * D::CT;
    constexpr int np = D::CT / 2;
    for (int e = tid; e < Kp * np; e += D::NTH) {
      const int k = e / np, c2 = 2 * (e - k * np);
      const bool ok = k < K && c0 + c2 < ncols;   // ncols even or the last pair inside ld (ld % 4 == 0)
      cp16z(dst0 + (unsigned)(sizeof(double) * (k * D::SB + c2)), ok ? Vn + (size_t)k * ld + c0 + c2 : Vn, ok);
    }
  };
  pdl_wait();
  int tile = blockIdx.x;
  if (tile < ntiles) issue_b(tile, 0);
  cp_async_commit();                                  // group: P_t + the first V tile
  for (int j = 0; tile < ntiles; tile += gridDim.x, ++j) {
    const int nxt = tile + gridDim.x;
    if (nxt < ntiles) issue_b(nxt, (j + 1) & 1);
    cp_async_commit();
    cp_async_wait_group<1>();                         // tile j (and P_t) landed, this thread's copies ...
    __syncthreads();                                  // ... and everyone's
    const double* bs = Bs + (size_t)(j & 1) * Kp * D::SB + kq * D::SB + warp * (8 * NT) + g;
    const double* as = As + g * SA + kq;
    double acc[MTA][NT][2];
#pragma unroll
    for (int m = 0; m < MTA; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    for (int q = 0; q < Kp / 4; ++q) {
      double b[NT];
#pragma unroll
      for (int n = 0; n < NT; ++n) b[n] = bs[4 * q * D::SB + 8 * n];
#pragma unroll
      for (int m = 0; m < MTA; ++m) {
        const double a = as[m * 8 * SA + 4 * q];
#pragma unroll
        for (int n = 0; n < NT; ++n) dmma_8x8x4(acc[m][n][0], acc[m][n][1], a, b[n]);
      }
    }
#pragma unroll
    for (int m = 0; m < MTA; ++m) {
      const int r = m * 8 + g;
      if (r >= rows) continue;
      double* wr = Wt + (size_t)r * ld;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int c = tile * D::CT + warp * (8 * NT) + 8 * n + 2 * kq;   // even, ld % 4 == 0: 16-byte aligned
        if (c + 1 < ncols) *reinterpret_cast<double2*>(wr + c) = make_double2(acc[m][n][0], acc[m][n][1]);
        else if (c < ncols) wr[c] = acc[m][n][0];
      }
    }
    __syncthreads();                                  // stage j & 1 is refilled by the copies of tile j + 2
  }
  cp_async_wait_group<0>();
  pdl_trigger_late();
}

// mbarrier helpers (shared-memory barriers completed by async copies or tensor-core commits)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}

__device__ __forceinline__ void gemv_cols(const double* __restrict__ pi, const double* __restrict__ Vn,
                                          double* __restrict__ Wt, int K, int S, int ld, int i) {
  if (i >= S) return;
  double acc = 0.0;
  for (int kp = 0; kp < K; ++kp) acc = __fma_rn(__ldg(pi + kp), __ldcg(Vn + (size_t)kp * ld + i), acc);
  Wt[i] = acc;
}

// ------------------------------------------------------------------------------------------------
// Max-plus action reduction with argmax (Alg. 1 lines 7-10; Eq. 5):
//   V_t[k][i] = max_a pay(t,k,a) + Wint(i,a,k),  pol = smallest maximizing a  (R8).
// The W row is staged in shared memory with -inf outside [0, S-1]: an infeasible action
// (Alg. 1 line 8) then yields -inf and can never win, exactly like skipping it.
// Grid: (ceil(S/256), K).  Block: 4 warps; warp c reduces action chunk c for 256 columns
// (8 consecutive columns per lane, register window over the recombining run), then the four
// partial (value, index) pairs are merged in ascending chunk order with a strict '>'.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void upd(double c, int a, double& best, int& arg) {
  if (c > best) { best = c; arg = a; }
}

// One group of R steps of a recombining run.  wl = this lane's view of the skewed tile
// (wl[u] = tile index lane*R + c with u = c + (c >> 3)); base_c = tile offset of (column lane*R,
// current step) minus lane*R (warp-uniform).  Step d evaluates action a + d; column r reads W at
// lane-relative tile offset base_c - d + r.
template <bool kMask>
__device__ __forceinline__ void run_group(const double* __restrict__ wl, const double* __restrict__ pay,
                                          int base_c, int a, int m_left, double (&hi)[R], double (&best)[R],
                                          int (&arg)[R]) {
  double lo[R], p[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int c = base_c - R + q;                 // >= 0 by construction (kPad >= R)
    lo[q] = wl[c + (c >> 3)];
    p[q] = pay[a + q];
  }
#pragma unroll
  for (int d = 0; d < R; ++d) {
    const double pd = kMask ? ((d < m_left) ? p[d] : -INFINITY) : p[d];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double x = (r - d >= 0) ? hi[r - d] : lo[R + r - d];
      upd(__dadd_rn(pd, x), a + d, best[r], arg[r]);
    }
  }
#pragma unroll
  for (int q = 0; q < R; ++q) hi[q] = lo[q];
}

// One (k, 256-column tile) item of the brute-force stencil, executed by a 256-thread block.
__device__ __forceinline__ void stencil_item(const StencilParams& prm, int k, int i0, double* smem) {
  const int L = kTile + prm.o_span + kPad + 1;
  double* ws = smem;                           // skew(L) doubles
  double* pay = ws + skew(L) + 8;              // A + 8 doubles
  double* pv = pay + prm.A + 8;                // [kStencilWarps][skew(kTile)]
  int* pa = (int*)(pv + kStencilWarps * skew(kTile));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  const double lam = prm.lambda_t[k];
  for (int a = tid; a < prm.A; a += blockDim.x) {
    double p;
    if (prm.kind == 2) p = prm.g[(size_t)k * prm.A + a];                               // TABLE
    else if (prm.kind == 1) p = __dsub_rn(__dmul_rn(lam, prm.act[a]), prm.g[a]);        // lambda p - g
    else p = __dmul_rn(lam, prm.act[a]);                                                 // lambda p
    pay[a] = p;
  }
  const double* Wrow = prm.W + (prm.rank1 ? 0 : (size_t)k * prm.ld);
  const int g0 = i0 + prm.o_min - kPad;  // global column of tile index 0
  for (int j = tid; j < L; j += blockDim.x) {
    int col = g0 + j;
    ws[skew(j)] = (col >= 0 && col < prm.S) ? __ldcg(Wrow + col) : -INFINITY;
  }
  __syncthreads();

  double best[R];
  int arg[R];
#pragma unroll
  for (int r = 0; r < R; ++r) { best[r] = -INFINITY; arg[r] = -1; }
  const int a_lo = (prm.A * warp) / kStencilWarps, a_hi = (prm.A * (warp + 1)) / kStencilWarps;
  const double* wl = ws + lane * (R + 1);          // skew(lane*R + c) = lane*(R+1) + c + (c>>3)
  const int cbase = kPad - prm.o_min;              // lane-relative tile offset of offset 0

  for (int s = 0; s < prm.nseg; ++s) {
    const Seg sg = prm.segs[s];
    const int sb = max(sg.a0, a_lo), se = min(sg.a0 + sg.n, a_hi);
    if (sb >= se) continue;
    if (sg.interp || sg.n < 4) {
      for (int a = sb; a < se; ++a) {
        const int c0 = cbase + sg.o0 - (a - sg.a0);
        const double p = pay[a];
        if (sg.interp) {
          const double w = prm.w[a], om = prm.omw[a];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int c = c0 + r;
            const double x0 = wl[c + (c >> 3)], x1 = wl[(c + 1) + ((c + 1) >> 3)];
            const double wi = __dadd_rn(__dmul_rn(om, x0), __dmul_rn(w, x1));
            upd(__dadd_rn(p, wi), a, best[r], arg[r]);
          }
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int c = c0 + r;
            upd(__dadd_rn(p, wl[c + (c >> 3)]), a, best[r], arg[r]);
          }
        }
      }
      continue;
    }
    // recombining run: action a = sb + m has offset o(sb) - m
    int base_c = cbase + sg.o0 - (sb - sg.a0);
    double hi[R];
#pragma unroll
    for (int q = 0; q < R; ++q) { const int c = base_c + q; hi[q] = wl[c + (c >> 3)]; }
    int a = sb;
    for (; a + R <= se; a += R, base_c -= R) run_group<false>(wl, pay, base_c, a, R, hi, best, arg);
    if (a < se) run_group<true>(wl, pay, base_c, a, se - a, hi, best, arg);
  }

  // merge the chunk partials in ascending action order (strict '>' keeps the smallest index)
#pragma unroll
  for (int r = 0; r < R; ++r) {
    pv[warp * skew(kTile) + skew(lane * R + r)] = best[r];
    pa[warp * skew(kTile) + skew(lane * R + r)] = arg[r];
  }
  __syncthreads();
  for (int c = tid; c < kTile; c += blockDim.x) {
    const int i = i0 + c;
    if (i >= prm.S) continue;
    double b = -INFINITY;
    int ar = -1;
#pragma unroll
    for (int w = 0; w < kStencilWarps; ++w) {
      double v = pv[w * skew(kTile) + skew(c)];
      if (v > b) { b = v; ar = pa[w * skew(kTile) + skew(c)]; }
    }
    prm.V[(size_t)k * prm.ld + i] = b;
    prm.pol[(size_t)k * prm.S + i] = (int16_t)ar;
  }
}

__global__ void __launch_bounds__(kStencilWarps * 32) stencil_kernel(StencilParams prm) {
  extern __shared__ double smem[];
  pdl_wait();                          // W_t is the previous contraction's output
  stencil_item(prm, blockIdx.y, blockIdx.x * kTile, smem);
  pdl_trigger();
}

inline size_t stencil_smem_bytes(int A, int o_span) {
  int L = kTile + o_span + kPad + 1;
  return sizeof(double) * (size_t)(skew(L) + 8 + A + 8 + kStencilWarps * skew(kTile)) +
         sizeof(int) * (size_t)(kStencilWarps * skew(kTile));
}

// ------------------------------------------------------------------------------------------------
// Objective J = sum_k pi_1[k] V_1(s0, k) (Eq. 6 at t = 0), fma chain in k order; s0 off the
// grid is interpolated per k (R24).  One thread.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void objective_block(const double* __restrict__ V1, const double* __restrict__ pi1, int K,
                                                int ld, int f, double w0, int on_grid, double* __restrict__ J,
                                                double* vk /* smem [2][K] */) {
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const double* row = V1 + (size_t)k * ld;
    vk[k] = on_grid ? __ldcg(row + f)
                    : __dadd_rn(__dmul_rn(__dsub_rn(1.0, w0), __ldcg(row + f)), __dmul_rn(w0, __ldcg(row + f + 1)));
    vk[K + k] = pi1[k];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double acc = 0.0;
  for (int k = 0; k < K; ++k) acc = __fma_rn(vk[K + k], vk[k], acc);
  *J = acc;
}

__global__ void objective_kernel(const double* __restrict__ V1, const double* __restrict__ pi1, int K, int ld,
                                 int f, double w0, int on_grid, double* __restrict__ J) {
  extern __shared__ double vk[];  // [2][K]: V_1(s0, k) and pi_1[k], gathered in parallel
  pdl_wait();
  objective_block(V1, pi1, K, ld, f, w0, on_grid, J, vk);
}

// ------------------------------------------------------------------------------------------------
// Bid curves (Eqs. 7-12): one thread per request (t, i, k).  The caller's output rows
// serve as the hull stack (vert: action index, price: hull u value, overwritten by prices).
// ------------------------------------------------------------------------------------------------
struct BidParams {
  const double* Wall;     // [T][wrows][ld]
  const double* act; const double* w; const double* omw; const int* off; const double* g;
  int T, K, S, A, rank1, kind, ld;
  int wrows, k_lo, k_cnt;  // W rows per stage and this rank's price states [k_lo, k_lo + k_cnt)
};

// Per-action data staged in shared memory for the bid-curve kernel.
struct BidAct {
  const double* act; const double* w; const double* omw; const double* g; const int* off;
};

// u_a = Wint(i, a) - g_a (Eq. 7 with the non-linear part of the payoff, R13); feasible if both
// interpolation nodes lie on the grid (Eq. 4 / Alg. 1 line 8).  Wrow is indexed by global column.
__device__ __forceinline__ bool bid_point(const BidAct& ba, int S, int kind, const double* Wrow, int i, int a,
                                          double& u) {
  const int o = ba.off[a];
  const double wa = ba.w[a];
  if (i + o < 0 || i + o + (wa != 0.0 ? 1 : 0) > S - 1) return false;
  u = (wa == 0.0) ? Wrow[i + o] : __dadd_rn(__dmul_rn(ba.omw[a], Wrow[i + o]), __dmul_rn(wa, Wrow[i + o + 1]));
  if (kind == 1) u = __dsub_rn(u, ba.g[a]);
  return true;
}

constexpr int kBidThreads = 128;

// stack entries: 8-bit action indices when A <= 255, else 16-bit
inline size_t bid_smem_bytes(int A, int o_span, bool stack_in_smem, size_t idx_bytes) {
  return (((size_t)A * (4 * sizeof(double) + sizeof(int)) + 15) & ~(size_t)15) + sizeof(double) * (kBidThreads + o_span + 4) +
         (stack_in_smem ? idx_bytes * (size_t)A * kBidThreads : 0) + 64;
}

// Per-action tables of the bid-curve kernel (shared memory).
struct BidTables {
  const double* act; const double* w; const double* omw; const double* g;
  const int* ow;          // 2 o_a + [w_a != 0]
};

// The monotone chain and the price emission of one curve (t, i, k): Wi points at column i of the W row
// (shared memory when the block staged its segment, else global), bs at this thread's stack column.
template <bool kSmem, typename IdxT, bool kG>
__device__ __forceinline__ void bid_curve(const BidTables& tb, const double* Wi, IdxT* bs, unsigned bstride, int a_lo,
                                          int a_hi, int16_t* __restrict__ vo, double* __restrict__ qo,
                                          double* __restrict__ pro, int64_t nout, int32_t* __restrict__ nvo) {
  auto u_of = [&](int a) -> double {                 // Eq. 7 point value, a known feasible
    const int ow = tb.ow[a];
    const double* wp = Wi + (ow >> 1);
    double u = wp[0];
    if (ow & 1) u = __dadd_rn(__dmul_rn(tb.omw[a], u), __dmul_rn(tb.w[a], wp[1]));
    if (kG) u = __dsub_rn(u, tb.g[a]);
    return u;
  };
  auto st_set = [&](int j, int a) { if (kSmem) bs[(unsigned)j * bstride] = (IdxT)a; else vo[(size_t)j * nout] = (int16_t)a; };
  auto st_get = [&](int j) -> int { return kSmem ? (int)bs[(unsigned)j * bstride] : (int)vo[(size_t)j * nout]; };
  int nh = 0;
  int ao = -1, ab = -1;          // vertices nh-2 (o) and nh-1 (b)
  double uo = 0.0, ub = 0.0, po = 0.0, pb = 0.0;
  double dp = 0.0, du = 0.0;     // fl(pb - po), fl(ub - uo): the cross product's stack-side factors
  for (int a = a_lo; a <= a_hi; ++a) {
    const double u = u_of(a), pc = tb.act[a];
    while (nh >= 2) {
      const double cr = __dsub_rn(__dmul_rn(dp, __dsub_rn(u, uo)), __dmul_rn(du, __dsub_rn(pc, po)));
      if (cr < 0.0) break;
      --nh;                      // pop b; o becomes the top, the vertex below o resurfaces
      ab = ao; ub = uo; pb = po;
      if (nh >= 2) {
        ao = st_get(nh - 2);
        uo = u_of(ao);
        po = tb.act[ao];
        dp = __dsub_rn(pb, po); du = __dsub_rn(ub, uo);
      }
    }
    ESDP_ASSERT(nh <= a_hi - a_lo);
    st_set(nh, a);
    if (nh >= 1) { ao = ab; uo = ub; po = pb; }
    ab = a; ub = u; pb = pc;
    ++nh;
    if (nh >= 2) { dp = __dsub_rn(pb, po); du = __dsub_rn(ub, uo); }
  }
  // emit vertices, quantities and segment prices (Eq. 12) with the running-max repair (R20)
  int a_prev = st_get(0);
  double u_prev = u_of(a_prev);
  double p_prev = tb.act[a_prev], prev_price = 0.0;
  // curve outputs are written once and read by the host or a later kernel: streaming stores (evict-first
  // in L2), so that 0.5 GB of cfg2 curves do not push the policy table out before the simulation
  if (kSmem) __stcs(vo, (short)a_prev);
  if (qo) __stcs(qo, p_prev);
  // two segments per step: their divisions are independent (the repair is a running max after them)
  int j2 = 1;
  for (; j2 + 1 < nh; j2 += 2) {
    const int a1 = st_get(j2), a2 = st_get(j2 + 1);
    const double u1 = u_of(a1), p1 = tb.act[a1], u2 = u_of(a2), p2 = tb.act[a2];
    double r1 = -__ddiv_rn(__dsub_rn(u1, u_prev), __dsub_rn(p1, p_prev));
    double r2 = -__ddiv_rn(__dsub_rn(u2, u1), __dsub_rn(p2, p1));
    if (j2 > 1 && r1 < prev_price) r1 = prev_price;
    if (r2 < r1) r2 = r1;
    __stcs(pro + (size_t)(j2 - 1) * nout, r1);
    __stcs(pro + (size_t)j2 * nout, r2);
    if (kSmem) { __stcs(vo + (size_t)j2 * nout, (short)a1); __stcs(vo + (size_t)(j2 + 1) * nout, (short)a2); }
    if (qo) { __stcs(qo + (size_t)j2 * nout, p1); __stcs(qo + (size_t)(j2 + 1) * nout, p2); }
    prev_price = r2; u_prev = u2; p_prev = p2;
  }
  for (int j = j2; j < nh; ++j) {
    const int a = st_get(j);
    const double u = u_of(a), pc = tb.act[a];
    double pj = -__ddiv_rn(__dsub_rn(u, u_prev), __dsub_rn(pc, p_prev));
    if (j > 1 && pj < prev_price) pj = prev_price;
    __stcs(pro + (size_t)(j - 1) * nout, pj);
    if (kSmem) __stcs(vo + (size_t)j * nout, (short)a);
    if (qo) __stcs(qo + (size_t)j * nout, pc);
    prev_price = pj; u_prev = u; p_prev = pc;
  }
  *nvo = nh;
}

// One thread per requested curve.  The monotone chain keeps its two top vertices in registers and the
// rest of the stack as action indices in shared memory (column-major per thread: conflict-free); u of a
// deeper vertex is recomputed from its index when it resurfaces.  When every request of the block is on
// the same (t, k) row (the common "all i of a stage" case) the W row segment is staged in shared memory.
// kSmem = false: the stack lives in the caller's vert row (A > 255: occupancy, see launch_bids).  kG: payoff lambda p - g(p)
// (u = Wint - g_a, R13), else u = Wint.  Per-action offset and interpolation flag share one word.
template <bool kSmem, typename IdxT, bool kG>
__global__ void __launch_bounds__(kBidThreads) bidcurve_kernel(BidParams bp, int64_t n, const int32_t* __restrict__ req,
                                                               const int32_t* __restrict__ slot, int64_t nout,
                                                               int cap, int o_min, int o_span,
                                                               int32_t* __restrict__ nvert, int16_t* __restrict__ vert,
                                                               double* __restrict__ q, double* __restrict__ price) {
  // request rq writes output slot `slot[rq]` (or rq) of the vertex-major arrays [cap][nout]
  extern __shared__ __align__(16) unsigned char bsm_raw[];
  const int A = bp.A;
  double* s_act = (double*)bsm_raw;                  // shared-memory offsets only (no integer casts), so
  double* s_w = s_act + A;                           // every table access compiles to LDS/STS
  double* s_omw = s_w + A;
  double* s_g = s_omw + A;
  int* s_ow = (int*)(s_g + A);
  double* s_wt = (double*)(bsm_raw + (((size_t)A * 36 + 15) & ~(size_t)15));
  const int nwt = kBidThreads + o_span + 4;
  IdxT* bst = (IdxT*)(s_wt + nwt);
  __shared__ int s_tk[2], s_imin, s_imax, s_uniform;
  (void)cap;

  for (int a = threadIdx.x; a < A; a += blockDim.x) {
    const double wa = bp.w[a];
    s_act[a] = bp.act[a]; s_w[a] = wa; s_omw[a] = bp.omw[a]; s_ow[a] = 2 * bp.off[a] + (wa != 0.0 ? 1 : 0);
    if (kG) s_g[a] = bp.g[a];
  }
  const int64_t rq = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = rq < n;
  int t = 0, i = 0, k = 0;
  if (active) { t = req[3 * rq + 0]; i = req[3 * rq + 1]; k = req[3 * rq + 2]; }
  const bool valid = active && t >= 1 && t <= bp.T && i >= 0 && i < bp.S && k >= 0 && k < bp.K &&
                     (bp.rank1 || (k >= bp.k_lo && k < bp.k_lo + bp.k_cnt));
  if (threadIdx.x == 0) {
    s_tk[0] = t; s_tk[1] = k; s_imin = 1 << 30; s_imax = -1; s_uniform = 1;
  }
  __syncthreads();
  if (valid) { atomicMin(&s_imin, i); atomicMax(&s_imax, i); }
  if (active && (!valid || t != s_tk[0] || (k != s_tk[1] && !bp.rank1))) s_uniform = 0;
  __syncthreads();
  const bool staged = s_uniform && s_imax >= 0 && (s_imax - s_imin) < kBidThreads;
  const int c0 = s_imin + o_min;
  if (staged) {
    const double* Wb = bp.Wall + ((size_t)(s_tk[0] - 1) * bp.wrows + (bp.rank1 ? 0 : s_tk[1] - bp.k_lo)) * bp.ld;
    for (int x = threadIdx.x; x < nwt; x += blockDim.x) {
      const int col = c0 + x;
      s_wt[x] = (col >= 0 && col < bp.S) ? Wb[col] : 0.0;
    }
  }
  __syncthreads();
  const int64_t so = slot ? (int64_t)slot[rq < n ? rq : 0] : rq;
  if (!valid) { if (active) nvert[so] = -1; return; }
  // feasible actions of row i form one interval [a_lo, a_hi]: the offsets o_a and ceil(e_a) = o_a + [w_a > 0]
  // are non-increasing in a (F is decreasing), so Eq. 4's two bounds cut a prefix and a suffix
  int a_hi, a_lo;
  {
    int lo = 0, hi = A;                              // first a with o_a < -i  -> a_hi = that - 1
    while (lo < hi) { const int m = (lo + hi) >> 1; if ((s_ow[m] >> 1) < -i) hi = m; else lo = m + 1; }
    a_hi = lo - 1;
    lo = 0; hi = A;                                  // first a with o_a + [w_a > 0] <= S-1-i
    while (lo < hi) { const int m = (lo + hi) >> 1; const int ow = s_ow[m]; if ((ow >> 1) + (ow & 1) <= bp.S - 1 - i) hi = m; else lo = m + 1; }
    a_lo = lo;
  }
  const BidTables tb{s_act, s_w, s_omw, s_g, s_ow};
  // outputs are vertex-major ([cap][nout]: entry j of curve so at j*nout + so) so that a warp's 32 curves
  // write 32 consecutive words per vertex (coalesced)
  IdxT* bs = bst + threadIdx.x;
  double* qo = q ? q + so : nullptr;
  if (staged)
    bid_curve<kSmem, IdxT, kG>(tb, s_wt + (i - c0), bs, blockDim.x, a_lo, a_hi, vert + so, qo, price + so, nout, nvert + so);
  else
    bid_curve<kSmem, IdxT, kG>(tb, bp.Wall + ((size_t)(t - 1) * bp.wrows + (bp.rank1 ? 0 : k - bp.k_lo)) * bp.ld + i, bs,
                               blockDim.x, a_lo, a_hi, vert + so, qo, price + so, nout, nvert + so);
}

// ------------------------------------------------------------------------------------------------
// Forward simulation (R16/R17): one thread per path, Philox4x32-10.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
}

// The two draws of (path, t): 53-bit integers m (the sampler decides on them) and u = m 2^-53 (exact).
__device__ __forceinline__ void sim_uniforms(uint64_t seed, int64_t path, int t, double& u1, double& u2, uint64_t& m1,
                                             uint64_t& m2) {
  uint32_t c[4] = {(uint32_t)((uint64_t)path & 0xffffffffu), (uint32_t)((uint64_t)path >> 32), (uint32_t)t,
                   0x45534450u};
  philox4x32_10(c, (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
  m1 = (((uint64_t)c[0]) << 21) | (c[1] >> 11);
  m2 = (((uint64_t)c[2]) << 21) | (c[3] >> 11);
  u1 = (double)m1 * 0x1p-53;
  u2 = (double)m2 * 0x1p-53;
}
__device__ __forceinline__ void sim_uniforms(uint64_t seed, int64_t path, int t, double& u1, double& u2) {
  uint64_t m1, m2;
  sim_uniforms(seed, path, t, u1, u2, m1, m2);
}

// Sampling tables (DESIGN R17 and §5 "a7"): a cdf row is the running sum of a P (or pi) row in ascending
// order with the last entry forced to 1 (bit-identical to the oracle's), and a draw is the first j with
// u < cdf[j].  The guide splits [0, 1) into G = 2^g buckets of the draw's 53-bit integer m (u = m 2^-53):
// bucket b holds m in [b 2^s, (b+1) 2^s), s = 53 - g.  Its 64-bit entry decides most draws with ONE load:
//   bits 63..49  j_lo = the first j with cdf[j] > b 2^-g (the answer for the bucket's smallest m)
//   bits 48..43  dl:  0  the whole bucket maps to j_lo ("pure")
//                     1..62  one boundary inside: m < T ? j_lo : j_lo + dl, with T = ceil(cdf[j_lo] 2^53)
//                        (u < cdf[j_lo] <=> m < T, exactly) and j_lo + dl the next state of larger cdf
//                     63  several boundaries: scan the cdf row from j_lo (as the definition reads)
//   bits 42..0   T - b 2^s, aligned to 43 bits (exact when s <= 43; else truncated, and a draw that
//                ties the truncated bits compares u with cdf[j_lo] itself).
// One block per row; rows are (table u, state k), read from P row (src[u] K + k) (src: the stage whose
// slice a deduplicated table u stands for; NULL: u itself).
constexpr int kCdfThreads = 128;   // one block per sampling row
constexpr int kCdfSmemK = 1024;    // rows up to this K are staged in shared memory
constexpr int kGuideJ = 49, kGuideD = 43;
constexpr uint64_t kGuideThr = (1ull << kGuideD) - 1;
// One sampling row per block: the cumulative sums (ascending, the definition's order; the last entry is 1),
// then the 2^g guide entries, every thread walking its interleaved buckets from its previous answer.
// Blocks [0, rows) build rows of q (src: deduplicated slices, NULL: row r of q); block `rows` (if q1)
// builds the single row q1 (pi_1) -- both jobs of a load in one launch.
template <bool kSmem>
__global__ void __launch_bounds__(kCdfThreads) cdf_kernel(const double* __restrict__ q, const int* __restrict__ src,
                                                        int64_t rows, int K, int g, double* __restrict__ cdf,
                                                        uint64_t* __restrict__ guide, const double* __restrict__ q1,
                                                        int g1, double* __restrict__ cdf1, uint64_t* __restrict__ guide1) {
  __shared__ double cdf_sm[kSmem ? kCdfSmemK : 1];
  const int64_t r = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31;
  const double* qr;
  double* cg;
  uint64_t* gr;
  if (r < rows) {
    const int64_t u = r / K, k = r - u * K;
    qr = q + ((src ? (int64_t)src[u] : u) * K + k) * K;
    cg = cdf + r * K;
    gr = guide + (r << g);
  } else {   // the single-row job
    qr = q1; cg = cdf1; gr = guide1; g = g1;
  }
  double* cr = kSmem ? cdf_sm : cg;
  if (tid < 32) {
    if (kSmem) {   // every lane forms the same sequential sum over broadcast values and keeps its entries
      double sum = 0.0;
      for (int j0 = 0; j0 < K; j0 += 32) {
        const int j = j0 + lane;
        const double v = j < K ? __ldg(qr + j) : 0.0;
        const int n = min(32, K - j0);
        double mine = 0.0;
        for (int l = 0; l < n; ++l) {
          sum = __dadd_rn(sum, __shfl_sync(0xffffffffu, v, l));
          if (l == lane) mine = sum;
        }
        if (j < K) {
          const double c = (j == K - 1) ? 1.0 : mine;
          cr[j] = c;
          cg[j] = c;
        }
      }
    } else if (lane == 0) {
      double sum = 0.0;
      for (int j = 0; j < K; ++j) {
        sum = __dadd_rn(sum, qr[j]);
        cr[j] = (j == K - 1) ? 1.0 : sum;
      }
    }
  }
  __syncthreads();
  const int s = 53 - g;
  const double inv = ldexp(1.0, -g);
  int jl = 0;                                      // this thread's previous answer: monotone in the bucket
  for (int b = tid; b < (1 << g); b += kCdfThreads) {   // interleaved buckets: coalesced 8-byte stores
    const double lo = (double)b * inv, hi = (double)(b + 1) * inv;   // exact (powers of two)
    while (!(lo < cr[jl])) ++jl;                   // first j with lo < cdf[j] (cdf[K-1] = 1 > lo): a short walk
                                                   // from this thread's last bucket, not a binary search
    const double cl = cr[jl];
    uint64_t e = (uint64_t)jl << kGuideJ;
    if (cl < hi) {                                 // a boundary inside the bucket
      int jh = jl + 1;
      while (jh < K && !(cr[jh] > cl)) ++jh;       // next state of larger cdf (skips empty states)
      if (jh < K && jh - jl <= 62 && !(cr[jh] < hi)) {
        const uint64_t T = (uint64_t)ceil(cl * 0x1p53), thr = T - ((uint64_t)b << s);   // in [1, 2^s]
        if (thr < (1ull << s))                     // thr == 2^s: every m of the bucket is below T (pure)
          e |= ((uint64_t)(jh - jl) << kGuideD) | (s <= kGuideD ? thr << (kGuideD - s) : thr >> (s - kGuideD));
      } else {
        e |= 63ull << kGuideD;
      }
    }
    gr[b] = e;
  }
}

// rows of q (and, if q1, the single row q1) in one launch
inline void launch_cdf(const double* q, const int* src, int64_t rows, int K, int g, double* cdf, uint64_t* guide,
                       cudaStream_t s, const double* q1 = nullptr, int g1 = 0, double* cdf1 = nullptr,
                       uint64_t* guide1 = nullptr) {
  const int64_t nb = rows + (q1 ? 1 : 0);
  if (nb <= 0) return;
  if (K <= kCdfSmemK)
    cdf_kernel<true><<<(unsigned)nb, kCdfThreads, 0, s>>>(q, src, rows, K, g, cdf, guide, q1, g1, cdf1, guide1);
  else
    cdf_kernel<false><<<(unsigned)nb, kCdfThreads, 0, s>>>(q, src, rows, K, g, cdf, guide, q1, g1, cdf1, guide1);
}

// first j in [0, K) with u < cdf[j] (m: the draw's 53-bit integer, u = m 2^-53); gs = 53 - g.  Split into the
// guide load and its decoding, so a caller can issue the load early and work while it is in flight.
__device__ __forceinline__ int cdf_decode(const double* __restrict__ cdf, uint64_t e, int gs, uint64_t m, double u) {
  int j = (int)(e >> kGuideJ);
  const int dl = (int)(e >> kGuideD) & 63;
  if (dl == 0) return j;
  if (dl < 63) {
    const uint64_t thr = e & kGuideThr, ml = m & ((1ull << gs) - 1);
    if (gs <= kGuideD) return (ml << (kGuideD - gs)) < thr ? j : j + dl;
    const uint64_t x = ml >> (gs - kGuideD);
    if (x != thr) return x < thr ? j : j + dl;
    return u < __ldg(cdf + j) ? j : j + dl;        // tie on the truncated bits: compare exactly
  }
  while (!(u < __ldg(cdf + j))) ++j;               // several boundaries: the definition, from j_lo
  ESDP_ASSERT(u < 1.0);                            // the last cdf entry is 1: the scan stops inside the row
  return j;
}
__device__ __forceinline__ int cdf_sample(const double* __restrict__ cdf, const uint64_t* __restrict__ guide, int gs,
                                          uint64_t m, double u) {
  return cdf_decode(cdf, __ldg(guide + (m >> gs)), gs, m, u);
}

struct SimParams {
  const int16_t* pol;    // [T][K][S]
  const double* cdf;     // Markov: [T-1][K][K]; rank-1: [T][K] (row t = cdf of pi_{t+1})
  const uint64_t* guide; // same rows, 2^g entries each
  const double* cdf1;    // [K] cdf of pi_1
  const uint64_t* guide1; // [2^g]
  const int* tab;        // Markov: table of stage t's transitions (deduplicated slices); NULL: t - 1
  const double* lambda;  // [T][K]
  const double* act; const double* w; const int* off; const double* g;
  int T, K, S, A, gs, gs1, rank1, kind, on_grid, f0;   // gs / gs1 = 53 - g: guide bucket shifts (rows / pi_1)
  int Kp;                // policy rows per stage (K, or world * kmax after a multi-GPU backward)
  double w0;
};

// sampling-table row of the transition out of state k at stage t (t < T): rank-1 rows are the marginals
// pi_{t+1}; Markov rows the (deduplicated) slice of P_t
__device__ __forceinline__ size_t sim_row(const SimParams& sp, int t, int k) {
  return sp.rank1 ? (size_t)t : (size_t)(sp.tab ? __ldg(sp.tab + t - 1) : t - 1) * sp.K + k;
}

// One block of paths: blockIdx.x * blockDim.x + threadIdx.x (ssm: the per-action tables).
__device__ __forceinline__ void simulate_block(const SimParams& sp, int64_t n, uint64_t seed, double* __restrict__ out,
                                               double* ssm) {
  double* s_act = ssm;
  double* s_w = s_act + sp.A;
  double* s_g = s_w + sp.A;
  int* s_off = (int*)(s_g + sp.A);
  for (int a = threadIdx.x; a < sp.A; a += blockDim.x) {
    s_act[a] = sp.act[a]; s_w[a] = sp.w[a]; s_off[a] = sp.off[a];
    s_g[a] = sp.kind == 1 ? sp.g[a] : 0.0;
  }
  __syncthreads();
  const int64_t path = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (path >= n) return;
  double u1, u2;
  uint64_t m1, m2;
  sim_uniforms(seed, path, 0, u1, u2, m1, m2);
  int k = cdf_sample(sp.cdf1, sp.guide1, sp.gs1, m1, u1);
  int i = sp.on_grid ? sp.f0 : sp.f0 + (u2 < sp.w0 ? 1 : 0);
  double profit = 0.0;
  const size_t KS = (size_t)sp.Kp * sp.S;
  sim_uniforms(seed, path, 1, u1, u2, m1, m2);
  // stage t's table row base (sim_row(t, 0)) is loaded one stage ahead: the map load stays off the
  // draw's dependent chain
  size_t rb_next = sp.T > 1 ? sim_row(sp, 1, 0) : 0;
  for (int t = 1; t <= sp.T; ++t) {
    // both loads of the stage first (the policy entry, the price draw's guide entry), then the next stage's
    // draws -- they do not depend on the state -- while the loads are in flight, then the decoding
    ESDP_ASSERT(k >= 0 && k < sp.K && i >= 0 && i < sp.S);
    const int a = __ldg(sp.pol + (size_t)(t - 1) * KS + (size_t)k * sp.S + i);
    ESDP_ASSERT(a >= 0 && a < sp.A);
    const double lam = sp.kind == 2 ? 0.0 : __ldg(sp.lambda + (size_t)(t - 1) * sp.K + k);
    const size_t rb = rb_next;
    const size_t row = sp.rank1 ? rb : rb + k;
    const uint64_t ge = t < sp.T ? __ldg(sp.guide + (row << (53 - sp.gs)) + (m2 >> sp.gs)) : 0ull;
    if (t + 1 < sp.T) rb_next = sim_row(sp, t + 1, 0);
    const double u1t = u1, u2t = u2;
    const uint64_t m2t = m2;
    if (t < sp.T) sim_uniforms(seed, path, t + 1, u1, u2, m1, m2);
    const int kn = t < sp.T ? cdf_decode(sp.cdf + row * sp.K, ge, sp.gs, m2t, u2t) : k;
    double p;
    if (sp.kind == 2) p = __ldg(sp.g + ((size_t)(t - 1) * sp.K + k) * sp.A + a);
    else {
      p = __dmul_rn(lam, s_act[a]);
      if (sp.kind == 1) p = __dsub_rn(p, s_g[a]);
    }
    profit = __dadd_rn(profit, p);
    const double wa = s_w[a];
    i = i + s_off[a] + ((wa > 0.0 && u1t < wa) ? 1 : 0);
    k = kn;
  }
  out[path] = profit;
}

__global__ void __launch_bounds__(128) simulate_kernel(SimParams sp, int64_t n, uint64_t seed, double* __restrict__ out) {
  extern __shared__ __align__(16) double ssm[];   // per-action tables: act, w, g (kind 1), off
  simulate_block(sp, n, seed, out, ssm);
}

// Price-state paths of the lottery / strategy simulations (same draws as simulate_block): k_t and the
// realised price lambda_{t,k_t} of every path; kp / lamp: [T][n] (either may be null).
__global__ void __launch_bounds__(128) price_path_kernel(SimParams sp, int64_t n, uint64_t seed, int16_t* __restrict__ kp,
                                                         double* __restrict__ lamp) {
  const int64_t path = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (path >= n) return;
  double u1, u2;
  uint64_t m1, m2;
  sim_uniforms(seed, path, 0, u1, u2, m1, m2);
  int k = cdf_sample(sp.cdf1, sp.guide1, sp.gs1, m1, u1);
  for (int t = 1; t <= sp.T; ++t) {
    if (kp) kp[(size_t)(t - 1) * n + path] = (int16_t)k;
    if (lamp) lamp[(size_t)(t - 1) * n + path] = __ldg(sp.lambda + (size_t)(t - 1) * sp.K + k);
    if (t < sp.T) {
      sim_uniforms(seed, path, t, u1, u2, m1, m2);
      const size_t row = sim_row(sp, t, k);
      k = cdf_sample(sp.cdf + row * sp.K, sp.guide + (row << (53 - sp.gs)), sp.gs, m2, u2);
    }
  }
}

inline size_t sim_smem_bytes(int A) { return (size_t)A * (3 * sizeof(double) + sizeof(int)) + 16; }

// stats = {mean, M2 / (n - 1)} (the sample variance; 0 for one path), on the device.
__global__ void finalize_stats_kernel(const double* __restrict__ red, int64_t n, double* __restrict__ stats) {
  stats[0] = red[0];
  stats[1] = n > 1 ? red[1] / (double)(n - 1) : 0.0;
}

// Deterministic two-pass reduction of per-path profits: sum (then sum of squared deviations).
__global__ void reduce_kernel(const double* __restrict__ x, int64_t n, const double* __restrict__ mean_in,
                              double* __restrict__ out) {
  __shared__ double sh[1024];
  double acc = 0.0;
  const double m = mean_in ? *mean_in : 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    double v = x[j];
    if (mean_in) { double d = __dsub_rn(v, m); v = __dmul_rn(d, d); }
    acc = __dadd_rn(acc, v);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = mean_in ? sh[0] : __ddiv_rn(sh[0], (double)n);
}

}  // namespace esdp
