// window.cuh -- exact O(log A)-per-cell max-plus stencil for the recombining action grid.
//
// Same result as stencil_kernel (V and the smallest-index argmax, bit for bit), computed without
// visiting every (i, a) cell.  On the interior of the Eq. 10 grid the charge actions have
// integral SoC offsets o = 1..Lc and powers p = -o*delta/eta_c (up to rounding), the discharge actions
// o = -1..-Ld and p = -o*delta*eta_d.  With the linear payoff lambda*p the candidate of row i is
//     cand(i, o) = lambda*p(o) + W[i+o]  ~=  key(j) + beta*i,   j = i + o,   key(j) = W[j] - beta*j,
// with beta_c = lambda*delta/eta_c on the charge side and beta_d = lambda*delta*eta_d on the discharge
// side: a sliding-window maximum of a per-column key over a fixed-width window.  Each side keeps a
// sparse table of packed (key, position) maxima over power-of-two ranges: a window maximum is two
// lookups, and the runner-up (needed for the exactness test) is the maximum of the window minus its
// argmax (two more).
//
// Exactness.  The key form rounds differently from the canonical candidate fl(fl(lambda p) + W), by
// at most eps = 32 u (max|W| + |lambda| delta (S + span) / min(eta) + |lambda| pbar) plus the packed-key
// truncation 2^-41 (max|W| + |lambda| delta (S + span) / min(eta)).
// The remaining actions (zero action, the interpolated endpoints +-pbar, anything irregular) are
// evaluated canonically.  If the best approximate value beats the second best by more than 2 eps, the
// canonical argmax is that action and is unique; V is then recomputed canonically from it.  Otherwise
// (near ties) the row falls back to the full canonical scan in ascending a with a strict '>'.  Either
// way V and pol equal the oracle's bit for bit.
#pragma once
#include "kernels.cuh"

namespace esdp {

#ifndef ESDP_WIN_THREADS
#define ESDP_WIN_THREADS 256
#endif
#ifndef ESDP_WIN_MINB
#define ESDP_WIN_MINB 4
#endif
constexpr int kWinTile = ESDP_WIN_THREADS;     // output columns per block
__device__ unsigned long long g_window_fallbacks;  // rows that needed the full canonical scan (diagnostic)
__device__ unsigned long long g_window_level_tables;  // run tables that were not unimodal (built levels)
constexpr int kWinThreads = ESDP_WIN_THREADS;  // one output column per thread in the query phase
constexpr int kLevelSlots = (kWinTile + 512 + 2 * kWinThreads - 1) / (2 * kWinThreads);  // pairs per thread

constexpr int kMaxSingles = 16;

__device__ __forceinline__ void wtrace(int m) { ktrace(0, m); }  // singles staged in shared memory (more: read from global)

// static data of a single (canonically evaluated) action, carried in the kernel parameters so the
// block reads it from the constant bank instead of a dependent global gather
struct WinSingle {
  double act, w, omw;
  int off, a;
};

struct WinParams {
  const double* W; double* V; int16_t* pol; const double* lambda_t;
  const double* act; const double* w; const double* omw; const int* off;
  const int* singles;   // action indices evaluated canonically (zero action, endpoints, irregular)
  const int* live;      // all live action indices, ascending (fallback scan)
  int nsingle, nlive, A, S, K, rank1, ld;
  int a_z, Lc, Ld, pc, pd;  // zero action; run lengths; sparse-table levels (2^pc <= Lc < 2^(pc+1))
  int o_min, o_max;         // tile halo over all live actions
  double delta, eta_c, eta_d, pbar;
  double dc, dd;            // delta / eta_c and delta * eta_d (for the approximate keys only)
  double jspan;             // S + span + 2: bounds |j| over the tile, so |beta * j| <= |beta| jspan
  const double* g;          // [A] degradation g_a (LINEAR_MINUS_G): pay = fl(fl(lambda p) - g) when g_kind
  const double* gfit;       // [6] affine fit of g on the runs: gc0, gc1, gd0, gd1, max deviation, max |g|
  int g_kind;               // 1: payoff lambda p - g(p) (kind LINEAR_MINUS_G), 0: lambda p
  WinSingle sg[kMaxSingles];  // static data of singles[0 .. min(nsingle, kMaxSingles))
};

// Packed keys: an order-preserving 64-bit image of the (approximate) value with its table position in
// the low 10 bits.  One unsigned max then yields the maximum and where it is.  Clearing the low bits
// lowers the value by less than 1024 ulp; that truncation is added to the exactness margin below.
constexpr unsigned long long kPosMask = 1023ull;

__device__ __forceinline__ unsigned long long ord64(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord64(unsigned long long k) {  // below ord64(-DBL_MAX): -inf / empty range
  k &= ~kPosMask;
  if (k < 0x0010000000000000ull) return -INFINITY;
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}
__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) { return a > b ? a : b; }
// packed key of a value at table position pos (branch-free ord64 on the 32-bit halves; -inf packs below
// every finite key and decodes back to -inf)
__device__ __forceinline__ unsigned long long pack_key(double v, int pos) {
  const int hi = __double2hiint(v), lo = __double2loint(v);
  const int m = hi >> 31;                                   // 0 (v >= +0) or -1 (v <= -0)
  const unsigned h = (unsigned)(hi ^ (m | (int)0x80000000)), l = (unsigned)(lo ^ m);
  return ((((unsigned long long)h << 32) | l) & ~kPosMask) | (unsigned long long)pos;
}

// Sparse table over power-of-two ranges: level q entry x = max of packed keys in [x, x + 2^q).
// Rows are ns = n rounded up to even entries apart, so every row starts 16-byte aligned (pair access).
struct RangeMax {
  unsigned long long* v;   // [levels][ns]
  int n, ns;
  __device__ __forceinline__ unsigned long long query(int l, int r) const {   // 0 if l > r
    if (l > r) return 0ull;
    const int q = 31 - __clz(r - l + 1);
    const unsigned long long* row = v + q * ns;
    return umax64(row[l], row[r - (1 << q) + 1]);
  }
};

inline int window_levels(int L) { int q = 0; while ((2 << q) <= L) ++q; return q + 1; }

inline size_t window_smem_bytes(int Lc, int Ld, int o_span) {
  const size_t nw = (kWinTile + o_span + 2 + 1) & ~(size_t)1;
  const size_t nc = (kWinTile + Lc + 1) & ~(size_t)1, nd = (kWinTile + Ld + 1) & ~(size_t)1;
  return sizeof(double) * nw + sizeof(unsigned long long) * (window_levels(Lc) * nc + window_levels(Ld) * nd) + 64;
}

__device__ __forceinline__ double canon_single(const WinParams& p, const double* __restrict__ wt, int wbase, int i,
                                               int a, double lam) {
  // canonical candidate fl(pay + Wint), pay = fl(fl(lambda p_a) - g_a) (R14), -inf if infeasible (tile
  // is -inf padded)
  const int o = __ldg(p.off + a);
  const double wa = __ldg(p.w + a);
  const int x = i + o - wbase;
  const double wint = (wa == 0.0) ? wt[x] : __dadd_rn(__dmul_rn(__ldg(p.omw + a), wt[x]), __dmul_rn(wa, wt[x + 1]));
  double pay = __dmul_rn(lam, __ldg(p.act + a));
  if (p.g_kind) pay = __dsub_rn(pay, __ldg(p.g + a));
  return __dadd_rn(pay, wint);
}

// a single action's data staged in shared memory for the whole block
struct SingleAct {
  double pay;   // fl(fl(lambda * p_a) - g_a) for this block's k (R14; g = 0 for the linear payoff)
  double w, omw;
  int off, a;
};

__device__ __forceinline__ double canon_staged(const SingleAct& s, const double* __restrict__ wt, int wbase, int i) {
  const int x = i + s.off - wbase;
  const double wint = (s.w == 0.0) ? wt[x] : __dadd_rn(__dmul_rn(s.omw, wt[x]), __dmul_rn(s.w, wt[x + 1]));
  return __dadd_rn(s.pay, wint);
}

// level q of a table: entry x = max(level q-1 at x, at x + 2^(q-1)), for x <= n - 2^q.  Straight-line,
// two entries per thread and slot with 16-byte shared-memory accesses: x = 2 tid, 2 tid + 512 (n <= 768).
__device__ __forceinline__ void build_level(const RangeMax& t, int q, int tid) {
  const int h = 1 << (q - 1), lim = t.n - (1 << q);
  const unsigned long long* pv = t.v + (q - 1) * t.ns;
  unsigned long long* nv = t.v + q * t.ns;
#pragma unroll
  for (int u = 0; u < kLevelSlots; ++u) {
    const int x = 2 * (tid + u * kWinThreads);
    if (x <= lim) {
      const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(pv + x);
      ulonglong2 b;
      if (h == 1) { b.x = a.y; b.y = pv[x + 2]; }
      else b = *reinterpret_cast<const ulonglong2*>(pv + x + h);
      ulonglong2 r;
      r.x = umax64(a.x, b.x);
      r.y = umax64(a.y, b.y);
      if (x + 1 <= lim) *reinterpret_cast<ulonglong2*>(nv + x) = r;
      else nv[x] = r.x;
    }
  }
}

// levels q and q + 1 of a table in one pass from level q - 1 (h = 2^(q-1)): entry x of level q is
// max(L[x], L[x+h]) for x <= n - 2^q, of level q + 1 max(L[x], L[x+h], L[x+2h], L[x+3h]) for
// x <= n - 2^(q+1).  Halves the barriers between the level builds.
__device__ __forceinline__ void build_level2(const RangeMax& t, int q, int tid) {
  const int h = 1 << (q - 1), lim1 = t.n - (1 << q), lim2 = t.n - (2 << q);
  const unsigned long long* pv = t.v + (q - 1) * t.ns;
  unsigned long long* n1 = t.v + q * t.ns;
  unsigned long long* n2 = n1 + t.ns;
#pragma unroll
  for (int u = 0; u < kLevelSlots; ++u) {
    const int x = 2 * (tid + u * kWinThreads);
    if (x <= lim1) {
      const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(pv + x);
      ulonglong2 b;
      if (h == 1) { b.x = a.y; b.y = pv[x + 2]; }
      else b = *reinterpret_cast<const ulonglong2*>(pv + x + h);
      ulonglong2 r;
      r.x = umax64(a.x, b.x);
      r.y = umax64(a.y, b.y);
      if (x + 1 <= lim1) *reinterpret_cast<ulonglong2*>(n1 + x) = r;
      else n1[x] = r.x;
      if (x <= lim2) {
        // level q at x + 2h, from the same level q - 1 entries
        const ulonglong2 c = *reinterpret_cast<const ulonglong2*>(pv + x + 2 * h);
        ulonglong2 d;
        if (h == 1) { d.x = c.y; d.y = pv[x + 4]; }
        else d = *reinterpret_cast<const ulonglong2*>(pv + x + 3 * h);
        ulonglong2 e;
        e.x = umax64(r.x, umax64(c.x, d.x));
        e.y = umax64(r.y, umax64(c.y, d.y));
        if (x + 1 <= lim2) *reinterpret_cast<ulonglong2*>(n2 + x) = e;
        else n2[x] = e.x;
      }
    }
  }
}

// top-2 of the window [l, r] of table t: best (value, table position) and the runner-up value
__device__ __forceinline__ void window_top2(const RangeMax& t, int l, int r, double& m1, int& pos, double& m2) {
  const unsigned long long k1 = t.query(l, r);
  pos = (int)(k1 & kPosMask);
  m1 = unord64(k1);
  m2 = unord64(umax64(t.query(l, pos - 1), t.query(pos + 1, r)));
}

// Unimodal tables (the common case: W_t(., k) concave in the SoC, as for every linear-payoff workload
// measured -- tests/diag/unimodal.py finds 100 % of cfg2 / cfg4 / cfg5 tiles unimodal, cfg3's fixed cost
// 52 % / 73 % per side).  With ck(key) = 0 for -inf keys, a table is unimodal when every rising pair
// (x, x+1) precedes every falling pair; its maximum then sits at p* = 1 + the last rising x (0 if none),
// the maximum of any window [l, r] at clamp(p*, l, r) and the runner-up next to it.  Packed keys are
// distinct (positions in the low bits), so these are exactly the two largest keys the sparse-table
// queries return -- the same values, positions and decisions -- and a unimodal table needs no levels.
__device__ __forceinline__ unsigned long long ckey(unsigned long long k) { return k < 0x0010000000000000ull ? 0ull : k; }
// pair (idx - 1, idx): a rise records idx in up (max), a fall in dn (min)
__device__ __forceinline__ void uni_pair(unsigned long long a, unsigned long long b, unsigned idx, unsigned& up, unsigned& dn) {
  a = ckey(a);
  b = ckey(b);
  up = b > a ? umax(up, idx) : up;
  dn = b < a ? umin(dn, idx) : dn;
}
constexpr unsigned kNoFall = 0xffffu;

__device__ __forceinline__ void window_top2_uni(const RangeMax& t, int pstar, int l, int r, double& m1, int& pos,
                                                double& m2) {
  if (l > r) { pos = 0; m1 = m2 = -INFINITY; return; }   // empty run (as query() on an empty range)
  const int q = min(max(pstar, l), r);
  pos = q;
  m1 = unord64(t.v[q]);
  m2 = unord64(umax64(q > l ? t.v[q - 1] : 0ull, q < r ? t.v[q + 1] : 0ull));
}

// One (k, 256-column tile) item of the window stencil, executed by a 256-thread block.  kWait: the
// programmatic dependency wait (W_t is the previous kernel's output) is taken here, after the input loads
// (lambda, the g fit) are issued; the W loads follow it at once, and the singles come from the kernel
// parameters, so the block pays one memory latency before its first barrier.
struct WinStage {          // the per-stage pointers of an item (the rest of WinParams is stage-invariant)
  const double* W; double* V; int16_t* pol; const double* lambda_t;
};

template <bool kWait = false>
__device__ __forceinline__ void window_item(const WinParams& p, const WinStage& st, int k, int i0, double* wsm) {
  const int tid = threadIdx.x;
  wtrace(0);
  const int nw = kWinTile + (p.o_max - p.o_min) + 2;
  const int lc = p.pc + 1, ldl = p.pd + 1;
  RangeMax tc, td;
  tc.n = kWinTile + p.Lc;                  // charge table: columns [i0 + 1, i0 + nc]
  td.n = kWinTile + p.Ld;                  // discharge table: columns [i0 - Ld, i0 + kWinTile)
  tc.ns = (tc.n + 1) & ~1;
  td.ns = (td.n + 1) & ~1;
  double* wt = wsm;                        // W over columns [wbase, wbase + nw)
  tc.v = (unsigned long long*)(wt + ((nw + 1) & ~1));
  td.v = tc.v + (size_t)lc * tc.ns;
  __shared__ unsigned red[kWinThreads / 32];
  __shared__ unsigned ured[4][kWinThreads / 32];   // unimodality: rises (max) and falls (min) per table
  __shared__ SingleAct ss[kMaxSingles];

  const double* Wrow = st.W + (p.rank1 ? 0 : (size_t)k * p.ld);
  const int wbase = i0 + p.o_min;
  // inputs first (lambda_t and the g fit do not depend on the previous kernel)
  const double lam = st.lambda_t[k];
  const double gc0 = p.gfit[0], gc1 = p.gfit[1], gd0 = p.gfit[2], gd1 = p.gfit[3];
  if (kWait) pdl_wait();
  wtrace(1);
  // W_t over the tile: all of this thread's loads are issued before anything waits on them
  constexpr int kWReg = 3;
  double wv[kWReg];
#pragma unroll
  for (int u = 0; u < kWReg; ++u) {
    const int x = tid + u * kWinThreads, col = wbase + x;
    wv[u] = (x < nw && col >= 0 && col < p.S) ? __ldcg(Wrow + col) : -INFINITY;
  }
  // key slopes: the run payoffs lambda p - g are affine in the offset o (g fitted by gc0 + gc1 o on the
  // charge run, gd0 + gd1 |o| on the discharge run; g = 0 for the linear payoff), so
  //   cand(i, j) ~= key(j) + beta i - g0,  key(j) = W[j] - beta j,
  //   beta_c = lambda delta / eta_c + gc1,  beta_d = lambda delta eta_d - gd1   (any few-ulp rounding: see eps)
  const double beta_c = __dadd_rn(__dmul_rn(lam, p.dc), gc1);
  const double beta_d = __dsub_rn(__dmul_rn(lam, p.dd), gd1);
  const int nsg = p.nsingle < kMaxSingles ? p.nsingle : kMaxSingles;
  if (tid < nsg) {
    const WinSingle& g = p.sg[tid];
    SingleAct s;
    s.a = g.a; s.off = g.off; s.w = g.w; s.omw = g.omw;
    s.pay = __dmul_rn(lam, g.act);
    if (p.g_kind) s.pay = __dsub_rn(s.pay, __ldg(p.g + g.a));
    ss[tid] = s;
  }
  // max |W| over the tile: the high words of |W| (ordered like the values), reduced with REDUX; the
  // bound M below fills the low word with ones, so M >= max |W|
  unsigned mx = 0u;
#pragma unroll
  for (int u = 0; u < kWReg; ++u) {
    const int x = tid + u * kWinThreads;
    if (x < nw) {
      const double v = wv[u];
      if (v != -INFINITY) mx = umax(mx, (unsigned)__double2hiint(v) & 0x7fffffffu);
      wt[x] = v;
    }
  }
  for (int x = tid + kWReg * kWinThreads; x < nw; x += kWinThreads) {   // wide action spans
    const int col = wbase + x;
    double v = -INFINITY;
    if (col >= 0 && col < p.S) {
      v = __ldcg(Wrow + col);
      mx = umax(mx, (unsigned)__double2hiint(v) & 0x7fffffffu);
    }
    wt[x] = v;
  }
  __syncthreads();
  wtrace(2);
  // level 0: packed key(j) = W[j] - beta*j, position x (pairs of entries, 16-byte stores); the pairs
  // (x, x+1) and (x+1, x+2) feed the unimodality test (key x+2 recomputed here: no extra barrier)
  unsigned upc = 0u, dnc = kNoFall, upd = 0u, dnd = kNoFall;
#pragma unroll
  for (int u = 0; u < kLevelSlots; ++u) {   // n <= 768 (as the level builds)
    const int x = 2 * (tid + u * kWinThreads);
    if (x >= tc.n) break;
    const int j = i0 + 1 + x;
    ulonglong2 r;
    r.x = pack_key(__dsub_rn(wt[j - wbase], __dmul_rn(beta_c, (double)j)), x);
    r.y = pack_key(__dsub_rn(wt[j + 1 - wbase], __dmul_rn(beta_c, (double)(j + 1))), x + 1);
    *reinterpret_cast<ulonglong2*>(tc.v + x) = r;    // entry n (x + 1 == n) is padding
    if (x + 1 < tc.n) uni_pair(r.x, r.y, x + 1, upc, dnc);
    if (x + 2 < tc.n)
      uni_pair(r.y, pack_key(__dsub_rn(wt[j + 2 - wbase], __dmul_rn(beta_c, (double)(j + 2))), x + 2), x + 2, upc, dnc);
  }
#pragma unroll
  for (int u = 0; u < kLevelSlots; ++u) {
    const int x = 2 * (tid + u * kWinThreads);
    if (x >= td.n) break;
    const int j = i0 - p.Ld + x;
    ulonglong2 r;
    r.x = pack_key(__dsub_rn(wt[j - wbase], __dmul_rn(beta_d, (double)j)), x);
    r.y = pack_key(__dsub_rn(wt[j + 1 - wbase], __dmul_rn(beta_d, (double)(j + 1))), x + 1);
    *reinterpret_cast<ulonglong2*>(td.v + x) = r;
    if (x + 1 < td.n) uni_pair(r.x, r.y, x + 1, upd, dnd);
    if (x + 2 < td.n)
      uni_pair(r.y, pack_key(__dsub_rn(wt[j + 2 - wbase], __dmul_rn(beta_d, (double)(j + 2))), x + 2), x + 2, upd, dnd);
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  upc = __reduce_max_sync(0xffffffffu, upc);
  dnc = __reduce_min_sync(0xffffffffu, dnc);
  upd = __reduce_max_sync(0xffffffffu, upd);
  dnd = __reduce_min_sync(0xffffffffu, dnd);
  if ((tid & 31) == 0) {
    red[tid >> 5] = mx;
    ured[0][tid >> 5] = upc; ured[1][tid >> 5] = dnc; ured[2][tid >> 5] = upd; ured[3][tid >> 5] = dnd;
  }
  __syncthreads();
  upc = __reduce_max_sync(0xffffffffu, ured[0][tid % (kWinThreads / 32)]);
  dnc = __reduce_min_sync(0xffffffffu, ured[1][tid % (kWinThreads / 32)]);
  upd = __reduce_max_sync(0xffffffffu, ured[2][tid % (kWinThreads / 32)]);
  dnd = __reduce_min_sync(0xffffffffu, ured[3][tid % (kWinThreads / 32)]);
  const bool uni_c = upc < dnc, uni_d = upd < dnd;   // block-uniform
  const int pc = uni_c ? 0 : p.pc, pd = uni_d ? 0 : p.pd;
  if (tid == 0 && !(uni_c && uni_d)) atomicAdd(&g_window_level_tables, (unsigned long long)(!uni_c + !uni_d));
  wtrace(3);
  const int top = pc > pd ? pc : pd;      // unimodal tables need no levels
#pragma unroll
  for (int q = 1; q <= 9; q += 2) {     // levels <= 9 (L <= 512), two per barrier: unrolled, uniform exits
    if (q > top) break;
    if (q + 1 <= pc) build_level2(tc, q, tid);
    else if (q <= pc) build_level(tc, q, tid);
    if (q + 1 <= pd) build_level2(td, q, tid);
    else if (q <= pd) build_level(td, q, tid);
    __syncthreads();
  }
  wtrace(4);
  (void)ldl;
  const unsigned mb = __reduce_max_sync(0xffffffffu, red[tid % (kWinThreads / 32)]);
  const double M = __hiloint2double((int)mb, (int)0xffffffffu);
  const double bmax = fmax(fabs(beta_c), fabs(beta_d)) * p.jspan;   // >= |beta j| over the tile
  // 32u covers the rounding of key / beta*i / the canonical candidate; 2^-41 covers
  // the <1024-ulp truncation of the packed keys (|key| <= M + bmax); gfit[4] is the largest deviation
  // of g from its affine fit, gfit[5] bounds |g| (both 0 for the linear payoff)
  const double eps = 32.0 * 0x1p-53 * (M + bmax + fabs(lam) * p.pbar + p.gfit[5]) + 0x1p-41 * (M + bmax) + p.gfit[4];

  const int i = i0 + tid;
  const bool valid = i < p.S;
  const int lane = tid & 31;
  double best = -INFINITY;
  int arg = -1;
  bool near_tie = false;
  if (valid) {
    // charge window j in [i+1, i+Lc] = table [x, x+Lc-1]; discharge j in [i-Ld, i-1] = table [x, x+Ld-1]
    const int x = i - i0;
    double mc1, mc2, md1, md2;
    int xc, xd;
    if (uni_c) window_top2_uni(tc, (int)upc, x, x + p.Lc - 1, mc1, xc, mc2);
    else window_top2(tc, x, x + p.Lc - 1, mc1, xc, mc2);
    if (uni_d) window_top2_uni(td, (int)upd, x, x + p.Ld - 1, md1, xd, md2);
    else window_top2(td, x, x + p.Ld - 1, md1, xd, md2);
    const double bci = __dsub_rn(__dmul_rn(beta_c, (double)i), gc0), bdi = __dsub_rn(__dmul_rn(beta_d, (double)i), gd0);
    // candidates on a common scale y = key + beta*i; the action of column j is a_z - (j - i)
    double b1 = __dadd_rn(mc1, bci), b2 = __dadd_rn(mc2, bci);
    int a1 = p.a_z - ((i0 + 1 + xc) - i);
    {
      const double y1 = __dadd_rn(md1, bdi), y2 = __dadd_rn(md2, bdi);
      if (y1 > b1) { b2 = fmax(b1, y2); b1 = y1; a1 = p.a_z - ((i0 - p.Ld + xd) - i); }
      else b2 = fmax(b2, y1);
    }
    // singles, branch-free: b2 takes the smaller of (b1, c), b1 the larger; once a single leads, b1 is its
    // exact canonical value (a later single replaces it only by a larger canonical value)
    bool single_best = false;
    auto single_step = [&](const SingleAct& sa) {
      const double c = canon_staged(sa, wt, wbase, i);
      const bool gt = c > b1;
      b2 = fmax(b2, gt ? b1 : c);
      b1 = gt ? c : b1;
      a1 = gt ? sa.a : a1;
      single_best |= gt;
    };
    if (p.nsingle == 3) {                   // the Eq. 10 grid: zero action and the two endpoints
#pragma unroll
      for (int s = 0; s < 3; ++s) single_step(ss[s]);
    } else {
#pragma unroll 4
      for (int s = 0; s < nsg; ++s) single_step(ss[s]);
    }
    for (int s = nsg; s < p.nsingle; ++s) {
      const int a = __ldg(p.singles + s);
      const double c = canon_single(p, wt, wbase, i, a, lam);
      const bool gt = c > b1;
      b2 = fmax(b2, gt ? b1 : c);
      b1 = gt ? c : b1;
      a1 = gt ? a : a1;
      single_best |= gt;
    }
    if (__dsub_rn(b1, b2) > 2.0 * eps) {
      arg = a1;
      // canonical value of the unique argmax; a run action lies on the lattice (offset a_z - a1, w = 0), so
      // only its power (and g) is loaded: fl(fl(fl(lambda p) - g) + W[i + o])
      if (single_best) {
        best = b1;
      } else {
        double pay = __dmul_rn(lam, __ldg(p.act + a1));
        if (p.g_kind) pay = __dsub_rn(pay, __ldg(p.g + a1));
        best = __dadd_rn(pay, wt[i + (p.a_z - a1) - wbase]);
      }
    } else {
      near_tie = true;
    }
  }
  wtrace(5);
  // near ties (rare; every row for degenerate data such as zero prices): the whole warp re-scans the
  // row canonically, 32 actions at a time, and reduces (value desc, index asc) -- the smallest index
  // among exact ties, as in the oracle's ascending scan with a strict '>'.
  unsigned need = __ballot_sync(0xffffffffu, near_tie);
  while (need) {
    const int src = __ffs(need) - 1;
    need &= need - 1;
    const int ii = __shfl_sync(0xffffffffu, i, src);
    double v = -INFINITY;
    int va = 0x7fffffff;
    for (int s = lane; s < p.nlive; s += 32) {
      const int a = __ldg(p.live + s);
      const double c = canon_single(p, wt, wbase, ii, a, lam);
      if (c > v) { v = c; va = a; }          // ascending a within the lane
    }
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, sh);
      const int oa = __shfl_xor_sync(0xffffffffu, va, sh);
      if (ov > v || (ov == v && oa < va)) { v = ov; va = oa; }
    }
    if (lane == src) { best = v; arg = va; atomicAdd(&g_window_fallbacks, 1ull); }
  }
  if (!valid) { wtrace(6); return; }
  st.V[(size_t)k * p.ld + i] = best;
  st.pol[(size_t)k * p.S + i] = (int16_t)arg;
  wtrace(6);
}

template <bool kWait = false>
__device__ __forceinline__ void window_item(const WinParams& p, int k, int i0, double* wsm) {
  const WinStage st{p.W, p.V, p.pol, p.lambda_t};
  window_item<kWait>(p, st, k, i0, wsm);
}

__global__ void __launch_bounds__(kWinThreads, ESDP_WIN_MINB) window_stencil_kernel(WinParams p) {
  extern __shared__ __align__(16) double wsm[];
  window_item<true>(p, blockIdx.y, blockIdx.x * kWinTile, wsm);   // waits for W_t (the contraction) inside
  pdl_trigger_late();
}

}  // namespace esdp
