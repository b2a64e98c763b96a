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

__device__ __forceinline__ void wtrace(int m) { ktrace(0, m); }

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
  int force_nonuni;         // tests: treat every run table as non-unimodal (exercises the fallback paths)
  int eq10;                 // singles are exactly {charge endpoint (interpolated), zero action, discharge endpoint
                            // (interpolated)} in this order: the Eq. 10 grid with eta < 1 (branch-free queries)
  int force_generic;        // tests: take the generic query path even where the Eq. 10 one applies
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

__host__ __device__ constexpr int win_al2(int n) { return (n + 1) & ~1; }
// shared memory of one (k, tile) item, tile = kWinThreads * opt output columns: W tile [nw], raw key tables
// [nc], [nd], row payoffs [A], then (levels only) the packed sparse tables of the non-unimodal fallback
inline size_t window_smem_bytes(int Lc, int Ld, int o_span, int A, int opt = 1, bool levels = true) {
  const int tile = kWinThreads * opt;
  const size_t nw = win_al2(tile + o_span + 2), nc = win_al2(tile + Lc), nd = win_al2(tile + Ld);
  return sizeof(double) * (nw + nc + nd + win_al2(A)) +
         (levels ? sizeof(unsigned long long) * (window_levels(Lc) * nc + window_levels(Ld) * nd) : 0) + 64;
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

constexpr unsigned kNoFall = 0xffffu;   // "no fall" sentinel of the unimodality test

// max of two doubles that are never NaN (W is finite or -inf): one compare and a select, no NaN fix-up
__device__ __forceinline__ double dmx(double a, double b) { return a > b ? a : b; }

// Query of one output column on the fast path: both run tables unimodal (block-uniform) and the Eq. 10
// singles.  The window maximum of a unimodal table with peak p* sits at q = clamp(p*, l, r) and the
// runner-up next to it; the two runs, then the three singles (canonical candidates, R14) go through one
// top-2 with the action of the leader.  Returns false on a near tie (the caller rescans the row).
struct WinFastRow {        // per-thread row constants of the fast path (the rest is read from p: constant bank or,
                           // in the batch kernel, broadcast shared-memory loads)
  double beta_c, beta_d, gc0, gd0, pay_z;
  int pcs, pds;            // peaks of the charge / discharge tables
};
__device__ __forceinline__ bool window_query_fast(const WinParams& p, const WinFastRow& f, const double* __restrict__ kc,
                                                  const double* __restrict__ kd, const double* __restrict__ wt,
                                                  const double* __restrict__ pay, int wbase, int i, int x, double eps2,
                                                  double& best, int& arg) {
  const int Lc = p.Lc, Ld = p.Ld, a_z = p.a_z;
  const int rc = x + Lc - 1, rd = x + Ld - 1;
  const int qc = min(max(f.pcs, x), rc), qd = min(max(f.pds, x), rd);
  ESDP_ASSERT(Lc >= 2 && Ld >= 2 && qc >= x && qc <= rc && qd >= x && qd <= rd);
  const double kc1 = kc[qc], kd1 = kd[qd];
  // the runner-up of a unimodal window is a neighbour of q inside it (windows hold >= 2 entries: Lc, Ld >= 2)
  const double kcl = kc[qc == x ? qc + 1 : qc - 1], kcr = kc[qc == rc ? qc - 1 : qc + 1];
  const double kdl = kd[qd == x ? qd + 1 : qd - 1], kdr = kd[qd == rd ? qd - 1 : qd + 1];
  const double di = (double)i;
  const double bci = __dsub_rn(__dmul_rn(f.beta_c, di), f.gc0), bdi = __dsub_rn(__dmul_rn(f.beta_d, di), f.gd0);
  // the runs on the common scale y = key + beta i; the action of table position q is a_z - (j - i)
  const double yc1 = __dadd_rn(kc1, bci), yc2 = __dadd_rn(dmx(kcl, kcr), bci);
  const double yd1 = __dadd_rn(kd1, bdi), yd2 = __dadd_rn(dmx(kdl, kdr), bdi);
  // the singles, canonical
  const double* wi = wt + (i - wbase);
  const WinSingle &sc = p.sg[0], &sd = p.sg[2];
  ESDP_ASSERT(i - wbase + sc.off >= 0 && i - wbase + sd.off + 1 < kWinThreads * 4 + (p.o_max - p.o_min) + 2);
  const double ce = __dadd_rn(pay[sc.a], __dadd_rn(__dmul_rn(sc.omw, wi[sc.off]), __dmul_rn(sc.w, wi[sc.off + 1])));
  const double cz = __dadd_rn(f.pay_z, wi[0]);
  const double cd = __dadd_rn(pay[sd.a], __dadd_rn(__dmul_rn(sd.omw, wi[sd.off]), __dmul_rn(sd.w, wi[sd.off + 1])));
  // leader; once a single leads, b1 is its exact canonical value
  double b1 = yc1;
  int a1 = a_z - 1 - qc + x;
  bool sb = false;
  if (yd1 > b1) { b1 = yd1; a1 = a_z + Ld - qd + x; }
  if (ce > b1) { b1 = ce; a1 = sc.a; sb = true; }
  if (cz > b1) { b1 = cz; a1 = a_z; sb = true; }
  if (cd > b1) { b1 = cd; a1 = sd.a; sb = true; }
  // unique leader: every other candidate (the runs' runner-ups included) at most b1 - 2.25 eps, i.e. more than
  // 2 eps below it after the subtraction's rounding (u |b1| < eps / 4)
  const double thr = __dsub_rn(b1, 1.125 * eps2);
  const int above = (yc1 > thr) + (yd1 > thr) + (ce > thr) + (cz > thr) + (cd > thr) + (yc2 > thr) + (yd2 > thr);
  if (above != 1) return false;
  arg = a1;
  // canonical value of the unique argmax; a run action lies on the lattice (offset a_z - a1, weight 0)
  ESDP_ASSERT(a1 >= 0 && a1 < p.A && (sb || (a_z - a1 >= -Ld && a_z - a1 <= Lc)));
  best = sb ? b1 : __dadd_rn(pay[a1], wi[a_z - a1]);
  return true;
}

// One (k, 256-column tile) item of the window stencil, executed by a 256-thread block.
//   1. Row payoffs pay[a] = fl(fl(lambda_{t,k} p_a) - g_a) (R14) for every action, in shared memory: inputs
//      only, so they are formed before the programmatic dependency wait (kWait) on W_t.
//   2. W_t over the tile and its action halo, -inf outside [0, S-1] (Alg. 1 line 8: an infeasible action
//      never wins), and the high word of max |W| for the exactness margin.
//   3. The two run key tables key(j) = fl(W[j] - fl(beta j)) as plain doubles.  Every thread also records
//      the rises (key[x] > key[x-1]; the left key recomputed from W, the same bits) and falls of its
//      entries; one block reduction makes "every rise precedes every fall" (unimodal) block-uniform.  A
//      unimodal table answers any window from its peak p* = the last rise: the maximum sits at
//      clamp(p*, l, r), the runner-up next to it.  Only a non-unimodal table builds the packed sparse
//      tables (positions in the low bits, two lookups per window; their truncation widens eps).
//   4. One output per thread: the window top-2 of each run, the singles (zero action, interpolated
//      endpoints, irregular actions) canonically, the margin test; near ties rescan the row canonically.
struct WinStage {          // the per-stage pointers of an item (the rest of WinParams is stage-invariant)
  const double* W; double* V; int16_t* pol; const double* lambda_t;
};

// canonical candidate of action a from the staged row payoff: fl(pay_a + Wint), -inf if infeasible
__device__ __forceinline__ double canon_pay(const WinParams& p, const double* __restrict__ pay,
                                            const double* __restrict__ wt, int wbase, int i, int a) {
  const int o = __ldg(p.off + a);
  const double wa = __ldg(p.w + a);
  const int x = i + o - wbase;
  const double wint = (wa == 0.0) ? wt[x] : __dadd_rn(__dmul_rn(__ldg(p.omw + a), wt[x]), __dmul_rn(wa, wt[x + 1]));
  return __dadd_rn(pay[a], wint);
}

// Keys x and x + 1 of a raw key table (x even, 16-byte aligned pair store) with the rise / fall bookkeeping of
// entries x and x + 1: three W loads and three keys (key x - 1 recomputed, the same bits) per two entries.
__device__ __forceinline__ void win_key_pair(double* __restrict__ tb, const double* __restrict__ wt, int wbase, int j0,
                                             int x, int n, double beta, unsigned& up, unsigned& dn) {
  const int j = j0 + x;
  ESDP_ASSERT((x & 1) == 0 && x < n && j - wbase >= (x >= 1 ? 1 : 0));
  const double* w = wt + (j - wbase);
  const double jd = (double)j;
  const double k0 = __dsub_rn(w[0], __dmul_rn(beta, jd));
  const bool two = x + 1 < n;
  const double k1 = two ? __dsub_rn(w[1], __dmul_rn(beta, __dadd_rn(jd, 1.0))) : 0.0;
  if (x >= 1) {
    const double km = __dsub_rn(w[-1], __dmul_rn(beta, __dsub_rn(jd, 1.0)));
    if (k0 > km) up = umax(up, (unsigned)x);
    if (k0 < km) dn = umin(dn, (unsigned)x);
  }
  if (two) {
    if (k1 > k0) up = umax(up, (unsigned)(x + 1));
    if (k1 < k0) dn = umin(dn, (unsigned)(x + 1));
    *reinterpret_cast<double2*>(tb + x) = make_double2(k0, k1);
  } else {
    tb[x] = k0;
  }
}

// top-2 of the window [l, r] of a raw unimodal table with peak pstar
__device__ __forceinline__ void win_top2_uni(const double* __restrict__ tb, int pstar, int l, int r, double& m1, int& pos,
                                             double& m2) {
  const int q = min(max(pstar, l), r);
  pos = q;
  m1 = tb[q];
  m2 = fmax(q > l ? tb[q - 1] : -INFINITY, q < r ? tb[q + 1] : -INFINITY);
}

// raw-key window top-2 by a scan (a non-unimodal table without packed levels; ascending, ties keep the
// first -- an equal runner-up then fails the margin test and the row is rescanned canonically)
__device__ __forceinline__ void win_top2_scan(const double* __restrict__ tb, int l, int r, double& m1, int& pos,
                                              double& m2) {
  m1 = -INFINITY; m2 = -INFINITY; pos = l;
  for (int q = l; q <= r; ++q) {
    const double v = tb[q];
    if (v > m1) { m2 = m1; m1 = v; pos = q; }
    else m2 = fmax(m2, v);
  }
}

// OPT: outputs per thread (tile = kWinThreads * OPT columns; 2 amortizes the halo and the per-block work in
// the throughput regime).  kLevels: non-unimodal tables build packed sparse tables (else: a per-window scan
// of the raw keys; for payoffs whose tables are unimodal in practice -- the linear payoff).
template <bool kWait = false, int OPT = 1, bool kLevels = true>
__device__ __forceinline__ void window_item(const WinParams& p, const WinStage& st, int k, int i0, double* wsm) {
  static_assert(!kLevels || OPT == 1, "the level builds assume one output per thread");
  constexpr int kTile = kWinThreads * OPT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  wtrace(0);
  const int span = p.o_max - p.o_min;
  const int nw = kTile + span + 2;
  const int nc = kTile + p.Lc, nd = kTile + p.Ld;   // charge: columns [i0+1, i0+nc]; discharge [i0-Ld, ..)
  double* wt = wsm;                                        // W over columns [wbase, wbase + nw)
  double* kc = wt + win_al2(nw);
  double* kd = kc + win_al2(nc);
  double* pay = kd + win_al2(nd);
  __shared__ unsigned red[5][kWinThreads / 32];            // per warp: max|W| hi word, up_c, dn_c, up_d, dn_d
  const double* Wrow = st.W + (p.rank1 ? 0 : (size_t)k * p.ld);
  const int wbase = i0 + p.o_min;
  // 1. inputs: the row payoffs (and lambda, the g fit) before the dependency wait
  const double lam = st.lambda_t[k];
  const double gc0 = p.gfit[0], gc1 = p.gfit[1], gd0 = p.gfit[2], gd1 = p.gfit[3];
  for (int a = tid; a < p.A; a += kWinThreads) {
    double v = __dmul_rn(lam, __ldg(p.act + a));
    if (p.g_kind) v = __dsub_rn(v, __ldg(p.g + a));
    pay[a] = v;
  }
  if (kWait) pdl_wait();
  wtrace(1);
  // 2. W_t over the tile: all of this thread's loads are issued before anything waits on them
  constexpr int kWReg = 2 + OPT;
  double wv[kWReg];
  const double* wsrc = Wrow + (wbase + tid);   // dereferenced only inside [0, S)
#pragma unroll
  for (int u = 0; u < kWReg; ++u) {
    const int x = tid + u * kWinThreads;
    wv[u] = (x < nw && (unsigned)(wbase + x) < (unsigned)p.S) ? __ldcg(wsrc + u * kWinThreads) : -INFINITY;
  }
  unsigned mx = 0u;
#pragma unroll
  for (int u = 0; u < kWReg; ++u) {
    const int x = tid + u * kWinThreads;
    if (x < nw) {
      if (wv[u] != -INFINITY) mx = umax(mx, (unsigned)__double2hiint(wv[u]) & 0x7fffffffu);
      wt[x] = wv[u];
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
  const double beta_c = __dadd_rn(__dmul_rn(lam, p.dc), gc1);   // key slopes (see the header comment)
  const double beta_d = __dsub_rn(__dmul_rn(lam, p.dd), gd1);
  __syncthreads();
  wtrace(2);
  // 3. raw key tables with the unimodality bookkeeping
  unsigned upc = 0u, dnc = kNoFall, upd = 0u, dnd = kNoFall;
  for (int x = 2 * tid; x < nc || x < nd; x += 2 * kWinThreads) {
    if (x < nc) win_key_pair(kc, wt, wbase, i0 + 1, x, nc, beta_c, upc, dnc);
    if (x < nd) win_key_pair(kd, wt, wbase, i0 - p.Ld, x, nd, beta_d, upd, dnd);
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  upc = __reduce_max_sync(0xffffffffu, upc);
  dnc = __reduce_min_sync(0xffffffffu, dnc);
  upd = __reduce_max_sync(0xffffffffu, upd);
  dnd = __reduce_min_sync(0xffffffffu, dnd);
  if (lane == 0) { red[0][warp] = mx; red[1][warp] = upc; red[2][warp] = dnc; red[3][warp] = upd; red[4][warp] = dnd; }
  __syncthreads();
  mx = __reduce_max_sync(0xffffffffu, red[0][lane % (kWinThreads / 32)]);
  upc = __reduce_max_sync(0xffffffffu, red[1][lane % (kWinThreads / 32)]);
  dnc = __reduce_min_sync(0xffffffffu, red[2][lane % (kWinThreads / 32)]);
  upd = __reduce_max_sync(0xffffffffu, red[3][lane % (kWinThreads / 32)]);
  dnd = __reduce_min_sync(0xffffffffu, red[4][lane % (kWinThreads / 32)]);
  const bool uni_c = upc < dnc && !p.force_nonuni, uni_d = upd < dnd && !p.force_nonuni;   // block-uniform
  wtrace(3);
  // non-unimodal tables (rare for linear payoffs; cfg3's fixed cost): packed sparse tables
  RangeMax tc, td;
  tc.n = nc; td.n = nd;
  tc.ns = win_al2(nc); td.ns = win_al2(nd);
  tc.v = reinterpret_cast<unsigned long long*>(pay + win_al2(p.A));
  td.v = tc.v + (size_t)(p.pc + 1) * tc.ns;
  if (!(uni_c && uni_d)) {
    if (tid == 0) atomicAdd(&g_window_level_tables, (unsigned long long)(!uni_c + !uni_d));
    if (kLevels) {
      for (int x = tid; x < nc || x < nd; x += kWinThreads) {
        if (!uni_c && x < nc) tc.v[x] = pack_key(kc[x], x);
        if (!uni_d && x < nd) td.v[x] = pack_key(kd[x], x);
      }
      __syncthreads();
      const int pc = uni_c ? 0 : p.pc, pd = uni_d ? 0 : p.pd;
      const int top = pc > pd ? pc : pd;
#pragma unroll
      for (int q = 1; q <= 9; q += 2) {     // levels <= 9 (L <= 512), two per barrier: unrolled, uniform exits
        if (q > top) break;
        if (q + 1 <= pc) build_level2(tc, q, tid);
        else if (q <= pc) build_level(tc, q, tid);
        if (q + 1 <= pd) build_level2(td, q, tid);
        else if (q <= pd) build_level(td, q, tid);
        __syncthreads();
      }
    }
  }
  wtrace(4);
  const double M = __hiloint2double((int)mx, (int)0xffffffffu);     // >= max |W| over the tile
  const double bmax = fmax(fabs(beta_c), fabs(beta_d)) * p.jspan;   // >= |beta j| over the tile
  // 32u: rounding of key / beta i / the canonical candidate; 2^-41: the <1024-ulp
  // truncation of packed keys, only where a packed table answers; gfit[4] / gfit[5]: the g fit's deviation
  // and max |g| (both 0 for the linear payoff)
  const double eps = 32.0 * 0x1p-53 * (M + bmax + fabs(lam) * p.pbar + p.gfit[5]) +
                     ((!kLevels || (uni_c && uni_d)) ? 0.0 : 0x1p-41 * (M + bmax)) + p.gfit[4];
  // 4. OPT outputs per thread (columns i0 + tid + u * kWinThreads)
  const bool fast = uni_c && uni_d && p.eq10 && !p.force_generic;   // block-uniform
  double* const vrow = st.V + (size_t)k * p.ld;
  short* const prow = reinterpret_cast<short*>(st.pol + (size_t)k * p.S);
  WinFastRow fr;
  if (fast) {
    fr.beta_c = beta_c; fr.beta_d = beta_d; fr.gc0 = gc0; fr.gd0 = gd0; fr.pay_z = pay[p.a_z];
    fr.pcs = (int)upc; fr.pds = (int)upd;
  }
  const double eps2 = 2.0 * eps;
  double bestv[OPT];
  int argv[OPT];
  unsigned ties = 0u;   // bit u: output u is a near tie
#pragma unroll
  for (int u = 0; u < OPT; ++u) {
  const int i = i0 + tid + u * kWinThreads;
  const bool valid = i < p.S;
  double best = -INFINITY;
  int arg = -1;
  bool near_tie = false;
  if (valid && fast) {
    near_tie = !window_query_fast(p, fr, kc, kd, wt, pay, wbase, i, i - i0, eps2, best, arg);
  } else if (valid) {
    const int x = i - i0;   // charge window: table [x, x+Lc-1]; discharge: [x, x+Ld-1]
    double mc1, mc2, md1, md2;
    int xc, xd;
    if (uni_c) win_top2_uni(kc, (int)upc, x, x + p.Lc - 1, mc1, xc, mc2);
    else if (kLevels) window_top2(tc, x, x + p.Lc - 1, mc1, xc, mc2);
    else win_top2_scan(kc, x, x + p.Lc - 1, mc1, xc, mc2);
    if (uni_d) win_top2_uni(kd, (int)upd, x, x + p.Ld - 1, md1, xd, md2);
    else if (kLevels) window_top2(td, x, x + p.Ld - 1, md1, xd, md2);
    else win_top2_scan(kd, x, x + p.Ld - 1, md1, xd, md2);
    const double di = (double)i;
    const double bci = __dsub_rn(__dmul_rn(beta_c, di), gc0), bdi = __dsub_rn(__dmul_rn(beta_d, di), gd0);
    // candidates on a common scale y = key + beta i; the action of column j is a_z - (j - i)
    double b1 = __dadd_rn(mc1, bci), b2 = __dadd_rn(mc2, bci);
    int a1 = p.a_z - 1 - xc + x;                       // j = i0 + 1 + xc
    {
      const double y1 = __dadd_rn(md1, bdi), y2 = __dadd_rn(md2, bdi);
      if (y1 > b1) { b2 = fmax(b1, y2); b1 = y1; a1 = p.a_z + p.Ld - xd + x; }   // j = i0 - Ld + xd
      else b2 = fmax(b2, y1);
    }
    // singles, branch-free: b2 takes the smaller of (b1, c), b1 the larger; once a single leads, b1 is its
    // exact canonical value (a later single replaces it only by a larger canonical value)
    bool single_best = false;
    auto single_step = [&](const WinSingle& sg) {
      const int xx = i + sg.off - wbase;
      const double wint = (sg.w == 0.0) ? wt[xx] : __dadd_rn(__dmul_rn(sg.omw, wt[xx]), __dmul_rn(sg.w, wt[xx + 1]));
      const double c = __dadd_rn(pay[sg.a], wint);
      const bool gt = c > b1;
      b2 = fmax(b2, gt ? b1 : c);
      b1 = gt ? c : b1;
      a1 = gt ? sg.a : a1;
      single_best |= gt;
    };
    const int nsg = p.nsingle < kMaxSingles ? p.nsingle : kMaxSingles;
    if (p.nsingle == 3) {                   // the Eq. 10 grid: zero action and the two endpoints
#pragma unroll
      for (int s = 0; s < 3; ++s) single_step(p.sg[s]);
    } else {
      for (int s = 0; s < nsg; ++s) single_step(p.sg[s]);
    }
    for (int s = nsg; s < p.nsingle; ++s) {
      const int a = __ldg(p.singles + s);
      const double c = canon_pay(p, pay, wt, wbase, i, a);
      const bool gt = c > b1;
      b2 = fmax(b2, gt ? b1 : c);
      b1 = gt ? c : b1;
      a1 = gt ? a : a1;
      single_best |= gt;
    }
    if (__dsub_rn(b1, b2) > 2.0 * eps) {
      arg = a1;
      // canonical value of the unique argmax; a run action lies on the lattice (offset a_z - a1, weight 0)
      best = single_best ? b1 : __dadd_rn(pay[a1], wt[i + (p.a_z - a1) - wbase]);
    } else {
      near_tie = true;
    }
  }
  bestv[u] = best;
  argv[u] = arg;
  ties |= near_tie ? 1u << u : 0u;
  }
  wtrace(5);
  // near ties (rare; every row for degenerate data such as zero prices): the whole warp re-scans the
  // row canonically, 32 actions at a time, and reduces (value desc, index asc) -- the smallest index
  // among exact ties, as in the oracle's ascending scan with a strict '>'.
  if (__any_sync(0xffffffffu, ties != 0u)) {
#pragma unroll
    for (int u = 0; u < OPT; ++u) {
      unsigned need = __ballot_sync(0xffffffffu, (ties >> u) & 1u);
      while (need) {
        const int src = __ffs(need) - 1;
        need &= need - 1;
        const int ii = i0 + src + (warp << 5) + u * kWinThreads;
        double v = -INFINITY;
        int va = 0x7fffffff;
        for (int s = lane; s < p.nlive; s += 32) {
          const int a = __ldg(p.live + s);
          const double c = canon_pay(p, pay, wt, wbase, ii, a);
          if (c > v) { v = c; va = a; }          // ascending a within the lane
        }
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, v, sh);
          const int oa = __shfl_xor_sync(0xffffffffu, va, sh);
          if (ov > v || (ov == v && oa < va)) { v = ov; va = oa; }
        }
        if (lane == src) { bestv[u] = v; argv[u] = va; atomicAdd(&g_window_fallbacks, 1ull); }
      }
    }
  }
  // stores off one base pointer per row (immediate offsets); st.global: the compiler then knows they do not
  // alias the shared-memory tables
  double* const vp = vrow + i0 + tid;
  short* const pp = prow + i0 + tid;
  const int nvalid = p.S - i0 - tid;   // outputs u < ceil(nvalid / kWinThreads) are inside the row
#pragma unroll
  for (int u = 0; u < OPT; ++u) {
    if (u * kWinThreads < nvalid) {
      __stwb(vp + u * kWinThreads, bestv[u]);
      __stwb(pp + u * kWinThreads, (short)argv[u]);
    }
  }
  wtrace(6);
}

template <bool kWait = false, int OPT = 1, bool kLevels = true>
__device__ __forceinline__ void window_item(const WinParams& p, int k, int i0, double* wsm) {
  const WinStage st{p.W, p.V, p.pol, p.lambda_t};
  window_item<kWait, OPT, kLevels>(p, st, k, i0, wsm);
}

template <int OPT, bool kLevels>
__global__ void __launch_bounds__(kWinThreads, ESDP_WIN_MINB) window_stencil_kernel(WinParams p) {
  extern __shared__ __align__(16) double wsm[];
  window_item<true, OPT, kLevels>(p, blockIdx.y, blockIdx.x * (kWinThreads * OPT), wsm);   // waits for W_t inside
  pdl_trigger_late();
}

}  // namespace esdp
