// esdp.cu -- host side of libesdp.so: the C ABI of include/esdp.h.
//
// Validation, the state/action grid (Eq. 10) and the per-action transition data
// (Alg. 1 lines 2-5) are computed here on the host once per context, in binary64 with
// FMA contraction disabled (-Xcompiler -ffp-contract=off).  Everything per stage runs in the
// kernels of kernels.cuh; the whole backward pass is one CUDA graph (2T+1 launches).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <unordered_map>
#include <string>
#include <thread>
#include <vector>

#include "../../include/esdp.h"
#include "kernels.cuh"
#include "window.cuh"
#include "batch.cuh"
#include "simmodes.cuh"
#include "ozaki.cuh"

using namespace esdp;

namespace {

constexpr double kGridTol = 1e-9;  // DESIGN R6/R7
thread_local std::string g_create_error;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

}  // namespace

// One set of device inputs (double-buffered: a load fills the slot the running backward does not read).
struct InputSlot {
  double *lambda = nullptr, *P = nullptr, *pi = nullptr, *cdf = nullptr, *cdf1 = nullptr, *g = nullptr, *gfit = nullptr;
  uint64_t *guide = nullptr, *guide1 = nullptr;
  int *tab = nullptr, *src = nullptr;   // Markov: sampling table of each stage, representative stage of each table
  int nuniq = 0, gbits = 0;             // distinct P_t slices (tables) and guide bits of this slot's tables
  cudaEvent_t ev_head = nullptr, ev_tables = nullptr, use_ev = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  bool use_pending = false;
  bool tables_stale = false;   // P uploaded, its sampling tables (cdf / guide) not built yet
  bool pi_stale = false;       // pi uploaded, its sampling tables (cdf1 / guide1; rank-1: cdf / guide) not built yet
  // pinned host staging of the small host-computed uploads (tab, src, gfit): a copy from pageable memory is
  // not a plain asynchronous DMA; stage_ev (recorded after those copies) guards the staging's reuse
  int* stage_h = nullptr;      // [2 (T-1)] tab, then src
  double* gfit_stage = nullptr;   // [6]
  cudaEvent_t stage_ev = nullptr;
  // generation of the data each array holds (esdp_ctx::gen at its upload): a kept (NULL) array is copied
  // from the newest slot only when the generations differ
  uint64_t gen_lambda = 0, gen_P = 0, gen_pi = 0, gen_g = 0;
  double gfit_h[6] = {0, 0, 0, 0, 0, 0};
};

struct esdp_ctx {
  // problem
  int T = 0, K = 0, S = 0, A = 0, kind = 0, rank1 = 0;
  uint64_t gen = 0;   // upload generations (InputSlot::gen_*)
  int ld = 0;  // padded row length of V and W on the device (multiple of 4 doubles: 16-byte cp.async)
  // multi-GPU (esdp_create_dist): this rank owns price-state rows [k_lo, k_lo + k_cnt); V_t and pol_t are
  // all-gathered every stage in blocks of kmax rows (Kp = world * kmax rows per stage on every rank)
  int world = 1, rank = 0, kmax = 0, k_lo = 0, k_cnt = 0, Kp = 0;
  ncclComm_t comm = nullptr;
  uint32_t flags = 0;
  double pbar = 0, sbar = 0, s0 = 0, eta_c = 1, eta_d = 1, delta = 1;
  std::vector<double> act, w, omw;
  std::vector<int> off;
  std::vector<Seg> segs;
  int o_min = 0, o_max = 0;
  // exact sliding-window stencil plan (window.cuh); use_window = 0 -> brute-force stencil_kernel
  int use_window = 0, a_z = -1, Lc = 0, Ld = 0, pc = 0, pd = 0;
  std::vector<int> singles, live_list;
  int* d_singles = nullptr;
  int* d_live = nullptr;
  size_t window_smem = 0;
  int win_opt = 1, win_levels = 1;   // window kernel variant: outputs per thread, packed level tables
  int on_grid = 1, f0 = 0;
  double w0 = 0.0;
  // device
  double *d_lambda = nullptr, *d_P = nullptr, *d_pi = nullptr, *d_g = nullptr;
  double *d_act = nullptr, *d_w = nullptr, *d_omw = nullptr;
  int* d_off = nullptr;
  Seg* d_segs = nullptr;
  double* d_gfit = nullptr;   // [6] affine fit of g on the window runs (window.cuh WinParams::gfit)
  double* d_F = nullptr;      // [A] SoC change of each action (Eq. 2): physical simulation mode
  std::vector<double> F;
  int16_t* d_stack = nullptr; // bid-clearing simulation: [paths][A] hull stacks
  int64_t stack_cap = 0;
  double gfit[6] = {0, 0, 0, 0, 0, 0};
  double *d_V = nullptr, *d_W = nullptr, *d_J = nullptr, *d_cdf = nullptr, *d_cdf1 = nullptr;
  uint64_t *d_guide = nullptr, *d_guide1 = nullptr;
  int g_max = 10, g_r1 = 10;  // guide bits: at most (pi_1 table; Markov tables when they fit), rank-1 rows
  size_t guide_cap = 0;       // guide entries allocated per slot
  double *d_red = nullptr;
  int16_t* d_pol = nullptr;
  double* d_sim = nullptr;
  int64_t sim_cap = 0;
  int32_t* d_req = nullptr;
  int64_t req_cap = 0;
  int32_t* d_nv = nullptr;
  int16_t* d_vert = nullptr;
  double *d_q = nullptr, *d_price = nullptr;
  int64_t out_cap = 0;
  cudaStream_t stream = nullptr;
  // input uploads (upload): on their own stream, in the order the backward consumes them -- lambda/pi/g
  // first (ev_head), then P in stage chunks T-1.. (chunk_ev[j] covers stages [chunk_lo[j], chunk_hi[j]]);
  // the backward graph waits on these events (external event-wait nodes), so a load overlaps the solve
  cudaStream_t copy = nullptr;
  // two input slots: `active` holds the inputs of the last launched backward (read by the simulation,
  // the bid curves ...), `pending` (or -1) the inputs of the latest load that no backward has used yet.
  // The fields d_lambda ... d_gfit, ev_head, chunk_ev, ev_tables alias the slot selected by select_slot.
  InputSlot slot[2];
  int active = 0, pending = -1;
  cudaGraphExec_t graphs[2] = {nullptr, nullptr};
  cudaEvent_t ev_head = nullptr, ev_tables = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  std::vector<int> chunk_lo, chunk_hi;
  cudaGraphExec_t graph = nullptr;
  size_t stencil_smem = 0;
  int64_t launches = 0;
  // bid-curve requests extracted inside the backward graph (esdp_set_bid_requests)
  int64_t fb_n = 0;
  int32_t fb_cap = 0;
  int32_t *d_fb_req = nullptr, *d_fb_slot = nullptr;
  std::vector<int64_t> fb_off;   // [T+2]: requests of stage t are [fb_off[t], fb_off[t+1])
  int32_t* fb_nvert = nullptr;
  int16_t* fb_vert = nullptr;
  double *fb_q = nullptr, *fb_price = nullptr;
  int fb_batch = 1;
  std::vector<cudaStream_t> side;      // side streams of the bid-curve branches (lowest priority)
  int prio_lo = 0;
  std::vector<cudaEvent_t> fb_ev, join_ev;
  std::vector<cudaEvent_t> ev;  // ESDP_PROFILE: [t][4] = contract begin/end, stencil begin/end
  int prof_stride = 1;
  bool pdl = true;
  int dmma2 = 0;   // shared-memory-staged DMMA expectation (set when its tile fits)
  int dmma_probe_failed = 0;   // the DMMA-vs-fma-chain probe found a mismatch: expectation on DFMA
  bool solved = false;
  std::string err;
};

namespace {

// Point the input aliases (d_lambda ... d_gfit, ev_head, chunk_ev, ev_tables) at slot sl.
void select_slot(esdp_ctx* c, int sl) {
  InputSlot& x = c->slot[sl];
  c->d_lambda = x.lambda; c->d_P = x.P; c->d_pi = x.pi; c->d_cdf = x.cdf; c->d_cdf1 = x.cdf1;
  c->d_guide = x.guide; c->d_guide1 = x.guide1; c->d_g = x.g; c->d_gfit = x.gfit;
  c->ev_head = x.ev_head; c->ev_tables = x.ev_tables; c->chunk_ev = x.chunk_ev;
}

esdp_status fail(esdp_ctx* c, esdp_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf; else g_create_error = buf;
  return s;
}

#define CUDA_OR_FAIL(ctx, call)                                                             \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail((ctx), e_ == cudaErrorMemoryAllocation ? ESDP_E_NOMEM : ESDP_E_CUDA,      \
                  "%s: %s", #call, cudaGetErrorString(e_));                                 \
  } while (0)

bool simplex_ok(const double* q, int K) {
  double s = 0.0;
  for (int j = 0; j < K; ++j) {
    if (!std::isfinite(q[j]) || q[j] < 0.0) return false;
    s += q[j];
  }
  return std::fabs(s - 1.0) <= 1e-9;
}

// Eq. 10 with the R6 guard and endpoint clamp.
void paper_grid(double pbar, double eta_c, double eta_d, double delta, std::vector<double>& out) {
  const double qc = pbar * eta_c / delta;
  const double qd = pbar / (delta * eta_d);
  long long nc = (long long)std::ceil(qc - kGridTol), nd = (long long)std::ceil(qd - kGridTol);
  if (nc < 1) nc = 1;
  if (nd < 1) nd = 1;
  out.clear();
  for (long long j = nc; j >= 1; --j) {
    const double x = (double)j * delta / eta_c;
    out.push_back(-(x < pbar ? x : pbar));
  }
  out.push_back(0.0);
  for (long long j = 1; j <= nd; ++j) {
    const double x = (double)j * delta * eta_d;
    out.push_back(x < pbar ? x : pbar);
  }
}

// A small persistent host thread pool for input validation (one per process, created on first use):
// run(n, f) calls f(0..n-1) on the pool and the calling thread and returns when all are done.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  int size() const { return (int)th_.size() + 1; }
  void run(int n, const std::function<void(int)>& f) {
    std::unique_lock<std::mutex> lk(run_m_);   // one job at a time
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = &f; n_ = n; next_ = 0; left_ = n; ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [&] { return left_ == 0; });
    job_ = nullptr;
  }

 private:
  HostPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    const char* e = getenv("ESDP_HOST_THREADS");   // measurement: threads of the host pool (caller included)
    const unsigned cap = (e && atoi(e) > 0) ? (unsigned)atoi(e) : 16u;
    const int nw = (int)std::max<unsigned>(1, std::min<unsigned>(cap - 1, hw > 1 ? hw - 1 : 1));
    for (int w = 0; w < nw; ++w) th_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    { std::lock_guard<std::mutex> g(m_); stop_ = true; }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void work() {   // take task indices until none is left
    for (;;) {
      int k;
      const std::function<void(int)>* f;
      {
        std::lock_guard<std::mutex> g(m_);
        if (!job_ || next_ >= n_) return;
        k = next_++;
        f = job_;
      }
      (*f)(k);
      std::lock_guard<std::mutex> g(m_);
      if (--left_ == 0) done_.notify_all();
    }
  }
  void loop() {
    long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_, run_m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0, next_ = 0, left_ = 0;
  long long gen_ = 0;
  bool stop_ = false;
};

// Guide geometry of the sampling tables (kernels.cuh cdf_kernel): 2^g buckets per row, g in [6, 14],
// at most the first power of two >= kGuideRatio K (at most 2^14); g_for: the most bits for `rows` rows within `cap` entries.
constexpr int kGuideMinG = 6;
constexpr int kGuideRatio = 64;   // cfg2 simulation 259 -> 242 us against 16 (tools/guidesweep.py)
// buckets per state of a sampling row: ESDP_GUIDE_RATIO in the environment overrides (measurement)
int guide_gmax(int K) {
  const char* e = getenv("ESDP_GUIDE_RATIO");
  const int ratio = (e && atoi(e) > 0) ? atoi(e) : kGuideRatio;
  int g = kGuideMinG;
  while (g < 14 && (1 << g) < ratio * K) ++g;
  return g;
}
int guide_g_for(size_t rows, size_t cap, int gmax) {
  int g = gmax;
  while (g > kGuideMinG && (rows << g) > cap) --g;
  return g;
}

// Identical stage slices P_t ([K][K]) share one sampling table (a time-homogeneous chain needs one, an
// hour-of-day chain 24): tab[t] = table of stage t + 1, src[u] = the first stage with table u.  Slices
// are hashed on the host pool, equal hashes confirmed byte for byte.
void dedupe_slices(const double* P, int nst, int K, std::vector<int>& tab, std::vector<int>& src) {
  const size_t n = (size_t)K * K;
  std::vector<uint64_t> h((size_t)nst);
  std::function<void(int)> hash = [&](int t) {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(P + (size_t)t * n);
    uint64_t x[4] = {0xcbf29ce484222325ull, 0x84222325cbf29ce4ull, 0x9e3779b97f4a7c15ull, 0xbf58476d1ce4e5b9ull};
    size_t j = 0;
    for (; j + 4 <= n; j += 4)   // four independent FNV-1a lanes
      for (int l = 0; l < 4; ++l) x[l] = (x[l] ^ w[j + l]) * 0x100000001b3ull;
    for (; j < n; ++j) x[0] = (x[0] ^ w[j]) * 0x100000001b3ull;
    h[(size_t)t] = ((x[0] * 31 + x[1]) * 31 + x[2]) * 31 + x[3];
  };
  if (nst > 1 && (size_t)nst * n > (1u << 16)) HostPool::get().run(nst, hash);
  else for (int t = 0; t < nst; ++t) hash(t);
  tab.assign((size_t)nst, 0);
  src.clear();
  // tentative tables by hash alone, then every slice compared with its representative in parallel; a hash
  // collision (any mismatch) redoes the assignment with byte comparisons
  {
    std::unordered_map<uint64_t, int> first;
    for (int t = 0; t < nst; ++t) {
      auto it = first.find(h[(size_t)t]);
      if (it == first.end()) {
        it = first.emplace(h[(size_t)t], (int)src.size()).first;
        src.push_back(t);
      }
      tab[(size_t)t] = it->second;
    }
    std::vector<char> bad((size_t)nst, 0);
    std::function<void(int)> check = [&](int t) {
      const int r = src[(size_t)tab[(size_t)t]];
      if (r != t) bad[(size_t)t] = std::memcmp(P + (size_t)r * n, P + (size_t)t * n, n * sizeof(double)) != 0;
    };
    if (nst > 1 && (size_t)nst * n > (1u << 16)) HostPool::get().run(nst, check);
    else for (int t = 0; t < nst; ++t) check(t);
    if (std::find(bad.begin(), bad.end(), 1) == bad.end()) return;
  }
  src.clear();
  std::unordered_map<uint64_t, std::vector<int>> seen;
  for (int t = 0; t < nst; ++t) {
    std::vector<int>& cand = seen[h[(size_t)t]];
    int u = -1;
    for (int v : cand)
      if (std::memcmp(P + (size_t)src[(size_t)v] * n, P + (size_t)t * n, n * sizeof(double)) == 0) { u = v; break; }
    if (u < 0) {
      u = (int)src.size();
      src.push_back(t);
      cand.push_back(u);
    }
    tab[(size_t)t] = u;
  }
}

esdp_status validate_data(esdp_ctx* c, const double* lambda, const double* P, const double* pi, const double* g) {
  for (long long j = 0; j < (long long)c->T * c->K; ++j)
    if (!std::isfinite(lambda[j])) return fail(c, ESDP_E_DATA, "lambda[%lld] is not finite", j);
  if (c->kind == ESDP_PAYOFF_LINEAR_MINUS_G && g) {   // g == NULL: the payoff is not being replaced
    for (int a = 0; a < c->A; ++a)
      if (!std::isfinite(g[a])) return fail(c, ESDP_E_DATA, "g[%d] is not finite", a);
  } else if (c->kind == ESDP_PAYOFF_TABLE && g) {
    for (long long j = 0; j < (long long)c->T * c->K * c->A; ++j)
      if (!std::isfinite(g[j])) return fail(c, ESDP_E_DATA, "payoff table entry %lld is not finite", j);
  }
  if (!c->rank1) {
    // the (T-1) K rows of P on the host thread pool; the first failing row is reported, as sequentially
    const long long rows = (long long)(c->T - 1) * c->K;
    const int nth = (int)std::max<long long>(1, std::min<long long>(4 * HostPool::get().size(), rows / 2048));
    std::vector<long long> bad((size_t)nth, rows);
    std::function<void(int)> scan = [&](int w) {
      const long long lo = rows * w / nth, hi = rows * (w + 1) / nth;
      for (long long r = lo; r < hi; ++r)
        if (!simplex_ok(P + r * c->K, c->K)) { bad[w] = r; return; }
    };
    if (nth == 1) scan(0);
    else HostPool::get().run(nth, scan);
    const long long r = *std::min_element(bad.begin(), bad.end());
    if (r < rows) return fail(c, ESDP_E_DATA, "row %lld of P is not a probability simplex", r);
    if (!simplex_ok(pi, c->K)) return fail(c, ESDP_E_DATA, "pi_1 is not a probability simplex");
  } else {
    for (int t = 0; t < c->T; ++t)
      if (!simplex_ok(pi + (long long)t * c->K, c->K)) return fail(c, ESDP_E_DATA, "pi_%d is not a probability simplex", t + 1);
  }
  return ESDP_OK;
}

// Alg. 1 lines 2-5 reduced to per-action (offset, weight); DESIGN §5 "layout".
// Affine fit of g over the window runs (NEXT-1 for payoffs lambda p - g(p) that are affine on each side,
// e.g. cfg3's linear degradation + fixed cycling cost): g(charge o) ~ gc0 + gc1 o, g(discharge |o|) ~
// gd0 + gd1 |o|.  f = {gc0, gc1, gd0, gd1, max deviation (+ slack for its own rounding), max |g|}.
// All zero for the linear payoff.
void fit_g(const esdp_ctx* c, const double* g, double f[6]) {
  for (int j = 0; j < 6; ++j) f[j] = 0.0;
  if (c->kind != ESDP_PAYOFF_LINEAR_MINUS_G || !g || c->a_z < 0 || c->Lc < 2 || c->Ld < 2) return;
  const int az = c->a_z, Lc = c->Lc, Ld = c->Ld;
  const double gc1 = (g[az - Lc] - g[az - 1]) / (double)(Lc - 1), gc0 = g[az - 1] - gc1;
  const double gd1 = (g[az + Ld] - g[az + 1]) / (double)(Ld - 1), gd0 = g[az + 1] - gd1;
  double dev = 0.0, gmax = 0.0;
  for (int o = 1; o <= Lc; ++o) dev = std::max(dev, std::fabs(g[az - o] - (gc0 + gc1 * o)));
  for (int o = 1; o <= Ld; ++o) dev = std::max(dev, std::fabs(g[az + o] - (gd0 + gd1 * o)));
  for (int b : c->live_list) gmax = std::max(gmax, std::fabs(g[b]));
  const double slack = 8.0 * 0x1p-53 * (gmax + std::fabs(gc0) + std::fabs(gd0) + std::fabs(gc1) * Lc + std::fabs(gd1) * Ld);
  f[0] = gc0; f[1] = gc1; f[2] = gd0; f[3] = gd1; f[4] = dev + slack; f[5] = gmax;
}

void build_tables(esdp_ctx* c, const double* g) {
  const int A = c->A;
  c->off.assign(A, 0);
  c->w.assign(A, 0.0);
  c->omw.assign(A, 1.0);
  c->F.assign(A, 0.0);
  for (int a = 0; a < A; ++a) {
    const double p = c->act[a];
    const double F = (p >= 0.0) ? -(p / c->eta_d) : -(c->eta_c * p);  // Eq. 2
    c->F[a] = F;
    const double e = F / c->delta;
    const double r = std::nearbyint(e);
    if (std::fabs(e - r) <= kGridTol) {
      c->off[a] = (int)r;
      c->w[a] = 0.0;
    } else {
      const double f = std::floor(e);
      c->off[a] = (int)f;
      c->w[a] = e - f;
    }
    c->omw[a] = 1.0 - c->w[a];
  }
  // An action is live if some row i in [0, S-1] can take it (i + o >= 0, i + o + [w > 0] <= S-1);
  // dead actions are infeasible everywhere (Eq. 4) and are left out of the stencil plan.
  auto live = [&](int b) {
    const int hi = c->off[b] + (c->w[b] != 0.0 ? 1 : 0);
    return c->off[b] >= -(c->S - 1) && hi <= c->S - 1;
  };
  // recombining runs: consecutive integral offsets decreasing by one
  c->segs.clear();
  int a = 0;
  while (a < A) {
    if (!live(a)) { ++a; continue; }
    Seg s{a, 1, c->off[a], c->w[a] != 0.0 ? 1 : 0};
    if (!s.interp) {
      while (a + s.n < A && live(a + s.n) && c->w[a + s.n] == 0.0 && c->off[a + s.n] == s.o0 - s.n) ++s.n;
    }
    c->segs.push_back(s);
    a += s.n;
  }
  c->o_min = 0;
  c->o_max = 0;
  for (int b = 0; b < A; ++b) {
    if (!live(b)) continue;
    c->o_min = std::min(c->o_min, c->off[b]);
    c->o_max = std::max(c->o_max, c->off[b] + (c->w[b] != 0.0 ? 1 : 0));
  }
  // window plan: zero action, charge run o = 1..Lc at a_z-1.., discharge run o = -1..-Ld at a_z+1..,
  // with powers matching -o*delta/eta_c resp. -o*delta*eta_d to a few ulps (the eps bound of
  // window.cuh assumes it).  Linear payoff, or lambda p - g(p) with g affine on each run (fit_g).
  c->use_window = 0;
  c->live_list.clear();
  c->singles.clear();
  for (int b = 0; b < A; ++b)
    if (live(b)) c->live_list.push_back(b);
  c->a_z = -1;
  for (int b = 0; b < A; ++b)
    if (c->act[b] == 0.0) c->a_z = b;
  if ((c->kind == ESDP_PAYOFF_LINEAR || c->kind == ESDP_PAYOFF_LINEAR_MINUS_G) && c->a_z >= 0 &&
      !(c->flags & ESDP_FORCE_BRUTE)) {
    const double u8 = 8.0 * 0x1p-53;
    int Lc = 0, Ld = 0;
    for (int b = c->a_z - 1; b >= 0; --b) {
      const int o = c->a_z - b;
      const double ideal = -((double)o * c->delta / c->eta_c);
      if (!live(b) || c->w[b] != 0.0 || c->off[b] != o || std::fabs(c->act[b] - ideal) > u8 * std::fabs(ideal)) break;
      ++Lc;
    }
    for (int b = c->a_z + 1; b < A; ++b) {
      const int o = c->a_z - b;
      const double ideal = (double)(-o) * c->delta * c->eta_d;
      if (!live(b) || c->w[b] != 0.0 || c->off[b] != o || std::fabs(c->act[b] - ideal) > u8 * std::fabs(ideal)) break;
      ++Ld;
    }
    c->Lc = Lc; c->Ld = Ld;
    double f[6];
    fit_g(c, g, f);
    const bool affine = c->kind == ESDP_PAYOFF_LINEAR || f[4] <= 1e-9 * (1.0 + f[5]);
    if (Lc >= 2 && Ld >= 2 && Lc <= 512 && Ld <= 512 && affine) {
      c->use_window = 1;
      c->pc = 0; while ((2 << c->pc) <= Lc) ++c->pc;
      c->pd = 0; while ((2 << c->pd) <= Ld) ++c->pd;
      for (int b : c->live_list)
        if (b < c->a_z - Lc || b > c->a_z + Ld || b == c->a_z) c->singles.push_back(b);
    }
  }
  const double x = c->s0 / c->delta;
  const double r = std::nearbyint(x);
  c->on_grid = std::fabs(x - r) <= kGridTol;
  c->f0 = c->on_grid ? (int)r : (int)std::floor(x);
  c->w0 = c->on_grid ? 0.0 : x - std::floor(x);
}

template <class T>
esdp_status dev_alloc(esdp_ctx* c, T** p, size_t n) {
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc((void**)p, n * sizeof(T));
  if (e != cudaSuccess) return fail(c, ESDP_E_NOMEM, "cudaMalloc(%zu bytes): %s", n * sizeof(T), cudaGetErrorString(e));
  return ESDP_OK;
}

void free_all(esdp_ctx* c) {
  for (cudaGraphExec_t g : c->graphs)
    if (g) cudaGraphExecDestroy(g);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->slot[0].lambda) {   // full context: the input aliases point into the slots
    for (InputSlot& x : c->slot) {
      void* sp[] = {x.lambda, x.P, x.pi, x.cdf, x.cdf1, x.g, x.gfit, x.guide, x.guide1, x.tab, x.src};
      for (void* p : sp)
        if (p) cudaFree(p);
      for (cudaEvent_t e : x.chunk_ev) cudaEventDestroy(e);
      if (x.ev_head) cudaEventDestroy(x.ev_head);
      if (x.ev_tables) cudaEventDestroy(x.ev_tables);
      if (x.use_ev) cudaEventDestroy(x.use_ev);
      if (x.stage_ev) cudaEventDestroy(x.stage_ev);
      if (x.stage_h) cudaFreeHost(x.stage_h);
      if (x.gfit_stage) cudaFreeHost(x.gfit_stage);
    }
    c->d_lambda = c->d_P = c->d_pi = c->d_cdf = c->d_cdf1 = c->d_g = c->d_gfit = nullptr;
    c->d_guide = c->d_guide1 = nullptr;
  }
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  for (cudaEvent_t e : c->fb_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : c->join_ev) cudaEventDestroy(e);
  for (cudaStream_t x : c->side) cudaStreamDestroy(x);
  if (c->copy) cudaStreamDestroy(c->copy);
  void* ps[] = {c->d_lambda, c->d_P, c->d_pi, c->d_g, c->d_act, c->d_w, c->d_omw, c->d_off, c->d_segs,
                c->d_V, c->d_W, c->d_J, c->d_cdf, c->d_cdf1, c->d_guide, c->d_guide1, c->d_singles, c->d_live, c->d_gfit, c->d_F, c->d_stack, c->d_fb_req, c->d_fb_slot, c->d_red, c->d_pol, c->d_sim, c->d_req,
                c->d_nv, c->d_vert, c->d_q, c->d_price};
  for (void* p : ps)
    if (p) cudaFree(p);
  if (c->stream) cudaStreamDestroy(c->stream);
}

// Enqueue the upload of the given inputs into slot dst on the copy stream, after every enqueued use of
// that slot; a NULL array keeps the data of slot src (device-to-device copy when src != dst).  lambda /
// pi / g and their tables first (ev_head), then P in stage chunks in the order the backward needs them
// (chunk_ev), then the simulation's sampling tables of P (ev_tables).  Does not synchronize.
esdp_status upload(esdp_ctx* c, int dst, int src, const double* lambda, const double* P, const double* pi,
                   const double* g) {
  const size_t TK = (size_t)c->T * c->K, K = c->K;
  InputSlot& d = c->slot[dst];
  const InputSlot& o = c->slot[src];
  const bool copy_old = src != dst;
  cudaStream_t s = c->copy;
  const auto h2d = cudaMemcpyHostToDevice;
  const auto d2d = cudaMemcpyDeviceToDevice;
  if (d.use_pending) CUDA_OR_FAIL(c, cudaStreamWaitEvent(s, d.use_ev, 0));
  // Copies out of slot src must see its sampling tables complete: ready_tables() may have enqueued
  // their (lazy) build on a simulation stream and re-recorded ev_tables there.
  // No kernel runs on the copy stream while a backward graph may be running: ONE kernel of another stream
  // enqueued during the pipelined loop's graph cost it ~0.22 ms on B200 (tools/e2eprobe.py kernel / evrec /
  // dma: a DMA or an event record costs nothing), and small device-to-device copies run as kernels.  So the sampling tables are
  // built by the first simulation that needs them (ready_tables, after the backward), and a kept (NULL)
  // array is copied from slot src only if dst does not already hold the same data (generations).
  const bool cp_lam = !lambda && copy_old && d.gen_lambda != o.gen_lambda;
  const bool cp_pi = !pi && copy_old && d.gen_pi != o.gen_pi;
  const bool new_g = g && (c->kind == ESDP_PAYOFF_LINEAR_MINUS_G || c->kind == ESDP_PAYOFF_TABLE);
  const bool cp_g = !new_g && copy_old && d.gen_g != o.gen_g;
  const bool cp_P = !c->rank1 && !P && copy_old && d.gen_P != o.gen_P;
  if (cp_lam || cp_pi || cp_g || cp_P) CUDA_OR_FAIL(c, cudaStreamWaitEvent(s, o.ev_tables, 0));
  if (lambda) {
    CUDA_OR_FAIL(c, cudaMemcpyAsync(d.lambda, lambda, TK * sizeof(double), h2d, s));
    d.gen_lambda = ++c->gen;
  } else if (cp_lam) {
    CUDA_OR_FAIL(c, cudaMemcpyAsync(d.lambda, o.lambda, TK * sizeof(double), d2d, s));
    d.gen_lambda = o.gen_lambda;
  }
  const size_t npi = c->rank1 ? TK : K;
  if (pi) {
    CUDA_OR_FAIL(c, cudaMemcpyAsync(d.pi, pi, npi * sizeof(double), h2d, s));
    d.pi_stale = true;
    d.gen_pi = ++c->gen;
  } else if (cp_pi) {
    d.gen_pi = o.gen_pi;
    CUDA_OR_FAIL(c, cudaMemcpyAsync(d.pi, o.pi, npi * sizeof(double), d2d, s));
    d.pi_stale = o.pi_stale;
    if (!o.pi_stale) {
      CUDA_OR_FAIL(c, cudaMemcpyAsync(d.cdf1, o.cdf1, K * sizeof(double), d2d, s));
      CUDA_OR_FAIL(c, cudaMemcpyAsync(d.guide1, o.guide1, sizeof(uint64_t) << c->g_max, d2d, s));
      if (c->rank1) {
        CUDA_OR_FAIL(c, cudaMemcpyAsync(d.cdf, o.cdf, TK * sizeof(double), d2d, s));
        CUDA_OR_FAIL(c, cudaMemcpyAsync(d.guide, o.guide, ((size_t)c->T << c->g_r1) * sizeof(uint64_t), d2d, s));
      }
    }
  }
  const size_t ng = c->kind == ESDP_PAYOFF_TABLE ? TK * c->A : (size_t)c->A;
  // the staging of dst is rewritten below: its previous copies (an earlier upload into dst) must have run
  if (g || P) CUDA_OR_FAIL(c, cudaEventSynchronize(d.stage_ev));
  bool staged = false;
  if (g && c->kind == ESDP_PAYOFF_LINEAR_MINUS_G) {
    CUDA_OR_FAIL(c, cudaMemcpyAsync(d.g, g, c->A * sizeof(double), h2d, s));
    // a later g that is not affine on the runs only widens eps (more canonical fallbacks, same result)
    if (c->use_window) fit_g(c, g, d.gfit_h);
    std::memcpy(d.gfit_stage, d.gfit_h, sizeof d.gfit_h);
    CUDA_OR_FAIL(c, cudaMemcpyAsync(d.gfit, d.gfit_stage, sizeof d.gfit_h, h2d, s));
    staged = true;
    d.gen_g = ++c->gen;
  } else if (g && c->kind == ESDP_PAYOFF_TABLE) {
    CUDA_OR_FAIL(c, cudaMemcpyAsync(d.g, g, ng * sizeof(double), h2d, s));
    d.gen_g = ++c->gen;
  } else if (cp_g) {   // (a g given with the LINEAR payoff is ignored, as a NULL one)
    d.gen_g = o.gen_g;
    CUDA_OR_FAIL(c, cudaMemcpyAsync(d.g, o.g, ng * sizeof(double), d2d, s));
    std::memcpy(d.gfit_h, o.gfit_h, sizeof d.gfit_h);
    CUDA_OR_FAIL(c, cudaMemcpyAsync(d.gfit, o.gfit, sizeof d.gfit_h, d2d, s));
  }
  CUDA_OR_FAIL(c, cudaEventRecord(d.ev_head, s));
  // P chunks: the backward waits only for the copy; the sampling tables (needed by the simulation
  // alone) are built after it and signalled by ev_tables
  for (size_t j = 0; j < d.chunk_ev.size(); ++j) {
    if (P || cp_P) {
      const size_t r0 = (size_t)(c->chunk_lo[j] - 1) * K, nr = (size_t)(c->chunk_hi[j] - c->chunk_lo[j] + 1) * K;
      if (P) CUDA_OR_FAIL(c, cudaMemcpyAsync(d.P + r0 * K, P + r0 * K, nr * K * sizeof(double), h2d, s));
      else CUDA_OR_FAIL(c, cudaMemcpyAsync(d.P + r0 * K, o.P + r0 * K, nr * K * sizeof(double), d2d, s));
    }
    CUDA_OR_FAIL(c, cudaEventRecord(d.chunk_ev[j], s));
  }
  // The sampling tables of P are built lazily by the first simulation that needs them (ready_tables), on
  // that simulation's stream (see above: even a few blocks here stretched the running backward).
  if (!c->rank1 && c->T > 1) {
    const int nst = c->T - 1;
    if (P) {   // one table per distinct slice P_t; as many guide bits as the allocation allows
      std::vector<int> tab, src;
      dedupe_slices(P, nst, c->K, tab, src);
      d.nuniq = (int)src.size();
      d.gbits = guide_g_for((size_t)d.nuniq * K, c->guide_cap, c->g_max);
      std::memcpy(d.stage_h, tab.data(), nst * sizeof(int));
      std::memcpy(d.stage_h + nst, src.data(), src.size() * sizeof(int));
      CUDA_OR_FAIL(c, cudaMemcpyAsync(d.tab, d.stage_h, nst * sizeof(int), h2d, s));
      CUDA_OR_FAIL(c, cudaMemcpyAsync(d.src, d.stage_h + nst, src.size() * sizeof(int), h2d, s));
      staged = true;
      d.tables_stale = true;
      d.gen_P = ++c->gen;
    } else if (cp_P) {
      d.gen_P = o.gen_P;
      d.nuniq = o.nuniq;
      d.gbits = o.gbits;
      CUDA_OR_FAIL(c, cudaMemcpyAsync(d.tab, o.tab, nst * sizeof(int), d2d, s));
      CUDA_OR_FAIL(c, cudaMemcpyAsync(d.src, o.src, nst * sizeof(int), d2d, s));
      if (o.tables_stale) {
        d.tables_stale = true;
      } else {
        const size_t nr = (size_t)d.nuniq * K;
        CUDA_OR_FAIL(c, cudaMemcpyAsync(d.cdf, o.cdf, nr * K * sizeof(double), d2d, s));
        CUDA_OR_FAIL(c, cudaMemcpyAsync(d.guide, o.guide, (nr << d.gbits) * sizeof(uint64_t), d2d, s));
        d.tables_stale = false;
      }
    }
  }
  if (staged) CUDA_OR_FAIL(c, cudaEventRecord(d.stage_ev, s));
  CUDA_OR_FAIL(c, cudaEventRecord(d.ev_tables, s));
  return ESDP_OK;
}

// The active slot's sampling tables in a simulation's parameters.
void sim_tables(const esdp_ctx* c, SimParams& sp) {
  const InputSlot& x = c->slot[c->active];
  sp.cdf = x.cdf; sp.cdf1 = x.cdf1; sp.guide = x.guide; sp.guide1 = x.guide1;
  sp.tab = c->rank1 ? nullptr : x.tab;
  sp.gs = 53 - x.gbits;
  sp.gs1 = 53 - c->g_max;
}

// Before a simulation on stream s: wait for the active slot's uploads and build whichever of its sampling
// tables (pi's, P's) the uploads left stale.
esdp_status ready_tables(esdp_ctx* c, cudaStream_t s) {
  InputSlot& x = c->slot[c->active];
  CUDA_OR_FAIL(c, cudaStreamWaitEvent(s, x.ev_tables, 0));
  if (!x.pi_stale && !x.tables_stale) return ESDP_OK;
  // one launch: the rows (rank-1: the per-stage marginals pi_{t+1}; Markov: the distinct slices of P) and
  // the single row pi_1 (row 0 of pi in rank-1), each only if stale
  const double* q1 = x.pi_stale ? x.pi : nullptr;
  if (c->rank1)
    launch_cdf(x.pi, nullptr, x.pi_stale ? c->T : 0, c->K, c->g_r1, x.cdf, x.guide, s, q1, c->g_max, x.cdf1, x.guide1);
  else
    launch_cdf(x.P, x.src, x.tables_stale ? (int64_t)x.nuniq * c->K : 0, c->K, x.gbits, x.cdf, x.guide, s, q1,
               c->g_max, x.cdf1, x.guide1);
  CUDA_OR_FAIL(c, cudaGetLastError());
  CUDA_OR_FAIL(c, cudaEventRecord(x.ev_tables, s));   // later copies out of this slot wait for the builds
  x.pi_stale = x.tables_stale = false;
  return ESDP_OK;
}

// After enqueueing work that reads the active slot's inputs on stream s: later uploads into that slot
// wait for it.
esdp_status mark_use(esdp_ctx* c, cudaStream_t s) {
  InputSlot& x = c->slot[c->active];
  CUDA_OR_FAIL(c, cudaEventRecord(x.use_ev, s));
  x.use_pending = true;
  return ESDP_OK;
}

size_t w_rows(const esdp_ctx* c) { return c->rank1 ? 1 : (size_t)c->kmax; }
bool keep(const esdp_ctx* c) { return (c->flags & ESDP_KEEP_VALUES) != 0; }
// V_t / W_t / pol_t device slices (stage t = 1..T)
double* V_of(esdp_ctx* c, int t) {
  const size_t KS = (size_t)c->Kp * c->ld;
  return keep(c) ? c->d_V + (size_t)(t - 1) * KS : c->d_V + (size_t)((t - 1) & 1) * KS;
}
double* W_of(esdp_ctx* c, int t) {
  const size_t RS = w_rows(c) * c->ld;
  return keep(c) ? c->d_W + (size_t)(t - 1) * RS : c->d_W;
}

// cudaLaunchKernelEx with the programmatic-stream-serialization attribute (PDL) when pdl is set, and a
// preferred shared-memory carveout (percent) when carve >= 0.
template <typename... KArgs, typename... Args>
cudaError_t launch_c(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl, int carve,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (carve >= 0) {
    attr[na].id = cudaLaunchAttributePreferredSharedMemoryCarveout;
    attr[na].val.sharedMemCarveout = (unsigned)carve;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl, Args... args) {
  return launch_c(kern, grid, block, smem, s, pdl, -1, args...);
}
// Carveout of a context's stage-chain launches: in the latency regime (the one-output-per-thread window plan,
// e.g. cfg2) the expectation, stencil and objective all ask for the maximum shared-memory carveout, so that
// consecutive kernels share one L1/shared split and the next grid's blocks can become resident beside the
// draining one: cfg2 step 2.416 -> 2.377 ms.  In the throughput regime (cfg4, the Table 3 largest row, batches)
// the same setting measured 0.8-1.3 % slower, so those keep the default.  ESDP_CARVEOUT=<percent> forces a
// value everywhere on the chain, ESDP_CARVEOUT=-1 disables it (measurement).
int chain_carveout(const esdp_ctx* c);

// k'-pipelined DMMA expectation (contract_dmma3_kernel), two tilings: 16 x 64 block tiles (four 16x16
// warp tiles) for large contractions (cfg4, cfg5 batches: >= 3e5 outputs), 8 x 32 block tiles (two 8x16
// warp tiles) below, where the grid must cover every SM (cfg2: 416 blocks).  Measured (tools/variants_d3*.sh,
// warm launches): cfg4 11.8 -> 9.6 us, cfg2 3.59 -> 3.25 us against dmma2.  ESDP_DMMA3=0 in the environment
// falls back to dmma2 (measurement).
#ifndef ESDP_D3_MT
#define ESDP_D3_MT 2
#endif
#ifndef ESDP_D3_NT
#define ESDP_D3_NT 2
#endif
#ifndef ESDP_D3_WC
#define ESDP_D3_WC 4
#endif
#ifndef ESDP_D3_KC
#define ESDP_D3_KC 16
#endif
#ifndef ESDP_D3_NS
#define ESDP_D3_NS 4
#endif
using D3 = Dmma3<ESDP_D3_MT, ESDP_D3_NT, ESDP_D3_WC, ESDP_D3_KC, ESDP_D3_NS>;
#define D3_KERNEL contract_dmma3_kernel<ESDP_D3_MT, ESDP_D3_NT, ESDP_D3_WC, ESDP_D3_KC, ESDP_D3_NS>
#ifndef ESDP_D3S_KC
#define ESDP_D3S_KC 16
#endif
#ifndef ESDP_D3S_NS
#define ESDP_D3S_NS 4
#endif
// Small tiling: 16 x 16 block tiles of two 16 x 8 warp tiles (MT = 2, NT = 1, WC = 2) since the
// latency-regime chain launches with the maximum shared-memory carveout: cfg2 backward 1.953 -> 1.935 ms, warm
// launch 3.27 -> 3.16 us (tools/variants_d3s.sh; before the carveout the 8 x 32 tiling of two 8 x 16 warps led).
// Rank-1 GEMVs (one live row) keep the 8-row tiling (D3r): a 16-row tile would idle 15 of its 16 rows.
#ifndef ESDP_D3S_NT
#define ESDP_D3S_NT 1
#endif
#ifndef ESDP_D3S_WC
#define ESDP_D3S_WC 2
#endif
#ifndef ESDP_D3S_MT
#define ESDP_D3S_MT 2
#endif
using D3s = Dmma3<ESDP_D3S_MT, ESDP_D3S_NT, ESDP_D3S_WC, ESDP_D3S_KC, ESDP_D3S_NS>;
#define D3S_KERNEL contract_dmma3_kernel<ESDP_D3S_MT, ESDP_D3S_NT, ESDP_D3S_WC, ESDP_D3S_KC, ESDP_D3S_NS>
using D3r = Dmma3<1, 2, 2, 16, 4>;
#define D3R_KERNEL contract_dmma3_kernel<1, 2, 2, 16, 4>
// Wide tiling for very large products (the cfg5 batch GEMM, [100] x [128,512]): 16 x 128 block tiles of four
// 16 x 32 warp tiles, two pipeline stages (40 KB: five blocks per SM).  Measured over 17 tilings
// (tools/variants_d3_cfg5.sh): 108.1 us per cfg5 stage against 122.5 us for the large tiling, which stays
// best on cfg4 (9.6 vs 13.2 us per launch).
using D3w = Dmma3<2, 4, 4, 16, 2>;
#define D3W_KERNEL contract_dmma3_kernel<2, 4, 4, 16, 2>
constexpr double kDmma3MinOutputs = 3.0e5, kDmma3WideOutputs = 4.0e6;
// 0: not applicable (odd K, fewer than 8 rows, or ESDP_DMMA3=0); 1: small tiling; 2: large; 3: wide (4: the
// rank-1 8-row tiling, chosen by launch_contract)
int use_dmma3(int rows, int64_t ncols, int K) {
  if (rows < 8 || (K & 1)) return 0;
  static const int force = [] { const char* e = getenv("ESDP_DMMA3"); return e ? atoi(e) : -1; }();
  if (force == 0) return 0;
  const double outs = (double)rows * (double)ncols;
  return outs >= kDmma3WideOutputs ? 3 : outs >= kDmma3MinOutputs ? 2 : 1;
}
template <typename DD>
cudaError_t launch_dmma3_as(void (*kern)(const double*, const double*, double*, int, int, int, int, int), const double* Pt,
                            const double* Vn, double* Wt, int rows, int K, int S, int ld, cudaStream_t s, bool pdl,
                            int carve) {
  if (DD::smem() > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DD::smem());
    if (e != cudaSuccess) return e;
  }
  const int nrb = (rows + DD::RB - 1) / DD::RB;
  const int64_t ncb = ((int64_t)S + DD::CB - 1) / DD::CB;
  return launch_c(kern, dim3((unsigned)(ncb * nrb)), dim3(DD::NTH), DD::smem(), s, pdl, carve, Pt, Vn, Wt, rows, K, S, ld,
                  nrb);
}
cudaError_t launch_dmma3(int which, const double* Pt, const double* Vn, double* Wt, int rows, int K, int S, int ld,
                         cudaStream_t s, bool pdl, int carve = -1) {
  if (which == 4) return launch_dmma3_as<D3r>(D3R_KERNEL, Pt, Vn, Wt, rows, K, S, ld, s, pdl, carve);
  return which == 3 ? launch_dmma3_as<D3w>(D3W_KERNEL, Pt, Vn, Wt, rows, K, S, ld, s, pdl, carve)
       : which == 2 ? launch_dmma3_as<D3>(D3_KERNEL, Pt, Vn, Wt, rows, K, S, ld, s, pdl, carve)
                    : launch_dmma3_as<D3s>(D3S_KERNEL, Pt, Vn, Wt, rows, K, S, ld, s, pdl, carve);
}

// P-resident persistent expectation (contract_pres_kernel) for wide products: rows, K <= 104 (13 row
// fragments), K and ncols even.  ESDP_PRES=0 in the environment keeps the block-tiled dmma3 (measurement).
#ifndef ESDP_PRES_NW
#define ESDP_PRES_NW 8
#endif
#ifndef ESDP_PRES_NT
#define ESDP_PRES_NT 1
#endif
constexpr int kPresMTA = 13, kPresNW = ESDP_PRES_NW, kPresNT = ESDP_PRES_NT;
using DPres = DmmaPres<kPresMTA, kPresNW, kPresNT>;
bool use_pres(int rows, int K, int64_t ncols) {
  const char* e = getenv("ESDP_PRES");
  if (e && atoi(e) == 0) return false;
  return rows <= 8 * kPresMTA && K <= 8 * kPresMTA && !(K & 1) && !(ncols & 1) && ncols <= INT32_MAX &&
         (double)rows * (double)ncols >= kDmma3WideOutputs && DPres::smem(K) <= 227 * 1024;
}
cudaError_t launch_pres(const double* Pt, const double* Vn, double* Wt, int rows, int K, int64_t ncols, int ld,
                        cudaStream_t s, bool pdl) {
  int dev = 0, nsm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const size_t sm = DPres::smem(K);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(contract_pres_kernel<kPresMTA, kPresNW, kPresNT>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (ncols + DPres::CT - 1) / DPres::CT;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, nsm));
  return launch(contract_pres_kernel<kPresMTA, kPresNW, kPresNT>, dim3(grid), dim3(DPres::NTH), sm, s, pdl, Pt, Vn, Wt, rows, K,
                (int)ncols, ld);
}

// Ozaki-sliced u8 tcgen05 expectation (ozaki.cuh): one persistent CTA per SM over 32-column tiles.
// Requires rows <= 128, K <= 128, non-negative P and V.
cudaError_t launch_ozaki(const double* Pt, const double* Vn, double* Wt, int rows, int K, long long ncols, long long ldv,
                         long long ldw, cudaStream_t s, bool pdl) {
  int dev = 0, nsm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(ozaki_contract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOzSmem);
  if (e != cudaSuccess) return e;
  const long long ntiles = (ncols + kOzN - 1) / kOzN;
  const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(ntiles, nsm));
  return launch(ozaki_contract_kernel, dim3(grid), dim3(kOzThreads), kOzSmem, s, pdl, Pt, Vn, Wt, rows, K, ncols, ldv, ldw);
}

int chain_carveout(const esdp_ctx* c) {
  const char* e = getenv("ESDP_CARVEOUT");   // read per launch (graph capture): tests and measurement
  if (e) return atoi(e);
  return (c->use_window && c->win_opt == 1) ? (int)cudaSharedmemCarveoutMaxShared : -1;
}

// The contraction of stage t (t < T): W_t = P_t V_{t+1}.
cudaError_t launch_contract(esdp_ctx* c, int t, cudaStream_t s, bool pdl) {
  const int K = c->K, S = c->S;
  const int rows = c->rank1 ? 1 : c->k_cnt;   // own rows of W_t (all rows on one GPU)
  if (rows == 0) return cudaSuccess;
  const double* Pt = c->rank1 ? c->d_pi + (size_t)t * K : c->d_P + ((size_t)(t - 1) * K + c->k_lo) * K;
  // rank-1 (the paper's Alg. 1 GEMV W = pi_{t+1}^T V_{t+1}): one A row of the 8-row DMMA tile is live; the
  // K/4-long DMMA chain per column replaces a K-long DFMA chain (same canonical order, same bits)
  const int cv = chain_carveout(c);
  if (rows == 1 && !(K & 1) && !(c->flags & ESDP_NO_DMMA) && use_dmma3(8, S, K))
    return launch_dmma3(4, Pt, (const double*)V_of(c, t + 1), W_of(c, t), 1, K, S, c->ld, s, pdl, cv);
  if (rows >= 8 && !(c->flags & ESDP_NO_DMMA)) {   // FP64 tensor cores (bit-identical chain, see kernels.cuh)
    if (const int d3 = use_dmma3(rows, S, K))
      return launch_dmma3(d3, Pt, (const double*)V_of(c, t + 1), W_of(c, t), rows, K, S, c->ld, s, pdl, cv);
    if (c->dmma2) {
      if (K > 128) {   // large K: taller tiles (fewer re-reads of the V column block)
        const int ncb = (S + kDCbig * 16 - 1) / (kDCbig * 16), nrb = (rows + kDRbig * 8 - 1) / (kDRbig * 8);
        return launch_c(contract_dmma2_kernel<kDRbig, kDCbig>, dim3(ncb * nrb), dim3(kDRbig * kDCbig * 32),
                        contract_dmma2_smem(K, kDRbig, kDCbig), s, pdl, cv, Pt, (const double*)V_of(c, t + 1), W_of(c, t),
                        rows, K, S, c->ld, ncb);
      }
      const int ncb = (S + kDC * 16 - 1) / (kDC * 16), nrb = (rows + kDR * 8 - 1) / (kDR * 8);
      return launch_c(contract_dmma2_kernel<kDR, kDC>, dim3(ncb * nrb), dim3(kDR * kDC * 32), contract_dmma2_smem(K), s,
                      pdl, cv, Pt, (const double*)V_of(c, t + 1), W_of(c, t), rows, K, S, c->ld, ncb);
    }
  }   // else (K too large for any staged DMMA tile): DFMA below
  dim3 grid((S + kColsC - 1) / kColsC, (rows + kRowsC - 1) / kRowsC);
  return launch_c(contract_kernel, grid, dim3(kThreadsC), contract_smem_bytes(K), s, pdl, cv, Pt,
                  (const double*)V_of(c, t + 1), W_of(c, t), rows, K, S, c->ld);
}

// Stage-invariant parameters of the window and brute-force stencils (W/V/pol/lambda set per launch).
WinParams win_params(const esdp_ctx* c) {
  WinParams wp{};
  wp.act = c->d_act; wp.w = c->d_w; wp.omw = c->d_omw; wp.off = c->d_off;
  wp.singles = c->d_singles; wp.live = c->d_live;
  wp.nsingle = (int)c->singles.size(); wp.nlive = (int)c->live_list.size();
  wp.A = c->A; wp.S = c->S; wp.K = c->k_cnt; wp.rank1 = c->rank1; wp.ld = c->ld;
  wp.a_z = c->a_z; wp.Lc = c->Lc; wp.Ld = c->Ld; wp.pc = c->pc; wp.pd = c->pd;
  wp.o_min = c->o_min; wp.o_max = c->o_max;
  wp.delta = c->delta; wp.eta_c = c->eta_c; wp.eta_d = c->eta_d; wp.pbar = c->pbar;
  wp.dc = c->delta / c->eta_c; wp.dd = c->delta * c->eta_d;
  wp.jspan = (double)(c->S + (c->o_max - c->o_min) + 2);
  wp.g = c->d_g; wp.gfit = c->d_gfit; wp.g_kind = c->kind == ESDP_PAYOFF_LINEAR_MINUS_G;
  { const char* e = getenv("ESDP_WIN_FORCE_NONUNI"); wp.force_nonuni = (e && atoi(e)) ? 1 : 0; }   // tests only
  for (int j = 0; j < (int)c->singles.size() && j < kMaxSingles; ++j) {
    const int a = c->singles[j];
    wp.sg[j].act = c->act[a]; wp.sg[j].w = c->w[a]; wp.sg[j].omw = c->omw[a]; wp.sg[j].off = c->off[a]; wp.sg[j].a = a;
  }
  // the Eq. 10 grid with interpolated endpoints: singles = {charge endpoint, zero action, discharge endpoint}
  wp.eq10 = c->singles.size() == 3 && c->singles[1] == c->a_z && c->w[c->singles[0]] != 0.0 &&
            c->w[c->singles[2]] != 0.0 && c->singles[0] < c->a_z && c->singles[2] > c->a_z;
  { const char* e = getenv("ESDP_WIN_GENERIC"); wp.force_generic = (e && atoi(e)) ? 1 : 0; }   // tests / measurement
  return wp;
}

StencilParams stencil_params(const esdp_ctx* c) {
  StencilParams prm{};
  prm.act = c->d_act; prm.g = c->d_g;
  prm.w = c->d_w; prm.omw = c->d_omw; prm.off = c->d_off; prm.segs = c->d_segs; prm.nseg = (int)c->segs.size();
  prm.A = c->A; prm.S = c->S; prm.K = c->k_cnt; prm.kind = c->kind; prm.rank1 = c->rank1;
  prm.o_min = c->o_min; prm.o_span = c->o_max - c->o_min; prm.ld = c->ld;
  return prm;
}

// window_stencil_kernel variants: OPT outputs per thread (2: throughput regime), packed level tables for
// payoffs with non-unimodal run tables (LINEAR_MINUS_G); the linear payoff scans a non-unimodal window.
void (*window_kernel_of(int opt, int levels))(WinParams) {
  if (levels) return window_stencil_kernel<1, true>;
  return opt == 4 ? window_stencil_kernel<4, false> : opt == 2 ? window_stencil_kernel<2, false>
                  : window_stencil_kernel<1, false>;
}
// Plan of the window kernel variant.  ESDP_WIN_OPT=1|2|4 in the environment overrides the choice (measurement).
void plan_window(esdp_ctx* c, int64_t blocks1) {
  const char* e = getenv("ESDP_WIN_OPT");   // read per context: tests switch variants within one process
  const int env = e ? atoi(e) : 0;
  c->win_levels = c->kind == ESDP_PAYOFF_LINEAR_MINUS_G;
  // four outputs per thread once the one-output grid exceeds ~2 waves (4 resident blocks per SM): cfg4 stencil
  // 7.26 (two) -> 6.31 us (four) per launch, measured (tools/winvariants.sh)
  c->win_opt = c->win_levels ? 1 : (env == 1 || env == 2 || env == 4) ? env : (blocks1 > 2 * 4 * 148 ? 4 : 1);
  c->window_smem = window_smem_bytes(c->Lc, c->Ld, c->o_max - c->o_min, c->A, c->win_opt, c->win_levels != 0);
}

// The max-plus stencil of stage t: V_t, pol_t from W_t (window or brute force).
cudaError_t launch_stencil(esdp_ctx* c, int t, cudaStream_t s, bool pdl, bool force_brute) {
  const int S = c->S;
  const int K = c->k_cnt;                      // stencil rows of this rank (local k = global k - k_lo)
  if (K == 0) return cudaSuccess;
  const double* Wt = W_of(c, t);
  int16_t* pol = c->d_pol + ((size_t)(t - 1) * c->Kp + c->k_lo) * S;
  const double* lam = c->d_lambda + (size_t)(t - 1) * c->K + c->k_lo;
  if (c->use_window && !force_brute) {
    WinParams wp = win_params(c);
    wp.W = Wt; wp.V = V_of(c, t) + (size_t)c->k_lo * c->ld; wp.pol = pol; wp.lambda_t = lam;
    const int tile = kWinThreads * c->win_opt;
    return launch_c(window_kernel_of(c->win_opt, c->win_levels), dim3((S + tile - 1) / tile, K), dim3(kWinThreads),
                    c->window_smem, s, pdl, chain_carveout(c), wp);
  }
  StencilParams prm = stencil_params(c);
  prm.W = Wt; prm.V = V_of(c, t) + (size_t)c->k_lo * c->ld; prm.pol = pol; prm.lambda_t = lam;
  prm.g = c->kind == ESDP_PAYOFF_TABLE ? c->d_g + ((size_t)(t - 1) * c->K + c->k_lo) * c->A : c->d_g;
  return launch_c(stencil_kernel, dim3((S + kTile - 1) / kTile, K), dim3(kStencilWarps * 32), c->stencil_smem, s, pdl,
                  chain_carveout(c), prm);
}

cudaError_t launch_objective(esdp_ctx* c, cudaStream_t s, bool pdl) {
  return launch_c(objective_kernel, dim3(1), dim3(128), 2 * sizeof(double) * c->K, s, pdl, chain_carveout(c),
                  (const double*)V_of(c, 1), (const double*)c->d_pi, c->K, c->ld, c->f0, c->w0, c->on_grid, c->d_J);
}

cudaError_t launch_bids(esdp_ctx* c, int64_t n, const int32_t* req_dev, const int32_t* slot_dev, int64_t nout, int32_t cap,
                        int32_t* nvert_dev, int16_t* vert_dev, double* q_dev, double* price_dev, cudaStream_t s) {
  BidParams bp{c->d_W, c->d_act, c->d_w, c->d_omw, c->d_off, c->d_g, c->T, c->K, c->S, c->A, c->rank1, c->kind, c->ld,
               (int)w_rows(c), c->k_lo, c->rank1 ? c->K : c->k_cnt};
  const int span = c->o_max - c->o_min;
  const unsigned blocks = (unsigned)((n + kBidThreads - 1) / kBidThreads);
  const bool g = c->kind == ESDP_PAYOFF_LINEAR_MINUS_G;
  auto go = [&](auto kern, size_t sm) {
    if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<blocks, kBidThreads, sm, s>>>(bp, n, req_dev, slot_dev, nout, cap, c->o_min, span, nvert_dev, vert_dev, q_dev,
                                         price_dev);
  };
  // Hull stacks in shared memory as 8-bit indices (A <= 255: 25 KB per block at A = 201, six blocks per SM);
  // wider grids keep the stack in the curve's own vertex row in global memory: a 16-bit shared-memory stack
  // (102 KB at A = 401) allowed one block per SM and measured 3x slower (cfg4: 110 -> 36 ms of bid curves
  // per step; on cfg2 the global stack is slower, 2.88 vs 2.43 ms per step).
  if (c->A <= 255) {
    const size_t sm = bid_smem_bytes(c->A, span, true, 1);
    if (g) go(bidcurve_kernel<true, uint8_t, true>, sm); else go(bidcurve_kernel<true, uint8_t, false>, sm);
  } else {
    const size_t sm = bid_smem_bytes(c->A, span, false, 2);
    if (g) go(bidcurve_kernel<false, int16_t, true>, sm); else go(bidcurve_kernel<false, int16_t, false>, sm);
  }
  return cudaGetLastError();
}

// Enqueue the 2T launches of one backward pass on stream s (PDL between consecutive kernels).
esdp_status enqueue_backward(esdp_ctx* c, cudaStream_t s) {
  const int T = c->T;
  int64_t n = 0;
  const bool prof = !c->ev.empty();
  const bool pdl = c->pdl;
  // ESDP_PROFILE: events around the kernels of every prof_stride-th stage only (a live sample of the
  // launch durations that keeps event nodes out of most of the graph)
  auto sampled = [&](int t) { return prof && t % c->prof_stride == 0; };
  auto mark = [&](int t, int j) {
    return sampled(t) ? cudaEventRecordWithFlags(c->ev[(size_t)(t - 1) * 4 + j], s, cudaEventRecordExternal) : cudaSuccess;
  };
  bool after_kernel = false;  // a PDL edge needs a kernel predecessor
  bool forked = false;
  // fused bid curves: 0 = side branches along the chain (default); 1 = the same batches, forked after stage 1;
  // 2 = one launch over every request on the chain stream after stage 1 (ESDP_FB_MODE, measurement)
  const int fb_mode = [] { const char* e = getenv("ESDP_FB_MODE"); return e ? atoi(e) : 0; }();
  std::vector<char> side_used(c->side.size(), 0);
  for (int t = T; t >= 1; --t) {
    if (t == T) {
      CUDA_OR_FAIL(c, cudaMemsetAsync(W_of(c, t), 0, w_rows(c) * c->ld * sizeof(double), s));  // W_T = 0
      CUDA_OR_FAIL(c, cudaStreamWaitEvent(s, c->ev_head, cudaEventWaitExternal));   // lambda, pi, g uploaded
      after_kernel = false;
    } else {
      for (size_t j = 0; j < c->chunk_ev.size(); ++j)   // P_t's upload chunk (first stage of the chunk)
        if (c->chunk_hi[j] == t) {
          CUDA_OR_FAIL(c, cudaStreamWaitEvent(s, c->chunk_ev[j], cudaEventWaitExternal));
          after_kernel = false;
        }
      CUDA_OR_FAIL(c, mark(t, 0));
      CUDA_OR_FAIL(c, launch_contract(c, t, s, pdl && after_kernel && !sampled(t)));
      CUDA_OR_FAIL(c, mark(t, 1));
      after_kernel = true;
      ++n;
    }
    // bid curves need only W_t.  Stages are batched (fb_batch stages per launch, so each launch has enough
    // curves to fill the GPU) and every batch is a side branch of the graph on its own stream: it runs
    // concurrently with the remaining, latency-bound stages of the chain.
    const int bt = (t - 1) / c->fb_batch;                       // batch of stage t (stages bt*B+1 .. bt*B+B)
    if (c->fb_n > 0 && fb_mode == 0 && (t - 1) % c->fb_batch == 0) {   // t: the lowest stage of its batch, W ready
      const int t_hi = std::min(c->T, t + c->fb_batch - 1);
      const int64_t lo = c->fb_off[t], cnt = c->fb_off[t_hi + 1] - lo;
      if (cnt > 0) {
        cudaStream_t sb = c->side[bt % c->side.size()];
        side_used[bt % c->side.size()] = 1;
        CUDA_OR_FAIL(c, cudaEventRecord(c->fb_ev[t - 1], s));
        CUDA_OR_FAIL(c, cudaStreamWaitEvent(sb, c->fb_ev[t - 1], 0));
        CUDA_OR_FAIL(c, launch_bids(c, cnt, c->d_fb_req + 3 * lo, c->d_fb_slot + lo, c->fb_n, c->fb_cap, c->fb_nvert,
                                    c->fb_vert, c->fb_q, c->fb_price, sb));
        forked = true;
        after_kernel = false;
        ++n;
      }
    }
    CUDA_OR_FAIL(c, mark(t, 2));
    CUDA_OR_FAIL(c, launch_stencil(c, t, s, pdl && after_kernel && !sampled(t), false));
    CUDA_OR_FAIL(c, mark(t, 3));
    after_kernel = !sampled(t);
    ++n;
    if (c->comm) {  // V_t rows of every rank to every rank (in place, blocks of kmax rows): the next stage's
                    // contraction needs all of V_t; the policy stays local until the backward is done
      double* Vt = V_of(c, t);
      const size_t vcount = (size_t)c->kmax * c->ld;
      ncclResult_t r = ncclGroupStart();
      if (r == ncclSuccess) r = ncclAllGather(Vt + c->rank * vcount, Vt, vcount, ncclDouble, c->comm, s);
      const ncclResult_t r2 = ncclGroupEnd();
      if (r != ncclSuccess || r2 != ncclSuccess)
        return fail(c, ESDP_E_NCCL, "ncclAllGather(V_%d): %s", t, ncclGetErrorString(r != ncclSuccess ? r : r2));
      after_kernel = false;
    }
  }
  if (c->fb_n > 0 && fb_mode == 2) {
    CUDA_OR_FAIL(c, launch_bids(c, c->fb_n, c->d_fb_req, c->d_fb_slot, c->fb_n, c->fb_cap, c->fb_nvert, c->fb_vert,
                                c->fb_q, c->fb_price, s));
    ++n;
  } else if (c->fb_n > 0 && fb_mode == 1) {
    for (int t = 1; t <= T; t += c->fb_batch) {
      const int t_hi = std::min(c->T, t + c->fb_batch - 1);
      const int64_t lo = c->fb_off[t], cnt = c->fb_off[t_hi + 1] - lo;
      if (cnt <= 0) continue;
      const int bt = (t - 1) / c->fb_batch;
      cudaStream_t sb = c->side[bt % c->side.size()];
      side_used[bt % c->side.size()] = 1;
      CUDA_OR_FAIL(c, cudaEventRecord(c->fb_ev[t - 1], s));
      CUDA_OR_FAIL(c, cudaStreamWaitEvent(sb, c->fb_ev[t - 1], 0));
      CUDA_OR_FAIL(c, launch_bids(c, cnt, c->d_fb_req + 3 * lo, c->d_fb_slot + lo, c->fb_n, c->fb_cap, c->fb_nvert,
                                  c->fb_vert, c->fb_q, c->fb_price, sb));
      forked = true;
      ++n;
    }
  }
  if (c->comm) {   // every stage's policy rows to every rank, once, off the stage chain (one NCCL group)
    const size_t pcount = (size_t)c->kmax * c->S;
    ncclResult_t r = ncclGroupStart();
    for (int t = 1; t <= T && r == ncclSuccess; ++t) {
      int16_t* pt = c->d_pol + (size_t)(t - 1) * c->Kp * c->S;
      r = ncclAllGather(pt + c->rank * pcount, pt, pcount * sizeof(int16_t), ncclUint8, c->comm, s);
    }
    const ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
      return fail(c, ESDP_E_NCCL, "ncclAllGather(pol): %s", ncclGetErrorString(r != ncclSuccess ? r : r2));
    after_kernel = false;
  }
  CUDA_OR_FAIL(c, launch_objective(c, s, pdl && after_kernel));
  ++n;
  if (forked) {   // join the bid-curve branches
    for (size_t j = 0; j < c->side.size(); ++j) {
      if (!side_used[j]) continue;   // only streams that joined the capture
      CUDA_OR_FAIL(c, cudaEventRecord(c->join_ev[j], c->side[j]));
      CUDA_OR_FAIL(c, cudaStreamWaitEvent(s, c->join_ev[j], 0));
    }
  }
  CUDA_OR_FAIL(c, cudaGetLastError());
  c->launches = n;
  return ESDP_OK;
}

// One graph per input slot (the inputs' device pointers and upload events are baked into a graph).
esdp_status capture_graph(esdp_ctx* c) {
  for (int sl = 0; sl < 2; ++sl) {
    if (c->graphs[sl]) { cudaGraphExecDestroy(c->graphs[sl]); c->graphs[sl] = nullptr; }
    select_slot(c, sl);
    cudaGraph_t g = nullptr;
    CUDA_OR_FAIL(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    esdp_status est = enqueue_backward(c, c->stream);
    cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
    if (est != ESDP_OK) { if (g) cudaGraphDestroy(g); select_slot(c, c->active); return est; }
    if (ce != cudaSuccess) { select_slot(c, c->active); return fail(c, ESDP_E_CUDA, "graph capture: %s", cudaGetErrorString(ce)); }
    ce = cudaGraphInstantiate(&c->graphs[sl], g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) { select_slot(c, c->active); return fail(c, ESDP_E_CUDA, "graph instantiate: %s", cudaGetErrorString(ce)); }
  }
  select_slot(c, c->active);
  return ESDP_OK;
}

// Wait for stream s.  Multi-GPU contexts poll the communicator while they wait: an asynchronous NCCL
// error, or no completion within ESDP_NCCL_TIMEOUT_S seconds (default 120; a dead or hung peer), aborts
// the communicator and returns ESDP_E_NCCL instead of blocking forever.
template <class Query>
esdp_status wait_polled(esdp_ctx* c, Query query) {
  static const double tmo = [] { const char* e = getenv("ESDP_NCCL_TIMEOUT_S"); return e ? atof(e) : 120.0; }();
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = query();
    if (q == cudaSuccess) return ESDP_OK;
    if (q != cudaErrorNotReady) return fail(c, ESDP_E_CUDA, "wait: %s", cudaGetErrorString(q));
    ncclResult_t ae = ncclSuccess;
    const ncclResult_t qr = ncclCommGetAsyncError(c->comm, &ae);
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (qr != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress) || dt > tmo) {
      ncclCommAbort(c->comm);
      c->comm = nullptr;
      c->solved = false;
      return fail(c, ESDP_E_NCCL, "%s; communicator aborted",
                  dt > tmo ? "timeout waiting for the multi-GPU backward" : ncclGetErrorString(qr != ncclSuccess ? qr : ae));
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}
esdp_status wait_stream(esdp_ctx* c, cudaStream_t s) {
  if (!c->comm) {
    CUDA_OR_FAIL(c, cudaStreamSynchronize(s));
    return ESDP_OK;
  }
  return wait_polled(c, [&] { return cudaStreamQuery(s); });
}
esdp_status wait_event(esdp_ctx* c, cudaEvent_t e) {
  if (!c->comm) {
    CUDA_OR_FAIL(c, cudaEventSynchronize(e));
    return ESDP_OK;
  }
  return wait_polled(c, [&] { return cudaEventQuery(e); });
}

// DMMA bit-exactness probe (kernels.cuh dmma_probe_kernel), once per process and device: random, wide-
// range and cancelling operands; returns the number of outputs whose DMMA chain differs from the fma chain
// (-1 if the probe could not run).  ESDP_DMMA_PROBE_FAIL=1 in the environment reports a mismatch (tests).
int dmma_probe_mismatches() {
  static std::mutex mu;
  static std::unordered_map<int, int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return -1; }
  std::lock_guard<std::mutex> lk(mu);
  const char* f = getenv("ESDP_DMMA_PROBE_FAIL");   // read per call: tests force the fallback mid-process
  const int forced = (f && atoi(f)) ? 1 : 0;
  auto it = done.find(dev);
  if (it != done.end()) return it->second < 0 ? it->second : it->second + forced;
  constexpr int ntiles = 64, na = 8 * 4 * kProbeQ, nb = 4 * kProbeQ * 8;
  std::vector<double> A((size_t)ntiles * na), B((size_t)ntiles * nb);
  uint64_t st = 0x2511156290ull;
  auto rnd = [&] { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; };
  auto val = [&](uint64_t r) {
    const double m = 1.0 + (double)(r >> 12) * 0x1p-52;                 // [1, 2)
    const int e = (int)((r >> 4) & 63) - 32;                             // 2^-32 .. 2^31
    return ((r & 1) ? -1.0 : 1.0) * std::ldexp(m, e);
  };
  for (int t = 0; t < ntiles; ++t) {
    for (int j = 0; j < na; ++j) A[(size_t)t * na + j] = val(rnd());
    for (int j = 0; j < nb; ++j) B[(size_t)t * nb + j] = val(rnd());
    if (t % 2) {   // cancelling pairs: the product of k' = 2m+1 undoes that of k' = 2m (exactly or nearly)
      for (int g = 0; g < 8; ++g)
        for (int k = 0; k + 1 < 4 * kProbeQ; k += 2)
          A[(size_t)t * na + g * 4 * kProbeQ + k + 1] = -A[(size_t)t * na + g * 4 * kProbeQ + k] * (1.0 + ((t / 2) % 3) * 0x1p-40);
      for (int k = 0; k + 1 < 4 * kProbeQ; k += 2)
        for (int c = 0; c < 8; ++c) B[(size_t)t * nb + (k + 1) * 8 + c] = B[(size_t)t * nb + k * 8 + c];
    }
  }
  double *dA = nullptr, *dB = nullptr;
  unsigned* dm = nullptr;
  unsigned bad = 0;
  int res = -1;
  if (cudaMalloc(&dA, A.size() * 8) == cudaSuccess && cudaMalloc(&dB, B.size() * 8) == cudaSuccess &&
      cudaMalloc(&dm, sizeof(unsigned)) == cudaSuccess &&
      cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess &&
      cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess &&
      cudaMemset(dm, 0, sizeof(unsigned)) == cudaSuccess) {
    dmma_probe_kernel<<<ntiles / 4, 128>>>(dA, dB, ntiles, dm);
    if (cudaMemcpy(&bad, dm, sizeof(unsigned), cudaMemcpyDeviceToHost) == cudaSuccess) res = (int)bad;
  }
  cudaFree(dA); cudaFree(dB); cudaFree(dm);
  cudaGetLastError();
  done[dev] = res;
  return res < 0 ? res : res + forced;
}

}  // namespace

extern "C" {

static esdp_status create_impl(const esdp_problem* pr, int32_t world, int32_t rank, const void* nccl_id, esdp_ctx** out,
                               bool tables_only = false);

esdp_status esdp_create(const esdp_problem* pr, esdp_ctx** out) { return create_impl(pr, 1, 0, nullptr, out); }

esdp_status esdp_partition(int32_t K, int32_t world, int32_t rank, int32_t* k_lo, int32_t* k_cnt, int32_t* kmax) {
  if (K < 1 || world < 1 || rank < 0 || rank >= world) return ESDP_E_CONFIG;
  const int32_t m = (K + world - 1) / world;
  const int32_t lo = std::min(K, rank * m), hi = std::min(K, (rank + 1) * m);
  if (k_lo) *k_lo = lo;
  if (k_cnt) *k_cnt = hi - lo;
  if (kmax) *kmax = m;
  return ESDP_OK;
}

esdp_status esdp_dist_info(const esdp_ctx* c, int32_t* world, int32_t* rank, int32_t* nccl_nranks) {
  if (!c) return ESDP_E_STATE;
  if (world) *world = c->world;
  if (rank) *rank = c->rank;
  if (nccl_nranks) {
    int n = 0;
    if (c->comm && ncclCommCount(c->comm, &n) != ncclSuccess) n = -1;
    *nccl_nranks = n;
  }
  return ESDP_OK;
}

esdp_status esdp_nccl_unique_id(void* id128) {
  if (!id128) return ESDP_E_CONFIG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return fail(nullptr, ESDP_E_NCCL, "ncclGetUniqueId failed");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id128, &id, sizeof(id));
  return ESDP_OK;
}

esdp_status esdp_create_dist(const esdp_problem* pr, int32_t world, int32_t rank, const void* nccl_id, esdp_ctx** out) {
  if (world < 1 || rank < 0 || rank >= world || !nccl_id) return fail(nullptr, ESDP_E_CONFIG, "bad world/rank/nccl id");
  return create_impl(pr, world, rank, nccl_id, out);
}

// tables_only: an instance of a batch (esdp_create_batch) -- parameters, action grid and per-action
// tables only; the shared inputs, the value buffers and the graph belong to the batch.
static esdp_status create_impl(const esdp_problem* pr, int32_t world, int32_t rank, const void* nccl_id, esdp_ctx** out,
                               bool tables_only) {
  g_create_error.clear();
  if (!pr || !out) return fail(nullptr, ESDP_E_CONFIG, "null argument");
  *out = nullptr;
  if (pr->T < 1 || pr->K < 1) return fail(nullptr, ESDP_E_CONFIG, "T and K must be >= 1");
  if (pr->K > 32767) return fail(nullptr, ESDP_E_CONFIG, "K exceeds 32767 (16-bit sampler guide entries)");
  if (!(std::isfinite(pr->pbar) && pr->pbar > 0)) return fail(nullptr, ESDP_E_CONFIG, "pbar must be > 0");
  if (!(std::isfinite(pr->sbar) && pr->sbar > 0)) return fail(nullptr, ESDP_E_CONFIG, "sbar must be > 0");
  if (!(std::isfinite(pr->delta) && pr->delta > 0)) return fail(nullptr, ESDP_E_CONFIG, "delta must be > 0");
  if (!(pr->eta_c > 0 && pr->eta_c <= 1) || !(pr->eta_d > 0 && pr->eta_d <= 1))
    return fail(nullptr, ESDP_E_CONFIG, "efficiencies must lie in (0, 1]");
  if (!(std::isfinite(pr->s0) && pr->s0 >= 0 && pr->s0 <= pr->sbar)) return fail(nullptr, ESDP_E_CONFIG, "s0 must lie in [0, sbar]");
  const double ns = pr->sbar / pr->delta;
  const double rs = std::nearbyint(ns);
  if (!(std::fabs(ns - rs) <= kGridTol * (ns > 1.0 ? ns : 1.0)) || rs < 1.0 || rs > 1e8)
    return fail(nullptr, ESDP_E_CONFIG, "sbar/delta = %.17g is not a positive integer (P:180)", ns);
  if (pr->payoff_kind < 0 || pr->payoff_kind > 2) return fail(nullptr, ESDP_E_CONFIG, "unknown payoff kind");
  if (pr->payoff_kind != ESDP_PAYOFF_LINEAR && !pr->g) return fail(nullptr, ESDP_E_CONFIG, "payoff needs g");
  if (!pr->lambda || !pr->pi) return fail(nullptr, ESDP_E_CONFIG, "lambda and pi are required");
  if (pr->flags & ~(uint32_t)ESDP_FLAGS_ALL) return fail(nullptr, ESDP_E_CONFIG, "unknown flag bits 0x%x", pr->flags & ~(uint32_t)ESDP_FLAGS_ALL);

  esdp_ctx* c = new esdp_ctx();
  c->T = pr->T; c->K = pr->K; c->S = (int)rs + 1; c->ld = (c->S + 3) & ~3;
  c->world = world; c->rank = rank;
  esdp_partition(c->K, world, rank, &c->k_lo, &c->k_cnt, &c->kmax);
  c->Kp = world * c->kmax;   // == K on one GPU
  c->pbar = pr->pbar; c->sbar = pr->sbar; c->s0 = pr->s0; c->eta_c = pr->eta_c; c->eta_d = pr->eta_d;
  c->delta = pr->delta; c->kind = pr->payoff_kind; c->rank1 = pr->P == nullptr; c->flags = pr->flags;
  c->pdl = (pr->flags & ESDP_NO_PDL) == 0;   // late-trigger PDL: dependents launch as the primary drains
  if (pr->A == 0) {
    paper_grid(pr->pbar, pr->eta_c, pr->eta_d, pr->delta, c->act);
    if ((long long)c->act.size() > kMaxA) { delete c; return fail(nullptr, ESDP_E_CONFIG, "A exceeds %d", kMaxA); }
    for (size_t a = 1; a < c->act.size(); ++a)
      if (!(c->act[a] > c->act[a - 1])) { delete c; return fail(nullptr, ESDP_E_CONFIG, "Eq. 10 grid has duplicate actions"); }
  } else {
    if (pr->A < 0 || pr->A > kMaxA || !pr->actions) { delete c; return fail(nullptr, ESDP_E_CONFIG, "bad action list"); }
    int zeros = 0;
    for (int a = 0; a < pr->A; ++a) {
      const double p = pr->actions[a];
      if (!std::isfinite(p) || std::fabs(p) > pr->pbar) { delete c; return fail(nullptr, ESDP_E_CONFIG, "action %d outside [-pbar, pbar]", a); }
      if (p == 0.0) ++zeros;
      if (a > 0 && !(p > pr->actions[a - 1])) { delete c; return fail(nullptr, ESDP_E_CONFIG, "actions not strictly ascending"); }
    }
    if (zeros != 1) { delete c; return fail(nullptr, ESDP_E_CONFIG, "the action list must contain 0 exactly once"); }
    c->act.assign(pr->actions, pr->actions + pr->A);
  }
  c->A = (int)c->act.size();
  if (!tables_only) {
    esdp_status st = validate_data(c, pr->lambda, pr->P, pr->pi, pr->g);
    if (st != ESDP_OK) { g_create_error = c->err; delete c; return st; }
  } else if (c->kind == ESDP_PAYOFF_LINEAR_MINUS_G) {
    for (int a = 0; a < c->A; ++a)
      if (!std::isfinite(pr->g[a])) { fail(c, ESDP_E_DATA, "g[%d] is not finite", a); g_create_error = c->err; delete c; return ESDP_E_DATA; }
  }
  build_tables(c, pr->g);

  auto bail = [&](esdp_status st) { g_create_error = c->err; free_all(c); delete c; return st; };
#define TRY(x) do { esdp_status st_ = (x); if (st_ != ESDP_OK) return bail(st_); } while (0)
  // the dependent stage chain runs at the highest stream priority, the bid-curve side branches at the
  // lowest (graph nodes keep the priority of the stream they were captured on)
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  c->prio_lo = prio_lo;
  if (cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess) {
    cudaGetLastError();
    fail(c, ESDP_E_CUDA, "cannot create a CUDA stream (no usable GPU?)");
    return bail(ESDP_E_CUDA);
  }
  const size_t T = c->T, K = c->K, S = c->S, A = c->A;
  {   // guide geometry (kernels.cuh cdf_kernel): up to 2^g_max >= kGuideRatio K buckets per row; the allocation is
      // capped at max(256 MB, the size of P) and always holds 2^6 buckets for every possible row
    c->g_max = guide_gmax((int)K);
    const size_t rows = c->rank1 ? T : (T > 1 ? (T - 1) * K : 1);
    const char* eb = getenv("ESDP_GUIDE_BUDGET_MB");   // measurement
    const size_t mb = (eb && atoi(eb) > 0) ? (size_t)atoi(eb) : 256u;
    const size_t budget = std::max<size_t>(mb << 20, (c->rank1 ? 0 : rows * K * 8)) / sizeof(uint64_t);
    c->guide_cap = std::max(rows << kGuideMinG, std::min(rows << c->g_max, budget));
    c->g_r1 = guide_g_for(T, c->guide_cap, c->g_max);
  }
  if (!tables_only) {   // two input slots (double-buffered loads); the aliases follow select_slot
    for (InputSlot& x : c->slot) {
      TRY(dev_alloc(c, &x.lambda, T * K));
      TRY(dev_alloc(c, &x.P, c->rank1 ? 1 : (T - 1) * K * K));
      TRY(dev_alloc(c, &x.pi, c->rank1 ? T * K : K));
      TRY(dev_alloc(c, &x.cdf, c->rank1 ? T * K : (T - 1) * K * K));
      TRY(dev_alloc(c, &x.cdf1, K));
      TRY(dev_alloc(c, &x.guide, c->guide_cap));
      TRY(dev_alloc(c, &x.guide1, (size_t)1 << c->g_max));
      if (!c->rank1 && T > 1) {
        TRY(dev_alloc(c, &x.tab, T - 1));
        TRY(dev_alloc(c, &x.src, T - 1));
      }
      x.gbits = c->rank1 ? c->g_r1 : c->g_max;
      TRY(dev_alloc(c, &x.g, c->kind == ESDP_PAYOFF_TABLE ? T * K * A : A));
      TRY(dev_alloc(c, &x.gfit, 6));
      cudaMemset(x.g, 0, (c->kind == ESDP_PAYOFF_TABLE ? T * K * A : A) * sizeof(double));
      cudaMemset(x.gfit, 0, 6 * sizeof(double));
    }
    select_slot(c, 0);
  } else {
    TRY(dev_alloc(c, &c->d_g, c->kind == ESDP_PAYOFF_TABLE ? T * K * A : A));
  }
  TRY(dev_alloc(c, &c->d_act, A));
  TRY(dev_alloc(c, &c->d_w, A));
  TRY(dev_alloc(c, &c->d_omw, A));
  TRY(dev_alloc(c, &c->d_off, A));
  TRY(dev_alloc(c, &c->d_segs, c->segs.size()));
  const size_t LD = c->ld;
  const size_t KP = c->Kp;
  if (tables_only) {   // per-action tables and the stencil plan; the batch owns everything else
    TRY(dev_alloc(c, &c->d_singles, c->singles.size()));
    TRY(dev_alloc(c, &c->d_live, c->live_list.size()));
    TRY(dev_alloc(c, &c->d_gfit, 6));
    fit_g(c, pr->g, c->gfit);
    if ((!c->singles.empty() && cudaMemcpy(c->d_singles, c->singles.data(), c->singles.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) ||
        cudaMemcpy(c->d_live, c->live_list.data(), c->live_list.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->d_act, c->act.data(), A * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->d_w, c->w.data(), A * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->d_omw, c->omw.data(), A * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->d_off, c->off.data(), A * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->d_segs, c->segs.data(), c->segs.size() * sizeof(Seg), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->d_gfit, c->gfit, sizeof c->gfit, cudaMemcpyHostToDevice) != cudaSuccess ||
        (c->kind == ESDP_PAYOFF_LINEAR_MINUS_G && cudaMemcpy(c->d_g, pr->g, A * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) ||
        (c->kind == ESDP_PAYOFF_LINEAR && cudaMemset(c->d_g, 0, A * sizeof(double)) != cudaSuccess)) {
      fail(c, ESDP_E_CUDA, "upload of the action tables failed");
      return bail(ESDP_E_CUDA);
    }
    c->stencil_smem = stencil_smem_bytes(c->A, c->o_max - c->o_min);
    if (c->use_window) {
      plan_window(c, 1 << 30);   // batch: throughput regime
      if (c->window_smem > 200 * 1024) c->use_window = 0;
    }
    if (c->stencil_smem > 227 * 1024) { fail(c, ESDP_E_CONFIG, "action span too wide for shared memory"); return bail(ESDP_E_CONFIG); }
    *out = c;
    return ESDP_OK;
  }
  TRY(dev_alloc(c, &c->d_V, keep(c) ? T * KP * LD : 2 * KP * LD));
  TRY(dev_alloc(c, &c->d_W, keep(c) ? T * w_rows(c) * LD : w_rows(c) * LD));
  // padding columns are never read as values; zero them once so no stale bits are staged
  cudaMemset(c->d_V, 0, (keep(c) ? T * KP * LD : 2 * KP * LD) * sizeof(double));
  cudaMemset(c->d_W, 0, (keep(c) ? T * w_rows(c) * LD : w_rows(c) * LD) * sizeof(double));
  TRY(dev_alloc(c, &c->d_pol, T * KP * S));
  if (nccl_id) {   // esdp_create_dist: NCCL communicator (also for world == 1: the all-gather is a copy)
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t nr = ncclCommInitRank(&c->comm, world, id, rank);
    if (nr != ncclSuccess) { fail(c, ESDP_E_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(nr)); c->comm = nullptr; return bail(ESDP_E_NCCL); }
  }
  TRY(dev_alloc(c, &c->d_J, 4));
  TRY(dev_alloc(c, &c->d_singles, c->singles.size()));
  TRY(dev_alloc(c, &c->d_live, c->live_list.size()));
  if (!c->singles.empty() && cudaMemcpy(c->d_singles, c->singles.data(), c->singles.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) { fail(c, ESDP_E_CUDA, "upload singles"); return bail(ESDP_E_CUDA); }
  if (cudaMemcpy(c->d_live, c->live_list.data(), c->live_list.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) { fail(c, ESDP_E_CUDA, "upload live list"); return bail(ESDP_E_CUDA); }
  TRY(dev_alloc(c, &c->d_red, 4));
  if (cudaMemcpy(c->d_act, c->act.data(), A * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(c->d_w, c->w.data(), A * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(c->d_omw, c->omw.data(), A * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(c->d_off, c->off.data(), A * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(c->d_segs, c->segs.data(), c->segs.size() * sizeof(Seg), cudaMemcpyHostToDevice) != cudaSuccess) {
    fail(c, ESDP_E_CUDA, "upload of the action tables failed");
    return bail(ESDP_E_CUDA);
  }
  TRY(dev_alloc(c, &c->d_F, A));
  if (cudaMemcpy(c->d_F, c->F.data(), A * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) { fail(c, ESDP_E_CUDA, "upload F"); return bail(ESDP_E_CUDA); }
  if (cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) != cudaSuccess) {
    fail(c, ESDP_E_CUDA, "copy stream");
    return bail(ESDP_E_CUDA);
  }
  {  // P chunks: ~8 stage ranges, highest stages first (the order the backward consumes them)
    const int nst = c->rank1 ? 0 : T - 1;
    const int nch = std::min(8, nst);
    for (int j = 0; j < nch; ++j) {
      c->chunk_hi.push_back(nst - (int)((long long)nst * j / nch));
      c->chunk_lo.push_back(nst - (int)((long long)nst * (j + 1) / nch) + 1);
    }
    for (InputSlot& x : c->slot) {
      bool ok = cudaEventCreateWithFlags(&x.ev_head, cudaEventDisableTiming) == cudaSuccess &&
                cudaEventCreateWithFlags(&x.ev_tables, cudaEventDisableTiming) == cudaSuccess &&
                cudaEventCreateWithFlags(&x.use_ev, cudaEventDisableTiming) == cudaSuccess &&
                cudaEventCreateWithFlags(&x.stage_ev, cudaEventDisableTiming) == cudaSuccess &&
                cudaMallocHost(&x.stage_h, sizeof(int) * 2 * (size_t)std::max(1, nst)) == cudaSuccess &&
                cudaMallocHost(&x.gfit_stage, sizeof(double) * 6) == cudaSuccess;
      x.chunk_ev.assign(nch, nullptr);
      for (int j = 0; j < nch && ok; ++j) ok = cudaEventCreateWithFlags(&x.chunk_ev[j], cudaEventDisableTiming) == cudaSuccess;
      if (!ok) { fail(c, ESDP_E_CUDA, "input events"); return bail(ESDP_E_CUDA); }
    }
    select_slot(c, 0);
  }
  TRY(upload(c, 0, 0, pr->lambda, pr->P, pr->pi, pr->g));
  if (cudaStreamSynchronize(c->copy) != cudaSuccess) { fail(c, ESDP_E_CUDA, "initial upload"); return bail(ESDP_E_CUDA); }
  c->stencil_smem = stencil_smem_bytes(c->A, c->o_max - c->o_min);
  if (c->use_window) {
    plan_window(c, (int64_t)c->k_cnt * ((c->S + kWinThreads - 1) / kWinThreads));
    if (c->window_smem > 200 * 1024) c->use_window = 0;
    else if (c->window_smem > 48 * 1024 &&
             cudaFuncSetAttribute(window_kernel_of(c->win_opt, c->win_levels), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)c->window_smem) != cudaSuccess)
      c->use_window = 0;
  }
  if (c->stencil_smem > 48 * 1024) {
    if (c->stencil_smem > 227 * 1024) { fail(c, ESDP_E_CONFIG, "action span too wide for shared memory"); return bail(ESDP_E_CONFIG); }
    if (cudaFuncSetAttribute(stencil_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->stencil_smem) != cudaSuccess) {
      fail(c, ESDP_E_CUDA, "cannot opt in to %zu bytes of shared memory", c->stencil_smem);
      return bail(ESDP_E_CUDA);
    }
  }
  if (contract_smem_bytes(K) > 227 * 1024) { fail(c, ESDP_E_CONFIG, "K too large for the contraction tile"); return bail(ESDP_E_CONFIG); }
  if (!(c->flags & ESDP_NO_DMMA) && dmma_probe_mismatches() != 0) {   // guard: DFMA unless DMMA == fma chain
    c->flags |= ESDP_NO_DMMA;
    c->dmma_probe_failed = 1;
  }
  {
    const size_t sm2 = K > 128 ? contract_dmma2_smem(K, kDRbig, kDCbig) : contract_dmma2_smem(K);
    c->dmma2 = sm2 <= 200 * 1024;
    if (c->dmma2 && sm2 > 48 * 1024 &&
        (K > 128 ? cudaFuncSetAttribute(contract_dmma2_kernel<kDRbig, kDCbig>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2)
                 : cudaFuncSetAttribute(contract_dmma2_kernel<kDR, kDC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2)) != cudaSuccess)
      c->dmma2 = 0;
  }
  if (contract_smem_bytes(K) > 48 * 1024)
    cudaFuncSetAttribute(contract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)contract_smem_bytes(K));
  if (2 * sizeof(double) * K > 48 * 1024)
    cudaFuncSetAttribute(objective_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * sizeof(double) * K));
  if (c->flags & ESDP_PROFILE) {
    c->prof_stride = std::max(1, c->T / 16);
    c->ev.resize((size_t)c->T * 4);
    for (auto& e : c->ev)
      if (cudaEventCreate(&e) != cudaSuccess) { fail(c, ESDP_E_CUDA, "cudaEventCreate failed"); return bail(ESDP_E_CUDA); }
  }
  // capture the whole backward pass once; replay it for every solve
  {   // ~8 bid-curve batches per backward (ESDP_FB_BATCHES=n overrides: measurement)
    const char* e = getenv("ESDP_FB_BATCHES");
    const int nb = (e && atoi(e) > 0) ? atoi(e) : 8;
    c->fb_batch = std::max(1, (c->T + nb - 1) / nb);
  }
  c->side.assign(4, nullptr);
  c->join_ev.assign(c->side.size(), nullptr);
  for (size_t j = 0; j < c->side.size(); ++j)
    if (cudaStreamCreateWithPriority(&c->side[j], cudaStreamNonBlocking, c->prio_lo) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->join_ev[j], cudaEventDisableTiming) != cudaSuccess) {
      fail(c, ESDP_E_CUDA, "side stream");
      return bail(ESDP_E_CUDA);
    }
  c->fb_ev.resize((size_t)c->T + 1);
  for (auto& ev : c->fb_ev)
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) { fail(c, ESDP_E_CUDA, "event"); return bail(ESDP_E_CUDA); }
  TRY(capture_graph(c));
#undef TRY
  *out = c;
  return ESDP_OK;
}

esdp_status esdp_dims(const esdp_ctx* c, int32_t* T, int32_t* S, int32_t* A, int32_t* K) {
  if (!c) return ESDP_E_STATE;
  if (T) *T = c->T;
  if (S) *S = c->S;
  if (A) *A = c->A;
  if (K) *K = c->K;
  return ESDP_OK;
}

esdp_status esdp_actions(const esdp_ctx* c, double* actions) {
  if (!c || !actions) return ESDP_E_STATE;
  std::memcpy(actions, c->act.data(), c->act.size() * sizeof(double));
  return ESDP_OK;
}

static esdp_status load_impl(esdp_ctx* c, const double* lambda, const double* P, const double* pi, const double* g) {
  // target: the slot no launched solve reads (or the pending one, replaced); NULL arrays keep the data of
  // the newest inputs (src)
  const int src = c->pending >= 0 ? c->pending : c->active;
  const int dst = c->pending >= 0 ? c->pending : 1 - c->active;
  InputSlot& d = c->slot[dst];
  const InputSlot& o = c->slot[src];
  // No host wait for the last solve that read dst: upload() orders dst's copies after it on the device
  // (cudaStreamWaitEvent on use_ev), and re-recording dst's upload events does not affect that solve's
  // graph, whose event-wait nodes resolved to the earlier records when it was launched.  (A host
  // synchronize here held a pipelined loop's host thread for a whole solve: measured 2.1 ms of host time
  // per cfg2 step, the e2e loop's bound.)
  // validate what is given against the current arrays' shapes
  std::vector<double> lam_h, P_h, pi_h, g_h;
  const size_t TK = (size_t)c->T * c->K;
  const bool read_back = !lambda || (!c->rank1 && !P && c->T > 1) || !pi || (!g && c->kind != ESDP_PAYOFF_LINEAR);
  if (read_back) CUDA_OR_FAIL(c, cudaStreamSynchronize(c->copy));   // kept arrays are validated from the device copy
  if (!lambda) { lam_h.resize(TK); CUDA_OR_FAIL(c, cudaMemcpy(lam_h.data(), o.lambda, TK * 8, cudaMemcpyDeviceToHost)); }
  if (!c->rank1 && !P && c->T > 1) { P_h.resize((size_t)(c->T - 1) * c->K * c->K); CUDA_OR_FAIL(c, cudaMemcpy(P_h.data(), o.P, P_h.size() * 8, cudaMemcpyDeviceToHost)); }
  if (!pi) { pi_h.resize(c->rank1 ? TK : c->K); CUDA_OR_FAIL(c, cudaMemcpy(pi_h.data(), o.pi, pi_h.size() * 8, cudaMemcpyDeviceToHost)); }
  if (!g && c->kind != ESDP_PAYOFF_LINEAR) { g_h.resize(c->kind == ESDP_PAYOFF_TABLE ? TK * c->A : c->A); CUDA_OR_FAIL(c, cudaMemcpy(g_h.data(), o.g, g_h.size() * 8, cudaMemcpyDeviceToHost)); }
  esdp_status st = validate_data(c, lambda ? lambda : lam_h.data(), P ? P : P_h.data(), pi ? pi : pi_h.data(),
                                 g ? g : g_h.data());
  if (st != ESDP_OK) return st;
  st = upload(c, dst, src, lambda, P, pi, g);
  if (st != ESDP_OK) return st;
  c->pending = dst;
  return ESDP_OK;
}

esdp_status esdp_load(esdp_ctx* c, const double* lambda, const double* P, const double* pi, const double* g) {
  if (!c) return ESDP_E_STATE;
  esdp_status st = load_impl(c, lambda, P, pi, g);
  if (st != ESDP_OK) return st;
  CUDA_OR_FAIL(c, cudaStreamSynchronize(c->copy));
  return ESDP_OK;
}

esdp_status esdp_load_async(esdp_ctx* c, const double* lambda, const double* P, const double* pi, const double* g) {
  if (!c) return ESDP_E_STATE;
  return load_impl(c, lambda, P, pi, g);
}

esdp_status esdp_backward_async(esdp_ctx* c, void* stream) {
  if (!c) return ESDP_E_STATE;
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  if (c->pending >= 0) {   // the latest load becomes the inputs of this (and later) solves
    c->active = c->pending;
    c->pending = -1;
  }
  select_slot(c, c->active);
  CUDA_OR_FAIL(c, cudaGraphLaunch(c->graphs[c->active], s));
  { const esdp_status mu = mark_use(c, s); if (mu != ESDP_OK) return mu; }
  c->solved = true;
  return ESDP_OK;
}

esdp_status esdp_objective(esdp_ctx* c, double* J) {
  if (!c || !c->solved) return c ? fail(c, ESDP_E_STATE, "no backward pass has run") : ESDP_E_STATE;
  { const esdp_status w = wait_event(c, c->slot[c->active].use_ev); if (w != ESDP_OK) return w; }   // the last use, any stream
  CUDA_OR_FAIL(c, cudaMemcpy(J, c->d_J, sizeof(double), cudaMemcpyDeviceToHost));
  return ESDP_OK;
}

esdp_status esdp_objective_async(esdp_ctx* c, double* J_host, void* stream) {
  if (!c || !J_host) return ESDP_E_STATE;
  if (!c->solved) return fail(c, ESDP_E_STATE, "no backward pass has run");
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  CUDA_OR_FAIL(c, cudaMemcpyAsync(J_host, c->d_J, sizeof(double), cudaMemcpyDeviceToHost, s));
  return ESDP_OK;
}

esdp_status esdp_backward(esdp_ctx* c, void* stream, double* J) {
  if (!c) return ESDP_E_STATE;
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  esdp_status st = esdp_backward_async(c, s);
  if (st != ESDP_OK) return st;
  st = wait_stream(c, s);
  if (st != ESDP_OK) return st;
  if (J) CUDA_OR_FAIL(c, cudaMemcpy(J, c->d_J, sizeof(double), cudaMemcpyDeviceToHost));
  return ESDP_OK;
}

esdp_status esdp_values(const esdp_ctx* cc, int32_t t, double* V, double* W) {
  esdp_ctx* c = const_cast<esdp_ctx*>(cc);
  if (!c) return ESDP_E_STATE;
  if (!c->solved) return fail(c, ESDP_E_STATE, "no backward pass has run");
  if (t < 1 || t > c->T) return fail(c, ESDP_E_STATE, "stage %d out of range", t);
  if (!keep(c) && (t != 1 || W)) return fail(c, ESDP_E_STATE, "only V_1 is kept without ESDP_KEEP_VALUES");
  if (W && c->world > 1 && !c->rank1) return fail(c, ESDP_E_STATE, "W_t rows live on their owning ranks (multi-GPU)");
  const size_t rowb = c->S * sizeof(double), ldb = c->ld * sizeof(double);
  if (V) CUDA_OR_FAIL(c, cudaMemcpy2D(V, rowb, V_of(c, t), ldb, rowb, c->K, cudaMemcpyDeviceToHost));
  if (W) {
    if (c->rank1) {
      for (int k = 0; k < c->K; ++k)
        CUDA_OR_FAIL(c, cudaMemcpy(W + (size_t)k * c->S, W_of(c, t), rowb, cudaMemcpyDeviceToHost));
    } else {
      CUDA_OR_FAIL(c, cudaMemcpy2D(W, rowb, W_of(c, t), ldb, rowb, c->K, cudaMemcpyDeviceToHost));
    }
  }
  return ESDP_OK;
}

esdp_status esdp_policy(const esdp_ctx* cc, int32_t t, int16_t* pol) {
  esdp_ctx* c = const_cast<esdp_ctx*>(cc);
  if (!c) return ESDP_E_STATE;
  if (!c->solved) return fail(c, ESDP_E_STATE, "no backward pass has run");
  if (t < 1 || t > c->T) return fail(c, ESDP_E_STATE, "stage %d out of range", t);
  const size_t KS = (size_t)c->K * c->S;
  CUDA_OR_FAIL(c, cudaMemcpy(pol, c->d_pol + (size_t)(t - 1) * c->Kp * c->S, KS * sizeof(int16_t), cudaMemcpyDeviceToHost));
  return ESDP_OK;
}

esdp_status esdp_bidcurves_dev(esdp_ctx* c, int64_t n, const int32_t* req_dev, int32_t cap, int32_t* nvert_dev,
                               int16_t* vert_dev, double* q_dev, double* price_dev, void* stream) {
  if (!c) return ESDP_E_STATE;
  if (!c->solved) return fail(c, ESDP_E_STATE, "no backward pass has run");
  if (!keep(c)) return fail(c, ESDP_E_STATE, "bid curves need ESDP_KEEP_VALUES");
  if (c->kind == ESDP_PAYOFF_TABLE) return fail(c, ESDP_E_STATE, "bid curves are not defined for TABLE payoffs (R13)");
  if (cap < c->A) return fail(c, ESDP_E_STATE, "cap %d < A %d", cap, c->A);
  if (n <= 0) return ESDP_OK;
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  CUDA_OR_FAIL(c, launch_bids(c, n, req_dev, nullptr, n, cap, nvert_dev, vert_dev, q_dev, price_dev, s));
  return mark_use(c, s);
}

esdp_status esdp_set_bid_requests(esdp_ctx* c, int64_t n, const int32_t* req, int32_t cap, int32_t* nvert_dev,
                                  int16_t* vert_dev, double* q_dev, double* price_dev) {
  if (!c) return ESDP_E_STATE;
  if (n > 0) {
    if (!keep(c)) return fail(c, ESDP_E_STATE, "fused bid curves need ESDP_KEEP_VALUES");
    if (c->kind == ESDP_PAYOFF_TABLE) return fail(c, ESDP_E_STATE, "bid curves are not defined for TABLE payoffs (R13)");
    if (cap < c->A || !req || !nvert_dev || !vert_dev || !price_dev) return fail(c, ESDP_E_STATE, "bad bid request arguments");
    for (int64_t r = 0; r < n; ++r) {
      const int t = req[3 * r], i = req[3 * r + 1], k = req[3 * r + 2];
      if (t < 1 || t > c->T || i < 0 || i >= c->S || k < 0 || k >= c->K || (!c->rank1 && (k < c->k_lo || k >= c->k_lo + c->k_cnt)))
        return fail(c, ESDP_E_STATE, "request %lld (t=%d, i=%d, k=%d) out of range for this rank", (long long)r, t, i, k);
    }
  }
  // stable counting sort by stage
  std::vector<int64_t> off((size_t)c->T + 2, 0);
  for (int64_t r = 0; r < n; ++r) off[req[3 * r] + 1]++;
  for (int t = 1; t <= c->T + 1; ++t) off[t] += off[t - 1];
  std::vector<int32_t> sreq((size_t)std::max<int64_t>(n, 1) * 3), slot((size_t)std::max<int64_t>(n, 1));
  std::vector<int64_t> pos(off.begin(), off.end());
  for (int64_t r = 0; r < n; ++r) {
    const int64_t p = pos[req[3 * r]]++;
    sreq[3 * p] = req[3 * r]; sreq[3 * p + 1] = req[3 * r + 1]; sreq[3 * p + 2] = req[3 * r + 2];
    slot[p] = (int32_t)r;
  }
  cudaFree(c->d_fb_req); cudaFree(c->d_fb_slot);
  c->d_fb_req = nullptr; c->d_fb_slot = nullptr;
  c->fb_n = 0;
  if (n > 0) {
    if (dev_alloc(c, &c->d_fb_req, 3 * n) || dev_alloc(c, &c->d_fb_slot, n)) return ESDP_E_NOMEM;
    CUDA_OR_FAIL(c, cudaMemcpy(c->d_fb_req, sreq.data(), 3 * n * sizeof(int32_t), cudaMemcpyHostToDevice));
    CUDA_OR_FAIL(c, cudaMemcpy(c->d_fb_slot, slot.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice));
    // off[t] is the first request of stage t (1-based stages)
    c->fb_off = off;   // stage t's requests are [off[t], off[t+1])
  }
  c->fb_n = n;
  c->fb_cap = cap;
  c->fb_nvert = nvert_dev; c->fb_vert = vert_dev; c->fb_q = q_dev; c->fb_price = price_dev;
  return capture_graph(c);
}

esdp_status esdp_bidcurves(esdp_ctx* c, int64_t n, const int32_t* req, int32_t cap, int32_t* nvert, int16_t* vert,
                           double* q, double* price) {
  if (!c) return ESDP_E_STATE;
  if (n <= 0) return ESDP_OK;
  for (int64_t r = 0; r < n; ++r) {
    const int t = req[3 * r], i = req[3 * r + 1], k = req[3 * r + 2];
    if (t < 1 || t > c->T || i < 0 || i >= c->S || k < 0 || k >= c->K)
      return fail(c, ESDP_E_STATE, "request %lld (t=%d, i=%d, k=%d) out of range", (long long)r, t, i, k);
    if (!c->rank1 && (k < c->k_lo || k >= c->k_lo + c->k_cnt))
      return fail(c, ESDP_E_STATE, "request %lld: price state %d is owned by another rank", (long long)r, k);
  }
  if (n > c->req_cap || (int64_t)cap * n > c->out_cap) {
    cudaFree(c->d_req); cudaFree(c->d_nv); cudaFree(c->d_vert); cudaFree(c->d_q); cudaFree(c->d_price);
    c->d_req = nullptr; c->d_nv = nullptr; c->d_vert = nullptr; c->d_q = nullptr; c->d_price = nullptr;
    c->req_cap = c->out_cap = 0;
    if (dev_alloc(c, &c->d_req, 3 * n) || dev_alloc(c, &c->d_nv, n) || dev_alloc(c, &c->d_vert, (size_t)cap * n) ||
        dev_alloc(c, &c->d_q, (size_t)cap * n) || dev_alloc(c, &c->d_price, (size_t)cap * n))
      return ESDP_E_NOMEM;
    c->req_cap = n;
    c->out_cap = (int64_t)cap * n;
  }
  CUDA_OR_FAIL(c, cudaMemcpyAsync(c->d_req, req, 3 * n * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
  esdp_status st = esdp_bidcurves_dev(c, n, c->d_req, cap, c->d_nv, c->d_vert, c->d_q, c->d_price, c->stream);
  if (st != ESDP_OK) return st;
  CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  CUDA_OR_FAIL(c, cudaMemcpy(nvert, c->d_nv, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
  // device layout is vertex-major [cap][n]; the host API returns curve-major [n][cap]
  std::vector<int16_t> hv((size_t)cap * n);
  std::vector<double> hq((size_t)cap * n), hp((size_t)cap * n);
  CUDA_OR_FAIL(c, cudaMemcpy(hv.data(), c->d_vert, hv.size() * sizeof(int16_t), cudaMemcpyDeviceToHost));
  CUDA_OR_FAIL(c, cudaMemcpy(hq.data(), c->d_q, hq.size() * sizeof(double), cudaMemcpyDeviceToHost));
  CUDA_OR_FAIL(c, cudaMemcpy(hp.data(), c->d_price, hp.size() * sizeof(double), cudaMemcpyDeviceToHost));
  for (int64_t r = 0; r < n; ++r)
    for (int j = 0; j < cap; ++j) {
      vert[r * cap + j] = hv[(size_t)j * n + r];
      q[r * cap + j] = hq[(size_t)j * n + r];
      price[r * cap + j] = hp[(size_t)j * n + r];
    }
  return ESDP_OK;
}

esdp_status esdp_simulate_dev(esdp_ctx* c, int64_t n_paths, uint64_t seed, double* per_path_dev, void* stream) {
  if (!c) return ESDP_E_STATE;
  if (!c->solved) return fail(c, ESDP_E_STATE, "no backward pass has run");
  if (n_paths < 1) return fail(c, ESDP_E_STATE, "n_paths must be >= 1");
  SimParams sp;
  sp.pol = c->d_pol; sp.lambda = c->d_lambda;
  sim_tables(c, sp);
  sp.act = c->d_act; sp.w = c->d_w; sp.off = c->d_off; sp.g = c->d_g;
  sp.T = c->T; sp.K = c->K; sp.S = c->S; sp.A = c->A; sp.rank1 = c->rank1; sp.kind = c->kind; sp.Kp = c->Kp;
  sp.on_grid = c->on_grid; sp.f0 = c->f0; sp.w0 = c->w0;
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  if (esdp_status e = ready_tables(c, s)) return e;   // sampling tables of the last upload
  const int thr = 128;
  const size_t sm = sim_smem_bytes(c->A);
  if (sm > 48 * 1024) cudaFuncSetAttribute(simulate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  simulate_kernel<<<(unsigned)((n_paths + thr - 1) / thr), thr, sm, s>>>(sp, n_paths, seed, per_path_dev);
  CUDA_OR_FAIL(c, cudaGetLastError());
  return mark_use(c, s);
}

esdp_status esdp_price_paths_dev(esdp_ctx* c, int64_t n_paths, uint64_t seed, int16_t* kpath_dev, double* lambda_dev,
                                 void* stream) {
  if (!c) return ESDP_E_STATE;
  if (n_paths < 1 || (!kpath_dev && !lambda_dev)) return fail(c, ESDP_E_STATE, "n_paths >= 1 and an output are required");
  SimParams sp{};
  sp.lambda = c->d_lambda;
  sim_tables(c, sp);
  sp.T = c->T; sp.K = c->K; sp.rank1 = c->rank1;
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  if (esdp_status e = ready_tables(c, s)) return e;
  price_path_kernel<<<(unsigned)((n_paths + 127) / 128), 128, 0, s>>>(sp, n_paths, seed, kpath_dev, lambda_dev);
  CUDA_OR_FAIL(c, cudaGetLastError());
  return mark_use(c, s);
}

esdp_status esdp_simulate_async(esdp_ctx* c, int64_t n_paths, uint64_t seed, double* stats_dev, void* stream) {
  if (!c || !stats_dev) return ESDP_E_STATE;
  if (n_paths > c->sim_cap) {
    cudaFree(c->d_sim);
    c->d_sim = nullptr;
    c->sim_cap = 0;
    if (dev_alloc(c, &c->d_sim, n_paths)) return ESDP_E_NOMEM;
    c->sim_cap = n_paths;
  }
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  esdp_status st = esdp_simulate_dev(c, n_paths, seed, c->d_sim, s);
  if (st != ESDP_OK) return st;
  reduce_kernel<<<1, 1024, 0, s>>>(c->d_sim, n_paths, nullptr, c->d_red);
  reduce_kernel<<<1, 1024, 0, s>>>(c->d_sim, n_paths, c->d_red, c->d_red + 1);
  finalize_stats_kernel<<<1, 1, 0, s>>>(c->d_red, n_paths, stats_dev);
  CUDA_OR_FAIL(c, cudaGetLastError());
  return ESDP_OK;
}

esdp_status esdp_simulate(esdp_ctx* c, int64_t n_paths, uint64_t seed, double* mean, double* var, double* per_path) {
  if (!c) return ESDP_E_STATE;
  if (n_paths > c->sim_cap) {
    cudaFree(c->d_sim);
    c->d_sim = nullptr;
    c->sim_cap = 0;
    if (dev_alloc(c, &c->d_sim, n_paths)) return ESDP_E_NOMEM;
    c->sim_cap = n_paths;
  }
  esdp_status st = esdp_simulate_dev(c, n_paths, seed, c->d_sim, c->stream);
  if (st != ESDP_OK) return st;
  reduce_kernel<<<1, 1024, 0, c->stream>>>(c->d_sim, n_paths, nullptr, c->d_red);
  reduce_kernel<<<1, 1024, 0, c->stream>>>(c->d_sim, n_paths, c->d_red, c->d_red + 1);
  CUDA_OR_FAIL(c, cudaGetLastError());
  CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  double h[2];
  CUDA_OR_FAIL(c, cudaMemcpy(h, c->d_red, 2 * sizeof(double), cudaMemcpyDeviceToHost));
  if (mean) *mean = h[0];
  if (var) *var = n_paths > 1 ? h[1] / (double)(n_paths - 1) : 0.0;
  if (per_path) CUDA_OR_FAIL(c, cudaMemcpy(per_path, c->d_sim, n_paths * sizeof(double), cudaMemcpyDeviceToHost));
  return ESDP_OK;
}

esdp_status esdp_simulate_strategy_dev(esdp_ctx* c, int64_t n_paths, uint64_t seed, int32_t mode,
                                       const int16_t* schedule_dev, int16_t* actions_dev, double* per_path_dev,
                                       void* stream) {
  if (!c) return ESDP_E_STATE;
  if (mode == ESDP_SIM_LOTTERY && !actions_dev) return esdp_simulate_dev(c, n_paths, seed, per_path_dev, stream);
  if (mode < ESDP_SIM_PHYSICAL || mode > ESDP_SIM_FIXED) return fail(c, ESDP_E_STATE, "unknown simulation mode %d", mode);
  if (!c->solved) return fail(c, ESDP_E_STATE, "no backward pass has run");
  if (n_paths < 1) return fail(c, ESDP_E_STATE, "n_paths must be >= 1");
  if (mode != ESDP_SIM_FIXED && !keep(c))
    return fail(c, ESDP_E_STATE, "physical / bid-clearing / self-scheduled simulation needs ESDP_KEEP_VALUES (W of every stage)");
  if (mode != ESDP_SIM_FIXED && c->world > 1)
    return fail(c, ESDP_E_STATE, "physical / bid-clearing / self-scheduled simulation needs every W row (world == 1)");
  if ((mode == ESDP_SIM_CLEAR_BIDS || mode == ESDP_SIM_SELF) && c->kind == ESDP_PAYOFF_TABLE)
    return fail(c, ESDP_E_STATE, "bid curves / lagged-price decisions are not defined for TABLE payoffs (R13)");
  if (mode == ESDP_SIM_FIXED && !schedule_dev) return fail(c, ESDP_E_STATE, "the fixed-schedule mode needs a schedule");
  if (actions_dev && mode == ESDP_SIM_CLEAR_BIDS) return fail(c, ESDP_E_STATE, "action recording: physical, self or fixed");
  if (mode == ESDP_SIM_CLEAR_BIDS && n_paths * c->A > c->stack_cap) {
    cudaFree(c->d_stack);
    c->d_stack = nullptr;
    c->stack_cap = 0;
    if (dev_alloc(c, &c->d_stack, (size_t)n_paths * c->A)) return ESDP_E_NOMEM;
    c->stack_cap = n_paths * c->A;
  }
  SimModeParams mp{};
  SimParams& sp = mp.base;
  sp.pol = c->d_pol; sp.lambda = c->d_lambda;
  sim_tables(c, sp);
  sp.act = c->d_act; sp.w = c->d_w; sp.off = c->d_off; sp.g = c->d_g;
  sp.T = c->T; sp.K = c->K; sp.S = c->S; sp.A = c->A; sp.rank1 = c->rank1; sp.kind = c->kind; sp.Kp = c->Kp;
  sp.on_grid = c->on_grid; sp.f0 = c->f0; sp.w0 = c->w0;
  mp.W = c->d_W; mp.F = c->d_F; mp.omw = c->d_omw; mp.stack = c->d_stack;
  mp.schedule = schedule_dev; mp.actions = actions_dev;
  mp.mode = mode; mp.wrows = (int)w_rows(c); mp.ld = c->ld; mp.delta = c->delta; mp.s0 = c->s0;
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  if (esdp_status e = ready_tables(c, s)) return e;
  const size_t sm = simmode_smem_bytes(c->A);
  if (sm > 48 * 1024) cudaFuncSetAttribute(simulate_mode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  simulate_mode_kernel<<<(unsigned)((n_paths + kSimModeThreads - 1) / kSimModeThreads), kSimModeThreads, sm, s>>>(
      mp, n_paths, seed, per_path_dev);
  CUDA_OR_FAIL(c, cudaGetLastError());
  return mark_use(c, s);
}

esdp_status esdp_simulate_mode_dev(esdp_ctx* c, int64_t n_paths, uint64_t seed, int32_t mode, double* per_path_dev,
                                   void* stream) {
  if (c && mode == ESDP_SIM_FIXED) return fail(c, ESDP_E_STATE, "the fixed-schedule mode needs esdp_simulate_strategy_dev");
  return esdp_simulate_strategy_dev(c, n_paths, seed, mode, nullptr, nullptr, per_path_dev, stream);
}

esdp_status esdp_simulate_mode(esdp_ctx* c, int64_t n_paths, uint64_t seed, int32_t mode, double* mean, double* var,
                               double* per_path) {
  if (!c) return ESDP_E_STATE;
  if (n_paths > c->sim_cap) {
    cudaFree(c->d_sim);
    c->d_sim = nullptr;
    c->sim_cap = 0;
    if (dev_alloc(c, &c->d_sim, n_paths)) return ESDP_E_NOMEM;
    c->sim_cap = n_paths;
  }
  esdp_status st = esdp_simulate_mode_dev(c, n_paths, seed, mode, c->d_sim, c->stream);
  if (st != ESDP_OK) return st;
  reduce_kernel<<<1, 1024, 0, c->stream>>>(c->d_sim, n_paths, nullptr, c->d_red);
  reduce_kernel<<<1, 1024, 0, c->stream>>>(c->d_sim, n_paths, c->d_red, c->d_red + 1);
  CUDA_OR_FAIL(c, cudaGetLastError());
  CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  double h[2];
  CUDA_OR_FAIL(c, cudaMemcpy(h, c->d_red, 2 * sizeof(double), cudaMemcpyDeviceToHost));
  if (mean) *mean = h[0];
  if (var) *var = n_paths > 1 ? h[1] / (double)(n_paths - 1) : 0.0;
  if (per_path) CUDA_OR_FAIL(c, cudaMemcpy(per_path, c->d_sim, n_paths * sizeof(double), cudaMemcpyDeviceToHost));
  return ESDP_OK;
}

esdp_status esdp_window_level_tables(esdp_ctx* c, int64_t* count) {
  if (!c || !count) return ESDP_E_STATE;
  unsigned long long v = 0, z = 0;
  CUDA_OR_FAIL(c, cudaMemcpyFromSymbol(&v, g_window_level_tables, sizeof(v)));
  CUDA_OR_FAIL(c, cudaMemcpyToSymbol(g_window_level_tables, &z, sizeof(z)));
  *count = (int64_t)v;
  return ESDP_OK;
}

esdp_status esdp_window_fallbacks(esdp_ctx* c, int64_t* count) {
  if (!c || !count) return ESDP_E_STATE;
  unsigned long long v = 0, z = 0;
  CUDA_OR_FAIL(c, cudaMemcpyFromSymbol(&v, g_window_fallbacks, sizeof(v)));
  CUDA_OR_FAIL(c, cudaMemcpyToSymbol(g_window_fallbacks, &z, sizeof(z)));
  *count = (int64_t)v;
  return ESDP_OK;
}

esdp_status esdp_stencil_kind(const esdp_ctx* c, int32_t* kind) {
  if (!c || !kind) return ESDP_E_STATE;
  // bit 0: window stencil; bit 1: expectation on the FP64 tensor cores (DMMA); bit 2: the DMMA probe failed
  *kind = c->use_window | ((c->flags & ESDP_NO_DMMA) ? 0 : 2) | (c->dmma_probe_failed ? 4 : 0);
  return ESDP_OK;
}

esdp_status esdp_launch_count(const esdp_ctx* c, int64_t* n) {
  if (!c || !n) return ESDP_E_STATE;
  *n = c->launches;
  return ESDP_OK;
}

esdp_status esdp_kernel_times(const esdp_ctx* cc, double* contract_ms, double* stencil_ms) {
  esdp_ctx* c = const_cast<esdp_ctx*>(cc);
  if (!c) return ESDP_E_STATE;
  if (c->ev.empty()) return fail(c, ESDP_E_STATE, "context was created without ESDP_PROFILE");
  if (!c->solved) return fail(c, ESDP_E_STATE, "no backward pass has run");
  double ct = 0.0, st = 0.0;
  int nc = 0, ns = 0;
  for (int t = 1; t <= c->T; ++t) {
    if (t % c->prof_stride != 0) continue;
    float ms = 0.f;
    if (t < c->T) {
      CUDA_OR_FAIL(c, cudaEventElapsedTime(&ms, c->ev[(size_t)(t - 1) * 4 + 0], c->ev[(size_t)(t - 1) * 4 + 1]));
      ct += ms;
      ++nc;
    }
    CUDA_OR_FAIL(c, cudaEventElapsedTime(&ms, c->ev[(size_t)(t - 1) * 4 + 2], c->ev[(size_t)(t - 1) * 4 + 3]));
    st += ms;
    ++ns;
  }
  if (contract_ms) *contract_ms = nc ? ct / nc : 0.0;
  if (stencil_ms) *stencil_ms = ns ? st / ns : 0.0;
  return ESDP_OK;
}

esdp_status esdp_debug_time(esdp_ctx* c, int32_t what, int32_t reps, double* us_per_launch) {
  // Diagnostic: warm back-to-back launches of one kernel kind of stage T-1 (0 = contraction, 1 = the
  // context's stencil, 2 = brute-force stencil, 3 = empty kernel), captured in a graph and timed with
  // CUDA events.  Requires a completed backward pass (its buffers are reused as inputs).
  if (!c || !us_per_launch || reps < 1) return ESDP_E_STATE;
  if (!c->solved) return fail(c, ESDP_E_STATE, "no backward pass has run");
  const int T = c->T, K = c->K, S = c->S;
  const int t = T > 1 ? T - 1 : T;
  cudaStream_t s = c->stream;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  CUDA_OR_FAIL(c, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int r = 0; r < reps; ++r) {
    cudaError_t le;
    if (what == 0 && T > 1) le = launch_contract(c, t, s, false);
    else if (what == 1 || what == 2) le = launch_stencil(c, t, s, false, what == 2);
    else le = launch_objective(c, s, false);
    if (le != cudaSuccess) { cudaStreamEndCapture(s, &g); if (g) cudaGraphDestroy(g); return fail(c, ESDP_E_CUDA, "debug launch: %s", cudaGetErrorString(le)); }
  }
  cudaError_t ce = cudaStreamEndCapture(s, &g);
  if (ce != cudaSuccess) return fail(c, ESDP_E_CUDA, "debug capture: %s", cudaGetErrorString(ce));
  ce = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  if (ce != cudaSuccess) return fail(c, ESDP_E_CUDA, "debug instantiate: %s", cudaGetErrorString(ce));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(e0, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  ce = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  cudaGraphExecDestroy(ge);
  if (ce != cudaSuccess) return fail(c, ESDP_E_CUDA, "debug run: %s", cudaGetErrorString(ce));
  *us_per_launch = 1e3 * ms / reps;
  return ESDP_OK;
}

void esdp_destroy(esdp_ctx* c) {
  if (!c) return;
  cudaStreamSynchronize(c->stream);
  free_all(c);
  delete c;
}

const char* esdp_last_error(const esdp_ctx* c) { return c ? c->err.c_str() : g_create_error.c_str(); }

// ------------------------------------------------------------------------------------------------
// Batch contexts (cfg5): see batch.cuh and include/esdp.h.
// ------------------------------------------------------------------------------------------------
}  // extern "C"

struct esdp_batch {
  int n = 0, T = 0, K = 0, S = 0, ld = 0, rank1 = 0, gbits = 0, g_max = 0;   // guide bits: tables, pi_1
  std::vector<esdp_ctx*> inst;        // per-instance parameters and action tables (tables_only contexts)
  double *d_lambda = nullptr, *d_P = nullptr, *d_pi = nullptr, *d_cdf = nullptr, *d_cdf1 = nullptr;
  uint64_t *d_guide = nullptr, *d_guide1 = nullptr;
  int *d_tab = nullptr, *d_src = nullptr;   // Markov: deduplicated sampling tables (as esdp_ctx's slots)
  double *d_V = nullptr, *d_W = nullptr, *d_J = nullptr;   // V [2][K][n][ld], W [rows][n][ld]
  int16_t* d_pol = nullptr;                                // [n][T][K][S]
  BatchInst* d_bi = nullptr;
  int* d_widx = nullptr;                                   // window-plan instances
  int* d_bidx = nullptr;                                   // brute-force instances
  int nwin = 0, nbrute = 0;
  int win_opt = 4, win_levels = 0;   // batch window kernel variant (window.cuh)
  int dmma = 1;   // expectation on the FP64 tensor cores (0: the DMMA probe failed -> DFMA)
  int ozaki = 0;  // expectation as Ozaki-sliced u8 tcgen05 products (ESDP_CONTRACT_OZAKI granted, ozaki.cuh)
  size_t ntab_cap = 0;   // sampling-table rows the guide allocation holds (distinct P_t slices x K)
  size_t win_smem = 0, brute_smem = 0;
  cudaStream_t stream = nullptr;
  // instance groups with independent stage chains (graph branches; ESDP_BATCH_GROUPS): group g's expectation
  // runs while another group's window stencil does
  int groups = 1;
  std::vector<cudaStream_t> gstream;   // groups - 1 extra capture streams
  std::vector<cudaEvent_t> gev;        // fork, offset and join events
  cudaGraphExec_t graph = nullptr;
  int64_t launches = 0;
  bool solved = false;
  std::string err;
};

namespace {

esdp_status bfail(esdp_batch* b, esdp_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (b) b->err = buf; else g_create_error = buf;
  return st;
}
#define BCUDA(b, call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) return bfail(b, ESDP_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

template <class T>
esdp_status balloc(esdp_batch* b, T** p, size_t n) {
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc((void**)p, n * sizeof(T));
  if (e != cudaSuccess) return bfail(b, ESDP_E_NOMEM, "cudaMalloc(%zu bytes): %s", n * sizeof(T), cudaGetErrorString(e));
  return ESDP_OK;
}

void batch_free(esdp_batch* b) {
  if (b->graph) cudaGraphExecDestroy(b->graph);
  void* ps[] = {b->d_lambda, b->d_P, b->d_pi, b->d_cdf, b->d_cdf1, b->d_guide, b->d_guide1, b->d_tab, b->d_src, b->d_V, b->d_W,
                b->d_J, b->d_pol, b->d_bi, b->d_widx, b->d_bidx};
  for (void* p : ps)
    if (p) cudaFree(p);
  for (esdp_ctx* c : b->inst) esdp_destroy(c);
  for (cudaStream_t x : b->gstream) if (x) cudaStreamDestroy(x);
  for (cudaEvent_t e : b->gev) if (e) cudaEventDestroy(e);
  if (b->stream) cudaStreamDestroy(b->stream);
}

// The batch's backward pass on stream s: per stage one expectation over [K] x [n ld], one window launch
// over every window-plan instance, one brute-force launch per other instance; then every J.
// One batch kernel of stage t: what = 0 the contraction W_t = P_t V_{t+1} over all instances' columns,
// 1 the window-plan instances' stencil, 2 the brute-force instances' stencil.
// g0, gn: the instances [g0, g0 + gn) (an instance group; columns [g0 ld, (g0 + gn) ld) of V and W).  Groups
// other than the whole batch only for the DMMA / Ozaki expectation and the window stencil (all instances
// window-plan: the window list is then 0 .. n-1).
cudaError_t batch_stage_kernel(esdp_batch* b, int t, int what, cudaStream_t s, bool pdl, int g0 = 0, int gn = -1) {
  const int T = b->T, K = b->K, S = b->S, n = b->n;
  const size_t NL = (size_t)n * b->ld;                  // row stride of V and W
  const int rows = b->rank1 ? 1 : K;
  double* V_t = b->d_V + (size_t)((t - 1) & 1) * K * NL;
  const double* V_n = b->d_V + (size_t)(t & 1) * K * NL;   // V_{t+1}
  if (gn < 0) gn = n;
  if (what == 0) {
    const double* Pt = b->rank1 ? b->d_pi + (size_t)t * K : b->d_P + (size_t)(t - 1) * K * K;
    const size_t c0 = (size_t)g0 * b->ld, nc = (size_t)gn * b->ld;
    if (b->ozaki)
      return launch_ozaki(Pt, V_n + c0, b->d_W + c0, K, K, (long long)nc, (long long)NL, (long long)NL, s, pdl);
    if (!b->rank1 && b->dmma && use_pres(rows, K, (int64_t)nc))
      return launch_pres(Pt, V_n + c0, b->d_W + c0, rows, K, (int64_t)nc, (int)NL, s, pdl);
    if (const int d3 = (b->rank1 || !b->dmma) ? 0 : use_dmma3(rows, (int64_t)nc, K))
      return launch_dmma3(d3, Pt, V_n + c0, b->d_W + c0, rows, K, (int)nc, (int)NL, s, pdl);
    if (gn != n) return cudaErrorInvalidValue;   // groups only on the DMMA / Ozaki expectations
    if (b->dmma && !b->rank1 && K > 128 && contract_dmma2_smem(K, kDRbig, kDCbig) <= 200 * 1024) {
      const int ncb = (int)((NL + kDCbig * 16 - 1) / (kDCbig * 16)), nrb = (K + kDRbig * 8 - 1) / (kDRbig * 8);
      return launch(contract_dmma2_kernel<kDRbig, kDCbig>, dim3(ncb * nrb), dim3(kDRbig * kDCbig * 32),
                    contract_dmma2_smem(K, kDRbig, kDCbig), s, pdl, Pt, V_n, b->d_W, rows, K, (int)NL, (int)NL, ncb);
    }
    if (b->dmma && !b->rank1 && contract_dmma2_smem(K) <= 200 * 1024) {
      const int ncb = (int)((NL + kDC * 16 - 1) / (kDC * 16)), nrb = (K + kDR * 8 - 1) / (kDR * 8);
      return launch(contract_dmma2_kernel<kDR, kDC>, dim3(ncb * nrb), dim3(kDR * kDC * 32), contract_dmma2_smem(K), s, pdl,
                    Pt, V_n, b->d_W, rows, K, (int)NL, (int)NL, ncb);
    }
    dim3 grid((unsigned)((NL + kColsC - 1) / kColsC), (rows + kRowsC - 1) / kRowsC);
    return launch(contract_kernel, grid, dim3(kThreadsC), contract_smem_bytes(K), s, pdl, Pt, V_n, b->d_W, rows, K, (int)NL,
                  (int)NL);
  }
  const double* lam = b->d_lambda + (size_t)(t - 1) * K;
  const size_t pol_inst = (size_t)T * K * S, pol_stage = (size_t)(t - 1) * K * S;
  if (what == 1)
    return launch(window_batch_kernel_of(b->win_opt, b->win_levels),
                  dim3((S + kWinThreads * b->win_opt - 1) / (kWinThreads * b->win_opt), K, gn == n ? b->nwin : gn),
                  dim3(kWinThreads), b->win_smem, s, pdl, (const BatchInst*)b->d_bi, (const int*)b->d_widx + g0,
                  (const double*)b->d_W, V_t, b->d_pol, pol_inst, pol_stage, lam, b->ld, (int)NL, b->rank1);
  return launch(stencil_batch_kernel, dim3((S + kTile - 1) / kTile, K, b->nbrute), dim3(kStencilWarps * 32), b->brute_smem,
                s, pdl, (const BatchInst*)b->d_bi, (const int*)b->d_bidx, (const double*)b->d_W, V_t, b->d_pol, pol_inst,
                pol_stage, lam, b->ld, (int)NL, b->rank1);
}

esdp_status batch_enqueue(esdp_batch* b, cudaStream_t s) {
  const int T = b->T, K = b->K, n = b->n;
  const size_t NL = (size_t)n * b->ld;                  // row stride of V and W
  const int rows = b->rank1 ? 1 : K;
  int64_t launches = 0;
  bool after_kernel = false;
  if (b->groups > 1) {   // independent chains of instance groups, each on its own capture stream
    const int G = b->groups;
    BCUDA(b, cudaMemsetAsync(b->d_W, 0, rows * NL * sizeof(double), s));   // W_T = 0
    BCUDA(b, cudaEventRecord(b->gev[0], s));
    std::vector<cudaStream_t> gs(G, s);
    for (int g = 1; g < G; ++g) { gs[g] = b->gstream[g - 1]; BCUDA(b, cudaStreamWaitEvent(gs[g], b->gev[0], 0)); }
    std::vector<char> ak(G, 0);
    for (int t = T; t >= 1; --t)
      for (int g = 0; g < G; ++g) {
        const int g0 = (int)((int64_t)n * g / G), gn = (int)((int64_t)n * (g + 1) / G) - g0;
        if (t < T) {
          const cudaError_t e = batch_stage_kernel(b, t, 0, gs[g], ak[g], g0, gn);
          if (e != cudaSuccess) return bfail(b, ESDP_E_CUDA, "batch contraction: %s", cudaGetErrorString(e));
          ak[g] = 1;
          ++launches;
        }
        if (t == T && g > 0) {   // start half a stage behind the previous group: its expectation overlaps our stencil
          BCUDA(b, cudaStreamWaitEvent(gs[g], b->gev[g], 0));
          ak[g] = 0;
        }
        const cudaError_t e = batch_stage_kernel(b, t, 1, gs[g], ak[g], g0, gn);
        if (e != cudaSuccess) return bfail(b, ESDP_E_CUDA, "batch window stencil: %s", cudaGetErrorString(e));
        ak[g] = 1;
        ++launches;
        if (t == T && g + 1 < G) BCUDA(b, cudaEventRecord(b->gev[g + 1], gs[g]));
      }
    for (int g = 1; g < G; ++g) {
      BCUDA(b, cudaEventRecord(b->gev[G + g], gs[g]));
      BCUDA(b, cudaStreamWaitEvent(s, b->gev[G + g], 0));
    }
    after_kernel = false;
  }
  for (int t = b->groups > 1 ? 0 : T; t >= 1; --t) {
    if (t == T) {
      BCUDA(b, cudaMemsetAsync(b->d_W, 0, rows * NL * sizeof(double), s));   // W_T = 0
      after_kernel = false;
    } else {
      const cudaError_t e = batch_stage_kernel(b, t, 0, s, after_kernel);
      if (e != cudaSuccess) return bfail(b, ESDP_E_CUDA, "batch contraction: %s", cudaGetErrorString(e));
      after_kernel = true;
      ++launches;
    }
    if (b->nwin > 0) {
      const cudaError_t e = batch_stage_kernel(b, t, 1, s, after_kernel);
      if (e != cudaSuccess) return bfail(b, ESDP_E_CUDA, "batch window stencil: %s", cudaGetErrorString(e));
      ++launches;
    }
    if (b->nbrute > 0) {
      const cudaError_t e = batch_stage_kernel(b, t, 2, s, after_kernel && b->nwin == 0);
      if (e != cudaSuccess) return bfail(b, ESDP_E_CUDA, "batch stencil: %s", cudaGetErrorString(e));
      ++launches;
    }
    after_kernel = b->nbrute == 0;   // a PDL edge needs a single kernel predecessor
  }
  {
    cudaError_t e = launch(objective_batch_kernel, dim3(n), dim3(128), 2 * sizeof(double) * K, s, after_kernel,
                           (const BatchInst*)b->d_bi, (const double*)(b->d_V), (const double*)b->d_pi, K, b->ld, (int)NL,
                           b->d_J);
    if (e != cudaSuccess) return bfail(b, ESDP_E_CUDA, "batch objective: %s", cudaGetErrorString(e));
    ++launches;
  }
  b->launches = launches;
  return ESDP_OK;
}

}  // namespace

extern "C" {

esdp_status esdp_create_batch(const esdp_problem* probs, int32_t n, esdp_batch** out) {
  g_create_error.clear();
  if (!probs || !out || n < 1) return bfail(nullptr, ESDP_E_CONFIG, "null argument or n < 1");
  *out = nullptr;
  const esdp_problem& p0 = probs[0];
  for (int m = 0; m < n; ++m) {
    const esdp_problem& q = probs[m];
    if (q.T != p0.T || q.K != p0.K || q.sbar != p0.sbar || q.delta != p0.delta || (q.P == nullptr) != (p0.P == nullptr))
      return bfail(nullptr, ESDP_E_CONFIG, "instance %d: T, K, sbar, delta and the price model must match instance 0", m);
    if (q.payoff_kind == ESDP_PAYOFF_TABLE)
      return bfail(nullptr, ESDP_E_CONFIG, "instance %d: TABLE payoffs are not supported in a batch", m);
    if (!q.lambda || !q.pi || (q.payoff_kind != ESDP_PAYOFF_LINEAR && !q.g))
      return bfail(nullptr, ESDP_E_CONFIG, "instance %d: lambda, pi (and g) are required", m);
    const size_t TK = (size_t)q.T * q.K;
    const bool same = std::memcmp(q.lambda, p0.lambda, TK * sizeof(double)) == 0 &&
                      std::memcmp(q.pi, p0.pi, (q.P ? (size_t)q.K : TK) * sizeof(double)) == 0 &&
                      (!q.P || q.P == p0.P || std::memcmp(q.P, p0.P, (size_t)(q.T - 1) * q.K * q.K * sizeof(double)) == 0);
    if (!same) return bfail(nullptr, ESDP_E_CONFIG, "instance %d: lambda, P and pi must equal instance 0's (shared price model)", m);
  }
  esdp_batch* b = new esdp_batch();
  auto bail = [&](esdp_status st) { if (b->err.size()) g_create_error = b->err; batch_free(b); delete b; return st; };
#define BTRY(x) do { esdp_status st_ = (x); if (st_ != ESDP_OK) return bail(st_); } while (0)
  b->n = n;
  b->dmma = !(probs[0].flags & ESDP_NO_DMMA) && dmma_probe_mismatches() == 0;   // guard as esdp_create
  for (int m = 0; m < n; ++m) {
    esdp_problem q = probs[m];
    q.flags &= ~(uint32_t)(ESDP_KEEP_VALUES | ESDP_PROFILE);
    esdp_ctx* c = nullptr;
    esdp_status st = create_impl(&q, 1, 0, nullptr, &c, true);
    if (st != ESDP_OK) {
      b->err = "instance " + std::to_string(m) + ": " + g_create_error;
      return bail(st);
    }
    b->inst.push_back(c);
  }
  esdp_ctx* c0 = b->inst[0];
  b->T = c0->T; b->K = c0->K; b->S = c0->S; b->ld = c0->ld; b->rank1 = c0->rank1; b->g_max = c0->g_max;
  if ((p0.flags & ESDP_CONTRACT_OZAKI) && !b->rank1 && b->K <= kOzM && b->K <= kOzK) {
    // granted when every V_{t+1} >= 0 (the digits are unsigned): the zero action's payoff is >= 0 in every
    // instance (R18: V_t >= P_t V_{t+1} >= 0); P is validated stochastic, so P >= 0
    bool nonneg = true;
    for (int m = 0; m < n; ++m) {
      const esdp_ctx* c = b->inst[m];
      if (c->kind == ESDP_PAYOFF_LINEAR_MINUS_G && !(probs[m].g[c->a_z] <= 0.0)) nonneg = false;
    }
    b->ozaki = nonneg ? 1 : 0;
  }
  {   // the shared inputs, validated once (as esdp_create does)
    esdp_status st = validate_data(c0, p0.lambda, p0.P, p0.pi, p0.g);
    if (st != ESDP_OK) { b->err = c0->err; return bail(st); }
  }
  if (cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(bfail(b, ESDP_E_CUDA, "cannot create a CUDA stream"));
  const size_t T = b->T, K = b->K, S = b->S, NL = (size_t)n * b->ld;
  std::vector<int> tab, src;   // Markov: one sampling table per distinct slice P_t
  if (!b->rank1 && T > 1) dedupe_slices(p0.P, (int)T - 1, (int)K, tab, src);
  const size_t ntab_rows = b->rank1 ? T : src.size() * K;
  b->gbits = b->rank1 ? c0->g_r1 : guide_g_for(ntab_rows, c0->guide_cap, c0->g_max);
  b->ntab_cap = std::max<size_t>(ntab_rows, 1);
  BTRY(balloc(b, &b->d_lambda, T * K));
  BTRY(balloc(b, &b->d_P, b->rank1 ? 1 : (T - 1) * K * K));
  BTRY(balloc(b, &b->d_pi, b->rank1 ? T * K : K));
  BTRY(balloc(b, &b->d_cdf, b->rank1 ? T * K : (T - 1) * K * K));
  BTRY(balloc(b, &b->d_cdf1, K));
  BTRY(balloc(b, &b->d_guide, std::max<size_t>(ntab_rows, 1) << b->gbits));
  BTRY(balloc(b, &b->d_guide1, (size_t)1 << b->g_max));
  if (!tab.empty()) {
    BTRY(balloc(b, &b->d_tab, tab.size()));
    BTRY(balloc(b, &b->d_src, src.size()));
  }
  BTRY(balloc(b, &b->d_V, 2 * K * NL));
  BTRY(balloc(b, &b->d_W, (b->rank1 ? 1 : K) * NL));
  BTRY(balloc(b, &b->d_pol, (size_t)n * T * K * S));
  BTRY(balloc(b, &b->d_J, (size_t)n));
  BTRY(balloc(b, &b->d_bi, (size_t)n));
  BTRY(balloc(b, &b->d_widx, (size_t)n));
  BTRY(balloc(b, &b->d_bidx, (size_t)n));
  cudaStream_t s = b->stream;
  cudaMemsetAsync(b->d_V, 0, 2 * K * NL * sizeof(double), s);
  cudaMemsetAsync(b->d_W, 0, (b->rank1 ? 1 : K) * NL * sizeof(double), s);
  BCUDA(b, cudaMemcpyAsync(b->d_lambda, p0.lambda, T * K * sizeof(double), cudaMemcpyHostToDevice, s));
  if (b->rank1) {
    BCUDA(b, cudaMemcpyAsync(b->d_pi, p0.pi, T * K * sizeof(double), cudaMemcpyHostToDevice, s));
    launch_cdf(b->d_pi, nullptr, (int64_t)T, (int)K, b->gbits, b->d_cdf, b->d_guide, s);
  } else {
    BCUDA(b, cudaMemcpyAsync(b->d_pi, p0.pi, K * sizeof(double), cudaMemcpyHostToDevice, s));
    if (T > 1) {
      BCUDA(b, cudaMemcpyAsync(b->d_P, p0.P, (T - 1) * K * K * sizeof(double), cudaMemcpyHostToDevice, s));
      BCUDA(b, cudaMemcpyAsync(b->d_tab, tab.data(), tab.size() * sizeof(int), cudaMemcpyHostToDevice, s));
      BCUDA(b, cudaMemcpyAsync(b->d_src, src.data(), src.size() * sizeof(int), cudaMemcpyHostToDevice, s));
      launch_cdf(b->d_P, b->d_src, (int64_t)ntab_rows, (int)K, b->gbits, b->d_cdf, b->d_guide, s);
    }
  }
  launch_cdf(b->d_pi, nullptr, 1, (int)K, b->g_max, b->d_cdf1, b->d_guide1, s);
  BCUDA(b, cudaGetLastError());
  // per-instance parameters
  std::vector<BatchInst> hbi((size_t)n);
  std::vector<int> widx, bidx;
  for (int m = 0; m < n; ++m) {
    esdp_ctx* c = b->inst[m];
    BatchInst& x = hbi[m];
    std::memset(&x, 0, sizeof x);
    x.wp = win_params(c);
    x.wp.K = (int)K;
    x.sp = stencil_params(c);
    x.sp.K = (int)K;
    SimParams& sp = x.sim;
    sp.pol = b->d_pol + (size_t)m * T * K * S; sp.cdf = b->d_cdf; sp.cdf1 = b->d_cdf1; sp.lambda = b->d_lambda;
    sp.guide = b->d_guide; sp.guide1 = b->d_guide1; sp.tab = b->d_tab;
    sp.gs = 53 - b->gbits; sp.gs1 = 53 - b->g_max;
    sp.act = c->d_act; sp.w = c->d_w; sp.off = c->d_off; sp.g = c->d_g;
    sp.T = (int)T; sp.K = (int)K; sp.S = (int)S; sp.A = c->A; sp.rank1 = b->rank1; sp.kind = c->kind; sp.Kp = (int)K;
    sp.on_grid = c->on_grid; sp.f0 = c->f0; sp.w0 = c->w0;
    x.f0 = c->f0; x.on_grid = c->on_grid; x.w0 = c->w0;
    if (c->use_window) {
      widx.push_back(m);
      b->win_levels |= c->win_levels;
    } else {
      bidx.push_back(m);
      b->brute_smem = std::max(b->brute_smem, c->stencil_smem);
    }
  }
  b->nwin = (int)widx.size();
  b->nbrute = (int)bidx.size();
  {   // one window variant for every window instance: levels if any instance needs them (then one output per thread)
    const char* e = getenv("ESDP_WIN_OPT");
    const int eo = e ? atoi(e) : 0;
    b->win_opt = b->win_levels ? 1 : (eo == 1 || eo == 2 || eo == 4) ? eo : 4;
    for (int m : widx) {
      const esdp_ctx* c = b->inst[m];
      b->win_smem = std::max(b->win_smem, window_smem_bytes(c->Lc, c->Ld, c->o_max - c->o_min, c->A, b->win_opt,
                                                            b->win_levels != 0));
    }
  }
  if (!bidx.empty()) BCUDA(b, cudaMemcpyAsync(b->d_bidx, bidx.data(), bidx.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  if (b->brute_smem > 48 * 1024)
    BCUDA(b, cudaFuncSetAttribute(stencil_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b->brute_smem));
  BCUDA(b, cudaMemcpyAsync(b->d_bi, hbi.data(), n * sizeof(BatchInst), cudaMemcpyHostToDevice, s));
  if (!widx.empty()) BCUDA(b, cudaMemcpyAsync(b->d_widx, widx.data(), widx.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  BCUDA(b, cudaStreamSynchronize(s));
  if (b->win_smem > 48 * 1024)
    BCUDA(b, cudaFuncSetAttribute(window_batch_kernel_of(b->win_opt, b->win_levels), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)b->win_smem));
  if (contract_dmma2_smem(K) > 48 * 1024 && contract_dmma2_smem(K) <= 200 * 1024)
    cudaFuncSetAttribute(contract_dmma2_kernel<kDR, kDC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)contract_dmma2_smem(K));
  if (K > 128 && contract_dmma2_smem(K, kDRbig, kDCbig) > 48 * 1024 && contract_dmma2_smem(K, kDRbig, kDCbig) <= 200 * 1024)
    cudaFuncSetAttribute(contract_dmma2_kernel<kDRbig, kDCbig>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)contract_dmma2_smem(K, kDRbig, kDCbig));
  if (contract_smem_bytes(K) > 48 * 1024)
    cudaFuncSetAttribute(contract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)contract_smem_bytes(K));
  if (2 * sizeof(double) * K > 48 * 1024)
    cudaFuncSetAttribute(objective_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * sizeof(double) * K));
  {   // instance groups: two independent stage chains (graph branches) from 128 instances on, so that one
      // group's expectation overlaps the other's window stencil: cfg5 at 128 instances 70.3 -> 68.5 ms per step;
      // at 64 instances 36.4 vs 36.6 ms, at 4 groups 73.3 ms (bench.py --config cfg5).  All instances on the
      // window plan, >= 2 per group, the DMMA or Ozaki expectation.  ESDP_BATCH_GROUPS=G overrides (1: off).
    const char* e = getenv("ESDP_BATCH_GROUPS");
    const int G = e ? atoi(e) : (n >= 128 ? 2 : 1);
    if (G > 1 && b->nbrute == 0 && n >= 2 * G && !b->rank1 && (b->dmma || b->ozaki)) {
      b->groups = G;
      b->gstream.assign(G - 1, nullptr);
      b->gev.assign(2 * G, nullptr);
      for (cudaStream_t& x : b->gstream)
        if (cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking) != cudaSuccess) return bail(bfail(b, ESDP_E_CUDA, "group streams"));
      for (cudaEvent_t& x : b->gev)
        if (cudaEventCreateWithFlags(&x, cudaEventDisableTiming) != cudaSuccess) return bail(bfail(b, ESDP_E_CUDA, "group events"));
    }
  }
  {   // capture the whole batch backward once
    cudaGraph_t g = nullptr;
    BCUDA(b, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    esdp_status est = batch_enqueue(b, s);
    cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (est != ESDP_OK) { if (g) cudaGraphDestroy(g); return bail(est); }
    if (ce != cudaSuccess) return bail(bfail(b, ESDP_E_CUDA, "graph capture: %s", cudaGetErrorString(ce)));
    ce = cudaGraphInstantiate(&b->graph, g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) return bail(bfail(b, ESDP_E_CUDA, "graph instantiate: %s", cudaGetErrorString(ce)));
  }
#undef BTRY
  *out = b;
  return ESDP_OK;
}

esdp_status esdp_batch_dims(const esdp_batch* b, int32_t* n, int32_t* T, int32_t* S, int32_t* K, int32_t* A) {
  if (!b) return ESDP_E_STATE;
  if (n) *n = b->n;
  if (T) *T = b->T;
  if (S) *S = b->S;
  if (K) *K = b->K;
  if (A) for (int m = 0; m < b->n; ++m) A[m] = b->inst[m]->A;
  return ESDP_OK;
}

esdp_status esdp_batch_backward_async(esdp_batch* b, void* stream) {
  if (!b) return ESDP_E_STATE;
  cudaStream_t s = stream ? (cudaStream_t)stream : b->stream;
  BCUDA(b, cudaGraphLaunch(b->graph, s));
  b->solved = true;
  return ESDP_OK;
}

esdp_status esdp_batch_objective(esdp_batch* b, double* J) {
  if (!b || !J) return ESDP_E_STATE;
  if (!b->solved) return bfail(b, ESDP_E_STATE, "no backward pass has run");
  BCUDA(b, cudaMemcpy(J, b->d_J, b->n * sizeof(double), cudaMemcpyDeviceToHost));
  return ESDP_OK;
}

esdp_status esdp_batch_backward(esdp_batch* b, void* stream, double* J) {
  if (!b) return ESDP_E_STATE;
  cudaStream_t s = stream ? (cudaStream_t)stream : b->stream;
  esdp_status st = esdp_batch_backward_async(b, s);
  if (st != ESDP_OK) return st;
  BCUDA(b, cudaStreamSynchronize(s));
  return J ? esdp_batch_objective(b, J) : ESDP_OK;
}

esdp_status esdp_batch_policy(esdp_batch* b, int32_t m, int32_t t, int16_t* pol) {
  if (!b || !pol) return ESDP_E_STATE;
  if (!b->solved) return bfail(b, ESDP_E_STATE, "no backward pass has run");
  if (m < 0 || m >= b->n || t < 1 || t > b->T) return bfail(b, ESDP_E_STATE, "instance %d / stage %d out of range", m, t);
  const size_t KS = (size_t)b->K * b->S;
  BCUDA(b, cudaMemcpy(pol, b->d_pol + ((size_t)m * b->T + (t - 1)) * KS, KS * sizeof(int16_t), cudaMemcpyDeviceToHost));
  return ESDP_OK;
}

esdp_status esdp_batch_value1(esdp_batch* b, int32_t m, double* V1) {
  if (!b || !V1) return ESDP_E_STATE;
  if (!b->solved) return bfail(b, ESDP_E_STATE, "no backward pass has run");
  if (m < 0 || m >= b->n) return bfail(b, ESDP_E_STATE, "instance %d out of range", m);
  const size_t NL = (size_t)b->n * b->ld;   // stage 1 lives in ping-pong slot 0
  BCUDA(b, cudaMemcpy2D(V1, b->S * sizeof(double), b->d_V + (size_t)m * b->ld, NL * sizeof(double), b->S * sizeof(double),
                        b->K, cudaMemcpyDeviceToHost));
  return ESDP_OK;
}

esdp_status esdp_batch_simulate_dev(esdp_batch* b, int64_t n_paths, uint64_t seed, double* out_dev, void* stream) {
  if (!b || !out_dev) return ESDP_E_STATE;
  if (!b->solved) return bfail(b, ESDP_E_STATE, "no backward pass has run");
  if (n_paths < 1) return bfail(b, ESDP_E_STATE, "n_paths must be >= 1");
  cudaStream_t s = stream ? (cudaStream_t)stream : b->stream;
  int amax = 0;
  for (esdp_ctx* c : b->inst) amax = std::max(amax, c->A);
  const size_t sm = sim_smem_bytes(amax);
  if (sm > 48 * 1024) cudaFuncSetAttribute(simulate_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  simulate_batch_kernel<<<dim3((unsigned)((n_paths + 127) / 128), b->n), 128, sm, s>>>(b->d_bi, n_paths, seed, out_dev);
  BCUDA(b, cudaGetLastError());
  return ESDP_OK;
}

esdp_status esdp_batch_load_async(esdp_batch* b, const double* lambda, const double* P, const double* pi, void* stream) {
  if (!b || !lambda || !pi || (!b->rank1 && b->T > 1 && !P)) return b ? bfail(b, ESDP_E_STATE, "null input") : ESDP_E_STATE;
  esdp_ctx* c0 = b->inst[0];
  const esdp_status st = validate_data(c0, lambda, P, pi, nullptr);
  if (st != ESDP_OK) return bfail(b, st, "%s", c0->err.c_str());
  const size_t T = b->T, K = b->K;
  std::vector<int> tab, src;
  if (!b->rank1 && T > 1) dedupe_slices(P, (int)T - 1, (int)K, tab, src);
  const size_t rows = b->rank1 ? T : src.size() * K;
  if (rows > b->ntab_cap)
    return bfail(b, ESDP_E_STATE, "the new P has %zu distinct stage slices; the batch was built for %zu", src.size(), b->ntab_cap / K);
  cudaStream_t s = stream ? (cudaStream_t)stream : b->stream;
  BCUDA(b, cudaMemcpyAsync(b->d_lambda, lambda, T * K * sizeof(double), cudaMemcpyHostToDevice, s));
  if (b->rank1) {
    BCUDA(b, cudaMemcpyAsync(b->d_pi, pi, T * K * sizeof(double), cudaMemcpyHostToDevice, s));
    launch_cdf(b->d_pi, nullptr, (int64_t)T, (int)K, b->gbits, b->d_cdf, b->d_guide, s);
  } else {
    BCUDA(b, cudaMemcpyAsync(b->d_pi, pi, K * sizeof(double), cudaMemcpyHostToDevice, s));
    if (T > 1) {
      BCUDA(b, cudaMemcpyAsync(b->d_P, P, (T - 1) * K * K * sizeof(double), cudaMemcpyHostToDevice, s));
      BCUDA(b, cudaMemcpyAsync(b->d_tab, tab.data(), tab.size() * sizeof(int), cudaMemcpyHostToDevice, s));
      BCUDA(b, cudaMemcpyAsync(b->d_src, src.data(), src.size() * sizeof(int), cudaMemcpyHostToDevice, s));
      launch_cdf(b->d_P, b->d_src, (int64_t)rows, (int)K, b->gbits, b->d_cdf, b->d_guide, s);
    }
  }
  launch_cdf(b->d_pi, nullptr, 1, (int)K, b->g_max, b->d_cdf1, b->d_guide1, s);
  BCUDA(b, cudaGetLastError());
  return ESDP_OK;   // tab / src are pageable: cudaMemcpyAsync has staged them before returning
}

esdp_status esdp_batch_plan(const esdp_batch* b, int32_t* contraction) {
  if (!b || !contraction) return ESDP_E_CONFIG;
  *contraction = b->ozaki ? 2 : b->dmma ? 0 : 1;
  return ESDP_OK;
}

esdp_status esdp_expectation_dev(const double* P_dev, const double* V_dev, double* W_dev, int32_t rows, int32_t K,
                                 int64_t ncols, int64_t ldv, int64_t ldw, int32_t method, void* stream) {
  g_create_error.clear();
  if (!P_dev || !V_dev || !W_dev || rows < 1 || K < 1 || ncols < 1 || ldv < ncols || ldw < ncols)
    return bfail(nullptr, ESDP_E_CONFIG, "esdp_expectation_dev: null buffer or bad size / stride");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (method == 1) {
    if (rows > kOzM || K > kOzK) return bfail(nullptr, ESDP_E_CONFIG, "esdp_expectation_dev: Ozaki needs rows, K <= 128");
    e = launch_ozaki(P_dev, V_dev, W_dev, rows, K, (long long)ncols, (long long)ldv, (long long)ldw, s, false);
  } else if (method == 0) {
    if (ldv != ldw || ldv > INT32_MAX) return bfail(nullptr, ESDP_E_CONFIG, "esdp_expectation_dev: method 0 needs ldv == ldw < 2^31");
    if (const int d3 = dmma_probe_mismatches() == 0 ? use_dmma3(rows, ncols, K) : 0) {
      e = launch_dmma3(d3, P_dev, V_dev, W_dev, rows, K, (int)ncols, (int)ldv, s, false);
    } else {
      if (contract_smem_bytes(K) > 227 * 1024) return bfail(nullptr, ESDP_E_CONFIG, "esdp_expectation_dev: K too large");
      if (contract_smem_bytes(K) > 48 * 1024)
        cudaFuncSetAttribute(contract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)contract_smem_bytes(K));
      dim3 grid((unsigned)((ncols + kColsC - 1) / kColsC), (rows + kRowsC - 1) / kRowsC);
      e = launch(contract_kernel, grid, dim3(kThreadsC), contract_smem_bytes(K), s, false, P_dev, V_dev, W_dev, rows, K,
                 (int)ncols, (int)ldv);
    }
  } else {
    return bfail(nullptr, ESDP_E_CONFIG, "esdp_expectation_dev: method must be 0 or 1");
  }
  if (e != cudaSuccess) return bfail(nullptr, ESDP_E_CUDA, "esdp_expectation_dev: %s", cudaGetErrorString(e));
  return ESDP_OK;
}

esdp_status esdp_batch_kernel_time(esdp_batch* b, int32_t what, int32_t reps, double* us_per_launch) {
  // Diagnostic: warm back-to-back launches of stage T-1's expectation (what = 0), window stencil (1) or
  // brute-force stencil (2) of the batch, captured in a graph, CUDA events; needs a completed backward (its buffers are the inputs)
  if (!b || !us_per_launch || reps < 1) return ESDP_E_STATE;
  if (!b->solved) return bfail(b, ESDP_E_STATE, "no backward pass has run");
  if (b->T < 2) return bfail(b, ESDP_E_STATE, "needs T >= 2");
  cudaStream_t s = b->stream;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  BCUDA(b, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int r = 0; r < reps; ++r) {
    if ((what == 1 && b->nwin == 0) || (what == 2 && b->nbrute == 0) || what < 0 || what > 2) {
      cudaStreamEndCapture(s, &g); if (g) cudaGraphDestroy(g);
      return bfail(b, ESDP_E_STATE, "no kernel of kind %d in this batch", what);
    }
    const cudaError_t le = batch_stage_kernel(b, b->T - 1, what, s, false);
    if (le != cudaSuccess) { cudaStreamEndCapture(s, &g); if (g) cudaGraphDestroy(g); return bfail(b, ESDP_E_CUDA, "%s", cudaGetErrorString(le)); }
  }
  cudaError_t ce = cudaStreamEndCapture(s, &g);
  if (ce == cudaSuccess) ce = cudaGraphInstantiate(&ge, g, 0);
  if (g) cudaGraphDestroy(g);
  if (ce != cudaSuccess) return bfail(b, ESDP_E_CUDA, "kernel-time graph: %s", cudaGetErrorString(ce));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(e0, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  ce = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  cudaGraphExecDestroy(ge);
  if (ce != cudaSuccess) return bfail(b, ESDP_E_CUDA, "kernel-time run: %s", cudaGetErrorString(ce));
  *us_per_launch = 1e3 * ms / reps;
  return ESDP_OK;
}

esdp_status esdp_batch_launch_count(const esdp_batch* b, int64_t* n) {
  if (!b || !n) return ESDP_E_STATE;
  *n = b->launches;
  return ESDP_OK;
}

void esdp_batch_destroy(esdp_batch* b) {
  if (!b) return;
  batch_free(b);
  delete b;
}

const char* esdp_batch_last_error(const esdp_batch* b) { return b ? b->err.c_str() : g_create_error.c_str(); }



}  // extern "C"

#ifdef ESDP_WIN_TRACE
// diagnostic (make -B EXTRA=-DESDP_WIN_TRACE): per-block phase marks of the last window-stencil launch
extern "C" esdp_status esdp_win_trace(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, esdp::g_ktrace, sizeof(esdp::g_ktrace)) == cudaSuccess ? ESDP_OK : ESDP_E_CUDA;
}
#endif
