// simmodes.cuh -- the other two forward-simulation modes of a7 (SURVEY §8(a) "take a = pol_t[k][i] (or
// clear the bid)", §8(c) step 7 physical mode; R25/R26).  One thread per path, the same
// Philox4x32-10 draws as the lottery kernel:
//   physical    real SoC s (from s0): every stage re-optimises over all actions with
//               cand = payoff + W_t(s + F(p_a)) interpolated at the off-grid index (Alg. 1 line 7's
//               formula), smallest maximising index; s <- s + F(p_a*), snapped to the grid within 1e-9;
//   clear_bids  grid state i with lottery moves: the action is the stage's bid curve at (t, i, k)
//               (monotone chain, Eqs. 7-12, as bidcurve_kernel) cleared at lambda_{t,k} (merit order,
//               P:305; the largest j with j == 0 or price_{j-1} <= lambda).
// Both need W_t of every stage (ESDP_KEEP_VALUES).
#pragma once
#include "kernels.cuh"

namespace esdp {

struct SimModeParams {
  SimParams base;        // tables, cdf/guide, lambda, pol (unused here), initial state
  const double* W;       // [T][wrows][ld]
  const double* F;       // [A] SoC change of each action (Eq. 2), energy units
  const double* omw;     // [A] 1 - w_a
  int16_t* stack;        // clear_bids: [n_paths][A] hull stacks (vertex-major per path: path + j * n)
  const int16_t* schedule;  // fixed: [T] actions
  int16_t* actions;      // nullable: [T][n_paths] chosen actions
  int mode, wrows, ld;
  double delta, s0;
};

constexpr int kSimModeThreads = 128;

inline size_t simmode_smem_bytes(int A) { return (size_t)A * (5 * sizeof(double) + sizeof(int)) + 16; }

__global__ void __launch_bounds__(kSimModeThreads) simulate_mode_kernel(SimModeParams mp, int64_t n, uint64_t seed,
                                                                        double* __restrict__ out) {
  extern __shared__ __align__(16) double msm[];
  const SimParams& sp = mp.base;
  const int A = sp.A;
  double* s_act = msm;
  double* s_w = s_act + A;
  double* s_omw = s_w + A;
  double* s_g = s_omw + A;
  double* s_F = s_g + A;
  int* s_ow = (int*)(s_F + A);                       // 2 o_a + [w_a != 0]
  for (int a = threadIdx.x; a < A; a += blockDim.x) {
    const double wa = sp.w[a];
    s_act[a] = sp.act[a]; s_w[a] = wa; s_omw[a] = mp.omw[a]; s_F[a] = mp.F[a];
    s_g[a] = sp.kind == 1 ? sp.g[a] : 0.0;
    s_ow[a] = 2 * sp.off[a] + (wa != 0.0 ? 1 : 0);
  }
  __syncthreads();
  const int64_t path = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (path >= n) return;
  const int S = sp.S, K = sp.K, T = sp.T;
  auto pay_of = [&](int t, int k, int a) -> double {   // R14: the payoff is formed first
    if (sp.kind == 2) return __ldg(sp.g + ((size_t)(t - 1) * K + k) * A + a);
    double p = __dmul_rn(__ldg(sp.lambda + (size_t)(t - 1) * K + k), s_act[a]);
    if (sp.kind == 1) p = __dsub_rn(p, s_g[a]);
    return p;
  };
  double u1, u2;
  uint64_t m1, m2;
  sim_uniforms(seed, path, 0, u1, u2, m1, m2);
  int k = cdf_sample(sp.cdf1, sp.guide1, sp.gs1, m1, u1);
  int i = sp.on_grid ? sp.f0 : sp.f0 + (u2 < sp.w0 ? 1 : 0);
  double s = mp.s0;                                    // physical mode: the real SoC, from s0 itself
  double profit = 0.0;
  int k_prev = k;                                      // self-scheduled: last observed state and price
  double lam_prev = __ldg(sp.lambda + k);              // stage 1's lag: its own price (R27)
  const double sbar_idx = (double)(S - 1);
  const double tol = 1e-9;
  for (int t = 1; t <= T; ++t) {
    sim_uniforms(seed, path, t, u1, u2, m1, m2);
    const int wrow = sp.rank1 ? 0 : (mp.mode == 3 ? k_prev : k);   // self: persistence forecast of k_t
    const double* Wrow = mp.W + ((size_t)(t - 1) * mp.wrows + wrow) * mp.ld;
    const double lam = __ldg(sp.lambda + (size_t)(t - 1) * K + k);
    int a_sel = 0;
    if (mp.mode == 4) {
      a_sel = __ldg(mp.schedule + (t - 1));
    } else if (mp.mode == 1 || mp.mode == 3) {
      double best = -INFINITY, best_s = s;
      int best_a = -1;
      for (int a = 0; a < A; ++a) {
        double sn = __dadd_rn(s, s_F[a]);
        const double x = __ddiv_rn(sn, mp.delta);
        if (x < -tol || x > sbar_idx + tol) continue;
        const double r = rint(x);
        double wint;
        if (fabs(__dsub_rn(x, r)) <= tol) {
          wint = __ldcg(Wrow + (int)r);
          sn = __dmul_rn(r, mp.delta);
        } else {
          const double f = floor(x);
          const double w = __dsub_rn(x, f);
          const int fi = (int)f;
          wint = __dadd_rn(__dmul_rn(__dsub_rn(1.0, w), __ldcg(Wrow + fi)), __dmul_rn(w, __ldcg(Wrow + fi + 1)));
        }
        double pay;
        if (mp.mode == 3) {            // decided at the lagged price (linear payoffs only)
          pay = __dmul_rn(lam_prev, s_act[a]);
          if (sp.kind == 1) pay = __dsub_rn(pay, s_g[a]);
        } else {
          pay = pay_of(t, k, a);
        }
        const double cand = __dadd_rn(pay, wint);
        if (cand > best) { best = cand; best_a = a; best_s = sn; }
      }
      a_sel = best_a;
      s = best_s;
    } else {
      // feasible actions of row i: one interval [a_lo, a_hi] (as bidcurve_kernel)
      int lo = 0, hi = A;
      while (lo < hi) { const int m = (lo + hi) >> 1; if ((s_ow[m] >> 1) < -i) hi = m; else lo = m + 1; }
      const int a_hi = lo - 1;
      lo = 0; hi = A;
      while (lo < hi) { const int m = (lo + hi) >> 1; const int ow = s_ow[m]; if ((ow >> 1) + (ow & 1) <= S - 1 - i) hi = m; else lo = m + 1; }
      const int a_lo = lo;
      const double* Wi = Wrow + i;
      auto u_of = [&](int a) -> double {               // Eq. 7 point value u_a = Wint - g_a (R13)
        const int ow = s_ow[a];
        const double* wp = Wi + (ow >> 1);
        double u = __ldcg(wp);
        if (ow & 1) u = __dadd_rn(__dmul_rn(s_omw[a], u), __dmul_rn(s_w[a], __ldcg(wp + 1)));
        if (sp.kind == 1) u = __dsub_rn(u, s_g[a]);
        return u;
      };
      int16_t* st = mp.stack + path;
      auto st_set = [&](int j, int a) { st[(size_t)j * n] = (int16_t)a; };
      auto st_get = [&](int j) -> int { return st[(size_t)j * n]; };
      int nh = 0, ao = -1, ab = -1;
      double uo = 0.0, ub = 0.0, po = 0.0, pb = 0.0;
      for (int a = a_lo; a <= a_hi; ++a) {
        const double u = u_of(a), pc = s_act[a];
        while (nh >= 2) {
          const double cr = __dsub_rn(__dmul_rn(__dsub_rn(pb, po), __dsub_rn(u, uo)),
                                      __dmul_rn(__dsub_rn(ub, uo), __dsub_rn(pc, po)));
          if (cr < 0.0) break;
          --nh;
          ab = ao; ub = uo; pb = po;
          if (nh >= 2) { ao = st_get(nh - 2); uo = u_of(ao); po = s_act[ao]; }
        }
        st_set(nh, a);
        if (nh >= 1) { ao = ab; uo = ub; po = pb; }
        ab = a; ub = u; pb = pc;
        ++nh;
      }
      // clearing: walk the vertices with the repaired prices; stop at the first price above lambda
      int a_prev = st_get(0);
      double u_prev = u_of(a_prev), p_prev = s_act[a_prev], prev_price = 0.0;
      a_sel = a_prev;
      for (int j = 1; j < nh; ++j) {
        const int a = st_get(j);
        const double u = u_of(a), pc = s_act[a];
        double pj = -__ddiv_rn(__dsub_rn(u, u_prev), __dsub_rn(pc, p_prev));
        if (j > 1 && pj < prev_price) pj = prev_price;
        if (!(pj <= lam)) break;                       // price_{j-1} > lambda: vertex j - 1 clears
        a_sel = a;
        prev_price = pj; u_prev = u; p_prev = pc;
      }
    }
    if (mp.actions) mp.actions[(size_t)(t - 1) * n + path] = (int16_t)a_sel;
    profit = __dadd_rn(profit, pay_of(t, k, a_sel));   // settled at the realised price
    lam_prev = lam;
    k_prev = k;
    if (mp.mode == 2) {
      const double wa = s_w[a_sel];
      i = i + (s_ow[a_sel] >> 1) + ((wa > 0.0 && u1 < wa) ? 1 : 0);
    }
    if (t < T) {
      const size_t row = sim_row(sp, t, k);
      k = cdf_sample(sp.cdf + row * K, sp.guide + (row << (53 - sp.gs)), sp.gs, m2, u2);
    }
  }
  out[path] = profit;
}

}  // namespace esdp
