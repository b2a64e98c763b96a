/*
 * esdp_oracle.c -- plain FP64 CPU oracle.  TEST INFRASTRUCTURE ONLY (see esdp_oracle.h).
 *
 * Written from the paper, /root/reference/PAPER.md (cited "P:NNN"), in the paper's order,
 * with the readings R1..R24 listed in DESIGN.md §3.  No blocking,
 * fusion or reordering: every loop is the definition written out.
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fopenmp -fPIC -shared (no -ffast-math).
 */
#include "esdp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_MAX_A 8191
#define GRID_TOL 1e-9 /* R6/R7: tolerance on integral quotients, index units */

/* Eq. 2, with eta_c on the charge side and eta_d on the discharge side (D2):
 * F(p) = -p/eta_d for p >= 0 (discharge), -eta_c p for p < 0 (charge). */
static double transition_F(double p, double eta_c, double eta_d) {
  if (p >= 0.0) return -(p / eta_d);
  return -(eta_c * p);
}

static int is_finite(double x) { return isfinite(x) ? 1 : 0; }

/* Eq. 10: n^c = ceil(pbar eta / delta), n^d = ceil(pbar / (delta eta)),
 * with the R6 guard (subtract 1e-9 before ceil so an integral quotient stays integral). */
static void paper_counts(const ref_problem* pr, int64_t* nc, int64_t* nd) {
  double qc = pr->pbar * pr->eta_c / pr->delta;
  double qd = pr->pbar / (pr->delta * pr->eta_d);
  *nc = (int64_t)ceil(qc - GRID_TOL);
  *nd = (int64_t)ceil(qd - GRID_TOL);
  if (*nc < 1) *nc = 1;
  if (*nd < 1) *nd = 1;
}

/* Eq. 10 vector p_hat = [-pbar, ..., -2 delta/eta, -delta/eta, 0, delta eta, 2 delta eta, ..., pbar]
 * (P:191-201): the last multiple on each side is clamped to pbar (R6). */
static void paper_actions(const ref_problem* pr, int64_t nc, int64_t nd, double* out) {
  int64_t idx = 0;
  for (int64_t j = nc; j >= 1; --j) {
    double x = (double)j * pr->delta / pr->eta_c;
    out[idx++] = -(x < pr->pbar ? x : pr->pbar);
  }
  out[idx++] = 0.0;
  for (int64_t j = 1; j <= nd; ++j) {
    double x = (double)j * pr->delta * pr->eta_d;
    out[idx++] = (x < pr->pbar ? x : pr->pbar);
  }
}

static int check_simplex(const double* q, int32_t K) {
  double s = 0.0;
  for (int32_t j = 0; j < K; ++j) {
    if (!is_finite(q[j]) || q[j] < 0.0) return 0;
    s += q[j];
  }
  return fabs(s - 1.0) <= 1e-9;
}

int ref_dims(const ref_problem* pr, int32_t* S_out, int32_t* A_out) {
  if (!pr) return REF_E_CONFIG;
  if (pr->T < 1 || pr->K < 1) return REF_E_CONFIG;
  if (!(is_finite(pr->pbar) && pr->pbar > 0.0)) return REF_E_CONFIG;
  if (!(is_finite(pr->sbar) && pr->sbar > 0.0)) return REF_E_CONFIG;
  if (!(is_finite(pr->delta) && pr->delta > 0.0)) return REF_E_CONFIG;
  if (!(pr->eta_c > 0.0 && pr->eta_c <= 1.0)) return REF_E_CONFIG;
  if (!(pr->eta_d > 0.0 && pr->eta_d <= 1.0)) return REF_E_CONFIG;
  if (!(is_finite(pr->s0) && pr->s0 >= 0.0 && pr->s0 <= pr->sbar)) return REF_E_CONFIG;
  /* n^s = sbar/delta must be a natural number (no silent rounding, R6). */
  double ns = pr->sbar / pr->delta;
  double r = nearbyint(ns);
  if (!(fabs(ns - r) <= GRID_TOL * (ns > 1.0 ? ns : 1.0)) || r < 1.0 || r > 1e8) return REF_E_CONFIG;
  int64_t S = (int64_t)r + 1;
  int64_t A;
  if (pr->A == 0) {
    int64_t nc, nd;
    paper_counts(pr, &nc, &nd);
    A = nc + nd + 1;
    if (A > ORACLE_MAX_A) return REF_E_CONFIG;
    double* tmp = (double*)malloc(sizeof(double) * (size_t)A);
    if (!tmp) return REF_E_INTERNAL;
    paper_actions(pr, nc, nd, tmp);
    int ok = 1;
    for (int64_t a = 1; a < A; ++a)
      if (!(tmp[a] > tmp[a - 1])) ok = 0;
    free(tmp);
    if (!ok) return REF_E_CONFIG;
  } else {
    if (pr->A < 0 || pr->A > ORACLE_MAX_A || !pr->actions) return REF_E_CONFIG;
    A = pr->A;
    int zeros = 0;
    for (int64_t a = 0; a < A; ++a) {
      double p = pr->actions[a];
      if (!is_finite(p) || fabs(p) > pr->pbar) return REF_E_CONFIG;
      if (p == 0.0) zeros++;
      if (a > 0 && !(p > pr->actions[a - 1])) return REF_E_CONFIG;
    }
    if (zeros != 1) return REF_E_CONFIG;
  }
  if (pr->payoff_kind < 0 || pr->payoff_kind > 2) return REF_E_CONFIG;
  if (pr->payoff_kind != REF_PAYOFF_LINEAR && !pr->g) return REF_E_CONFIG;
  if (!pr->lambda || !pr->pi) return REF_E_CONFIG;
  /* data checks */
  for (int64_t j = 0; j < (int64_t)pr->T * pr->K; ++j)
    if (!is_finite(pr->lambda[j])) return REF_E_DATA;
  if (pr->payoff_kind == REF_PAYOFF_LINEAR_MINUS_G) {
    for (int64_t a = 0; a < A; ++a)
      if (!is_finite(pr->g[a])) return REF_E_DATA;
  } else if (pr->payoff_kind == REF_PAYOFF_TABLE) {
    for (int64_t j = 0; j < (int64_t)pr->T * pr->K * A; ++j)
      if (!is_finite(pr->g[j])) return REF_E_DATA;
  }
  if (pr->P) {
    for (int64_t r2 = 0; r2 < (int64_t)(pr->T - 1) * pr->K; ++r2)
      if (!check_simplex(pr->P + r2 * pr->K, pr->K)) return REF_E_DATA;
    if (!check_simplex(pr->pi, pr->K)) return REF_E_DATA;
  } else {
    for (int32_t t = 0; t < pr->T; ++t)
      if (!check_simplex(pr->pi + (int64_t)t * pr->K, pr->K)) return REF_E_DATA;
  }
  if (S_out) *S_out = (int32_t)S;
  if (A_out) *A_out = (int32_t)A;
  return REF_OK;
}

int ref_actions(const ref_problem* pr, double* actions) {
  int32_t S, A;
  int rc = ref_dims(pr, &S, &A);
  if (rc) return rc;
  if (pr->A == 0) {
    int64_t nc, nd;
    paper_counts(pr, &nc, &nd);
    paper_actions(pr, nc, nd, actions);
  } else {
    memcpy(actions, pr->actions, sizeof(double) * (size_t)A);
  }
  return REF_OK;
}

/* Alg. 1 lines 2-5 with R1 (clamp), R2 (sigma > sbar), R4 (0/0 -> weight 0):
 * sigma_{i,a} = s_i + F(p_a); in index units e_a = F(p_a)/delta, so the next-state proxy is
 * z = i + e_a, z^- = i + o_a, z^+ = z^- + 1 (when w_a > 0), b = w_a.  The interior actions of
 * Eq. 10 recombine exactly: e_a is integral and w_a = 0. */
int ref_tables(const ref_problem* pr, int32_t* off, double* w, double* omw, int32_t* ilo, int32_t* ihi) {
  int32_t S, A;
  int rc = ref_dims(pr, &S, &A);
  if (rc) return rc;
  double* act = (double*)malloc(sizeof(double) * (size_t)A);
  if (!act) return REF_E_INTERNAL;
  ref_actions(pr, act);
  for (int32_t a = 0; a < A; ++a) {
    double e = transition_F(act[a], pr->eta_c, pr->eta_d) / pr->delta;
    double r = nearbyint(e);
    if (fabs(e - r) <= GRID_TOL) {
      off[a] = (int32_t)r;
      w[a] = 0.0;
    } else {
      double f = floor(e);
      off[a] = (int32_t)f;
      w[a] = e - f;
    }
    omw[a] = 1.0 - w[a];
    /* R7 / Alg. 1 line 8: row i is feasible iff 0 <= i + e_a <= S-1 (tolerance 1e-9). */
    double lo = ceil(-e - GRID_TOL);
    double hi = floor((double)(S - 1) - e + GRID_TOL);
    ilo[a] = lo > 0.0 ? (int32_t)lo : 0;
    ihi[a] = hi < (double)(S - 1) ? (int32_t)hi : S - 1;
  }
  free(act);
  return REF_OK;
}

/* payoff(lambda_{t,k}, p_a): Alg. 1 line 9's payoff matrix p_hat lambda_hat^T, with the
 * general payoff of D3: lambda p - g(p) (LINEAR_MINUS_G) or a table Pi[t][k][a] (TABLE).
 * Association (R14): the payoff is formed first, then added to the continuation. */
static double payoff(const ref_problem* pr, int32_t A, const double* act, int32_t t, int32_t k, int32_t a) {
  if (pr->payoff_kind == REF_PAYOFF_TABLE) return pr->g[((int64_t)(t - 1) * pr->K + k) * A + a];
  double lam = pr->lambda[(int64_t)(t - 1) * pr->K + k];
  double gv = pr->payoff_kind == REF_PAYOFF_LINEAR_MINUS_G ? pr->g[a] : 0.0;
  return (lam * act[a]) - gv;
}

/* Alg. 1 line 7: (1-b) V[z^-] + b V[z^+]; an integral offset reads one entry. */
static double interp(const double* row, int32_t i, int32_t o, double w, double omw) {
  if (w == 0.0) return row[i + o];
  return (omw * row[i + o]) + (w * row[i + o + 1]);
}

/* One stage t of the backward induction for the price-state rows [k_lo, k_hi) (Alg. 1 lines 7-11,
 * P:268-277, Markov form): W_t rows = P_t V_{t+1} (W_T = 0), then V_t, pol_t rows by the max-plus
 * reduction.  Vnext = V_{t+1} [K][S] (all rows; unused at t = T).  Wt, Vt, polt: [k_hi - k_lo][S]. */
static int stage_rows(const ref_problem* pr, int32_t S, int32_t A, const double* act, const int32_t* off,
                      const double* w, const double* omw, const int32_t* ilo, const int32_t* ihi, int32_t t,
                      int32_t k_lo, int32_t k_hi, int32_t nthreads, const double* Vnext, double* Wt, double* Vt,
                      int16_t* polt) {
  const int32_t T = pr->T, K = pr->K;
  int internal_error = 0;
  /* Expectation (Alg. 1 line 11; Eq. 6) in Markov form W_t = P_t V_{t+1} (D1): canonical
   * ascending-k' fma chain (R15).  Rank-1: P_t[k][k'] = pi_{t+1}[k'].  Base case W_T = 0. */
#pragma omp parallel for num_threads(nthreads) schedule(static)
  for (int32_t k = k_lo; k < k_hi; ++k) {
    double* Wrow = Wt + (int64_t)(k - k_lo) * S;
    if (t == T) {
      for (int32_t i = 0; i < S; ++i) Wrow[i] = 0.0;
      continue;
    }
    const double* Prow = pr->P ? pr->P + ((int64_t)(t - 1) * K + k) * K : pr->pi + (int64_t)t * K;
    for (int32_t i = 0; i < S; ++i) {
      double acc = 0.0;
      for (int32_t kp = 0; kp < K; ++kp) acc = fma(Prow[kp], Vnext[(int64_t)kp * S + i], acc);
      Wrow[i] = acc;
    }
  }
  /* Alg. 1 lines 7-10, Eq. 5: V_t(s_i,k) = max over feasible a of
   * payoff(lambda_{t,k}, p_a) + Wint_t(i, a, k); argmax = smallest maximizing a (R8). */
#pragma omp parallel for num_threads(nthreads) schedule(static)
  for (int32_t k = k_lo; k < k_hi; ++k) {
    const double* Wrow = Wt + (int64_t)(k - k_lo) * S;
    for (int32_t i = 0; i < S; ++i) {
      double best = -INFINITY;
      int32_t arg = -1;
      for (int32_t a = 0; a < A; ++a) {
        if (i < ilo[a] || i > ihi[a]) continue; /* Alg. 1 line 8: infeasible -> -inf */
        double cand = payoff(pr, A, act, t, k, a) + interp(Wrow, i, off[a], w[a], omw[a]);
        if (cand > best) {
          best = cand;
          arg = a;
        }
      }
      if (arg < 0) {
#pragma omp atomic write
        internal_error = 1;
      }
      Vt[(int64_t)(k - k_lo) * S + i] = best;
      polt[(int64_t)(k - k_lo) * S + i] = (int16_t)arg;
    }
  }
  return internal_error ? REF_E_INTERNAL : REF_OK;
}

typedef struct {
  double* act; int32_t* off; double* w; double* omw; int32_t* ilo; int32_t* ihi;
} ref_tabs;

static int tabs_make(const ref_problem* pr, int32_t A, ref_tabs* tb) {
  tb->act = (double*)malloc(sizeof(double) * (size_t)A);
  tb->off = (int32_t*)malloc(sizeof(int32_t) * (size_t)A);
  tb->w = (double*)malloc(sizeof(double) * (size_t)A);
  tb->omw = (double*)malloc(sizeof(double) * (size_t)A);
  tb->ilo = (int32_t*)malloc(sizeof(int32_t) * (size_t)A);
  tb->ihi = (int32_t*)malloc(sizeof(int32_t) * (size_t)A);
  if (!tb->act || !tb->off || !tb->w || !tb->omw || !tb->ilo || !tb->ihi) return REF_E_INTERNAL;
  ref_actions(pr, tb->act);
  ref_tables(pr, tb->off, tb->w, tb->omw, tb->ilo, tb->ihi);
  return REF_OK;
}

static void tabs_free(ref_tabs* tb) {
  free(tb->act); free(tb->off); free(tb->w); free(tb->omw); free(tb->ilo); free(tb->ihi);
}

int ref_stage(const ref_problem* pr, int32_t t, int32_t k_lo, int32_t k_hi, int32_t nthreads, const double* Vnext,
              double* Wt, double* Vt, int16_t* polt) {
  int32_t S, A;
  int rc = ref_dims(pr, &S, &A);
  if (rc) return rc;
  if (t < 1 || t > pr->T || k_lo < 0 || k_hi > pr->K || k_lo > k_hi || (t < pr->T && !Vnext)) return REF_E_STATE;
  ref_tabs tb;
  rc = tabs_make(pr, A, &tb);
  if (!rc) rc = stage_rows(pr, S, A, tb.act, tb.off, tb.w, tb.omw, tb.ilo, tb.ihi, t, k_lo, k_hi, nthreads, Vnext, Wt, Vt, polt);
  tabs_free(&tb);
  return rc;
}

int ref_objective(const ref_problem* pr, const double* V1, double* J) {
  int32_t S, A;
  int rc = ref_dims(pr, &S, &A);
  if (rc) return rc;
  /* Eq. 6 at t = 0: J = E[V_1(s0, k_1)], k_1 ~ pi_1 (R10/R11); s0 off-grid is
   * interpolated per k (R24). */
  const double* pi1 = pr->pi;
  double x = pr->s0 / pr->delta;
  double r = nearbyint(x);
  double acc = 0.0;
  for (int32_t k = 0; k < pr->K; ++k) {
    const double* row = V1 + (int64_t)k * S;
    double v;
    if (fabs(x - r) <= GRID_TOL) {
      v = row[(int32_t)r];
    } else {
      double f = floor(x);
      double w0 = x - f;
      v = ((1.0 - w0) * row[(int32_t)f]) + (w0 * row[(int32_t)f + 1]);
    }
    acc = fma(pi1[k], v, acc);
  }
  *J = acc;
  return REF_OK;
}

int ref_backward(const ref_problem* pr, int32_t t_stop, int32_t nthreads,
                 double* V, double* W, int16_t* pol, double* J) {
  int32_t S, A;
  int rc = ref_dims(pr, &S, &A);
  if (rc) return rc;
  const int32_t T = pr->T, K = pr->K;
  if (t_stop < 1 || t_stop > T) return REF_E_STATE;
  ref_tabs tb;
  rc = tabs_make(pr, A, &tb);
  const int64_t KS = (int64_t)K * S;
  /* Alg. 1 line 1: base case; R3: T iterations, t = T..1, every stage over all K rows. */
  for (int32_t t = T; t >= t_stop && !rc; --t)
    rc = stage_rows(pr, S, A, tb.act, tb.off, tb.w, tb.omw, tb.ilo, tb.ihi, t, 0, K, nthreads,
                    t < T ? V + (int64_t)t * KS : NULL, W + (int64_t)(t - 1) * KS, V + (int64_t)(t - 1) * KS,
                    pol + (int64_t)(t - 1) * KS);
  tabs_free(&tb);
  if (!rc && J && t_stop == 1) rc = ref_objective(pr, V, J);
  return rc;
}

int ref_bidcurve(const ref_problem* pr, const double* W, int32_t t, int32_t i, int32_t k,
                 int32_t cap, int32_t* nvert, int16_t* vert, double* q, double* price,
                 int32_t* n_repairs) {
  int32_t S, A;
  int rc = ref_dims(pr, &S, &A);
  if (rc) return rc;
  if (pr->payoff_kind == REF_PAYOFF_TABLE) return REF_E_STATE; /* R13 */
  if (t < 1 || t > pr->T || i < 0 || i >= S || k < 0 || k >= pr->K || cap < A) return REF_E_STATE;
  double* act = (double*)malloc(sizeof(double) * (size_t)A);
  int32_t* off = (int32_t*)malloc(sizeof(int32_t) * (size_t)A);
  double* w = (double*)malloc(sizeof(double) * (size_t)A);
  double* omw = (double*)malloc(sizeof(double) * (size_t)A);
  int32_t* ilo = (int32_t*)malloc(sizeof(int32_t) * (size_t)A);
  int32_t* ihi = (int32_t*)malloc(sizeof(int32_t) * (size_t)A);
  double* hu = (double*)malloc(sizeof(double) * (size_t)A);
  int32_t* ha = (int32_t*)malloc(sizeof(int32_t) * (size_t)A);
  ref_actions(pr, act);
  ref_tables(pr, off, w, omw, ilo, ihi);
  const double* Wrow = W + ((int64_t)(t - 1) * pr->K + k) * S;
  /* Eq. 7: U_t(p; s) = W_t(s + F(p)) on the feasible actions; the non-linear part
   * of the payoff (-g) belongs to the function being convexified (R13). */
  int32_t n = 0;
  for (int32_t a = 0; a < A; ++a) {
    if (i < ilo[a] || i > ihi[a]) continue;
    double gv = pr->payoff_kind == REF_PAYOFF_LINEAR_MINUS_G ? pr->g[a] : 0.0;
    double uc = interp(Wrow, i, off[a], w[a], omw[a]) - gv;
    double pc = act[a];
    /* hyp U~ = conv(hyp U), by the monotone-chain (Graham) scan over ascending p:
     * pop the last vertex b while (o, b, c) does not turn clockwise (cross >= 0 also drops
     * collinear points). */
    while (n >= 2) {
      double po = act[ha[n - 2]], uo = hu[n - 2];
      double pb = act[ha[n - 1]], ub = hu[n - 1];
      double cross = ((pb - po) * (uc - uo)) - ((ub - uo) * (pc - po));
      if (cross >= 0.0) n--;
      else break;
    }
    ha[n] = a;
    hu[n] = uc;
    n++;
  }
  /* Eq. 12: b~ = -dU~; segment price_j = -(u_{j+1} - u_j)/(p_{j+1} - p_j),
   * then a running max as the documented <= 1 ulp monotone repair (R20). */
  int32_t reps = 0;
  for (int32_t j = 0; j < n; ++j) {
    vert[j] = (int16_t)ha[j];
    q[j] = act[ha[j]];
  }
  for (int32_t j = 0; j + 1 < n; ++j) {
    double pj = -((hu[j + 1] - hu[j]) / (act[ha[j + 1]] - act[ha[j]]));
    if (j > 0 && pj < price[j - 1]) {
      pj = price[j - 1];
      reps++;
    }
    price[j] = pj;
  }
  *nvert = n;
  if (n_repairs) *n_repairs = reps;
  free(act); free(off); free(w); free(omw); free(ilo); free(ihi); free(hu); free(ha);
  return REF_OK;
}

int32_t ref_clear(int32_t nvert, const double* price, double lam) {
  int32_t j = 0;
  for (int32_t v = 1; v < nvert; ++v)
    if (price[v - 1] <= lam) j = v;
  return j;
}

/* Philox4x32-10: Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3",
 * SC'11.  Round: (L0,R0,L1,R1) -> (hi(M1 R1) ^ k0 ^ L1 ... ) in the Random123 form. */
void ref_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* R16/R17: counter = (path lo, path hi, t, 'ESDP'), key = (seed lo, seed hi); two uniforms
 * with 53 random bits each: u = ((x_a << 21) | (x_b >> 11)) * 2^-53. */
static void uniforms(uint64_t seed, int64_t path, int32_t t, double* u1, double* u2) {
  uint32_t ctr[4] = {(uint32_t)((uint64_t)path & 0xffffffffu), (uint32_t)((uint64_t)path >> 32),
                     (uint32_t)t, 0x45534450u};
  uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
  uint32_t x[4];
  ref_philox4x32_10(ctr, key, x);
  *u1 = (double)((((uint64_t)x[0]) << 21) | (x[1] >> 11)) * 0x1p-53;
  *u2 = (double)((((uint64_t)x[2]) << 21) | (x[3] >> 11)) * 0x1p-53;
}

/* first j with u < cdf[j]; the cdf is the running sum of q in ascending order, last entry 1. */
static int32_t sample_cdf(const double* q, int32_t K, double u) {
  double c = 0.0;
  for (int32_t j = 0; j < K; ++j) {
    c = c + q[j];
    if (j == K - 1) c = 1.0;
    if (u < c) return j;
  }
  return K - 1;
}

int ref_simulate(const ref_problem* pr, const int16_t* pol, int64_t n_paths, uint64_t seed,
                 double* per_path, double* mean, double* var) {
  int32_t S, A;
  int rc = ref_dims(pr, &S, &A);
  if (rc) return rc;
  if (n_paths < 1) return REF_E_STATE;
  const int32_t T = pr->T, K = pr->K;
  double* act = (double*)malloc(sizeof(double) * (size_t)A);
  int32_t* off = (int32_t*)malloc(sizeof(int32_t) * (size_t)A);
  double* w = (double*)malloc(sizeof(double) * (size_t)A);
  double* omw = (double*)malloc(sizeof(double) * (size_t)A);
  int32_t* ilo = (int32_t*)malloc(sizeof(int32_t) * (size_t)A);
  int32_t* ihi = (int32_t*)malloc(sizeof(int32_t) * (size_t)A);
  ref_actions(pr, act);
  ref_tables(pr, off, w, omw, ilo, ihi);
  const int64_t KS = (int64_t)K * S;
  double x0 = pr->s0 / pr->delta;
  double r0 = nearbyint(x0);
  int on_grid = fabs(x0 - r0) <= GRID_TOL;
  double f0 = floor(x0), w0 = x0 - f0;
  for (int64_t path = 0; path < n_paths; ++path) {
    double u1, u2;
    uniforms(seed, path, 0, &u1, &u2);
    int32_t k = sample_cdf(pr->pi, K, u1); /* k_1 ~ pi_1 (R11) */
    int32_t i = on_grid ? (int32_t)r0 : (int32_t)f0 + (u2 < w0 ? 1 : 0);
    double profit = 0.0;
    for (int32_t t = 1; t <= T; ++t) {
      uniforms(seed, path, t, &u1, &u2);
      int32_t a = pol[(int64_t)(t - 1) * KS + (int64_t)k * S + i];
      profit = profit + payoff(pr, A, act, t, k, a);
      /* lottery transition to the two neighbouring grid states (Alg. 1 line 7 weights). */
      i = i + off[a] + ((w[a] > 0.0 && u1 < w[a]) ? 1 : 0);
      if (t < T) {
        const double* q = pr->P ? pr->P + ((int64_t)(t - 1) * K + k) * K : pr->pi + (int64_t)t * K;
        k = sample_cdf(q, K, u2);
      }
    }
    per_path[path] = profit;
  }
  double s = 0.0;
  for (int64_t p = 0; p < n_paths; ++p) s += per_path[p];
  double m = s / (double)n_paths;
  double ss = 0.0;
  for (int64_t p = 0; p < n_paths; ++p) ss += (per_path[p] - m) * (per_path[p] - m);
  *mean = m;
  *var = n_paths > 1 ? ss / (double)(n_paths - 1) : 0.0;
  free(act); free(off); free(w); free(omw); free(ilo); free(ihi);
  return REF_OK;
}

/* Physical-mode decision at real SoC s (energy units), stage t, price state k, from row W_t[k] (R25):
 * every action a in ascending order, s' = s + F(p_a) (Eq. 2), feasible iff 0 <= s'/delta <= S-1 within
 * 1e-9 (Eq. 4 on the real state), cand = payoff + W_t(s') with Alg. 1 line 7's interpolation at the
 * off-grid index s'/delta; strict '>' keeps the smallest maximising index (R8). */
static int32_t physical_action_lam(const ref_problem* pr, int32_t S, int32_t A, const double* act,
                                   const double* Wrow, int32_t t, int32_t k, const double* lam_override, double s,
                                   double* s_next);

static int32_t physical_action(const ref_problem* pr, int32_t S, int32_t A, const double* act, const double* Wrow,
                               int32_t t, int32_t k, double s, double* s_next) {
  return physical_action_lam(pr, S, A, act, Wrow, t, k, NULL, s, s_next);
}

/* physical_action with the payoff formed at price *lam_override instead of lambda_{t,k} (linear payoffs). */
static int32_t physical_action_lam(const ref_problem* pr, int32_t S, int32_t A, const double* act,
                                   const double* Wrow, int32_t t, int32_t k, const double* lam_override, double s,
                                   double* s_next) {
  int32_t best_a = -1;
  double best = -INFINITY, best_s = s;
  for (int32_t a = 0; a < A; ++a) {
    double sn = s + transition_F(act[a], pr->eta_c, pr->eta_d);
    double x = sn / pr->delta;
    if (x < -GRID_TOL || x > (double)(S - 1) + GRID_TOL) continue;
    double r = nearbyint(x);
    double wint;
    if (fabs(x - r) <= GRID_TOL) {
      wint = Wrow[(int32_t)r];
      sn = r * pr->delta;                     /* snapped to the grid */
    } else {
      double f = floor(x);
      double w = x - f;
      wint = ((1.0 - w) * Wrow[(int32_t)f]) + (w * Wrow[(int32_t)f + 1]);
    }
    double pay;
    if (lam_override) {
      double gv = pr->payoff_kind == REF_PAYOFF_LINEAR_MINUS_G ? pr->g[a] : 0.0;
      pay = (*lam_override * act[a]) - gv;
    } else {
      pay = payoff(pr, A, act, t, k, a);
    }
    double cand = pay + wint;
    if (cand > best) { best = cand; best_a = a; best_s = sn; }
  }
  *s_next = best_s;
  return best_a;
}

int ref_simulate_mode(const ref_problem* pr, const int16_t* pol, const double* W, int32_t mode, int64_t n_paths,
                      uint64_t seed, double* per_path, double* mean, double* var) {
  if (mode == REF_SIM_LOTTERY) return ref_simulate(pr, pol, n_paths, seed, per_path, mean, var);
  int32_t S, A;
  int rc = ref_dims(pr, &S, &A);
  if (rc) return rc;
  if (n_paths < 1 || !W || (mode != REF_SIM_PHYSICAL && mode != REF_SIM_CLEAR_BIDS)) return REF_E_STATE;
  if (mode == REF_SIM_CLEAR_BIDS && pr->payoff_kind == REF_PAYOFF_TABLE) return REF_E_STATE;
  const int32_t T = pr->T, K = pr->K;
  double* act = (double*)malloc(sizeof(double) * (size_t)A);
  int32_t* off = (int32_t*)malloc(sizeof(int32_t) * (size_t)A);
  double* w = (double*)malloc(sizeof(double) * (size_t)A);
  double* omw = (double*)malloc(sizeof(double) * (size_t)A);
  int32_t* ilo = (int32_t*)malloc(sizeof(int32_t) * (size_t)A);
  int32_t* ihi = (int32_t*)malloc(sizeof(int32_t) * (size_t)A);
  int16_t* vert = (int16_t*)malloc(sizeof(int16_t) * (size_t)A);
  double* q = (double*)malloc(sizeof(double) * (size_t)A);
  double* price = (double*)malloc(sizeof(double) * (size_t)A);
  ref_actions(pr, act);
  ref_tables(pr, off, w, omw, ilo, ihi);
  const int64_t KS = (int64_t)K * S;
  double x0 = pr->s0 / pr->delta;
  double r0 = nearbyint(x0);
  int on_grid = fabs(x0 - r0) <= GRID_TOL;
  double f0 = floor(x0), w0 = x0 - f0;
  int err = REF_OK;
  for (int64_t path = 0; path < n_paths && !err; ++path) {
    double u1, u2;
    uniforms(seed, path, 0, &u1, &u2);
    int32_t k = sample_cdf(pr->pi, K, u1);
    int32_t i = on_grid ? (int32_t)r0 : (int32_t)f0 + (u2 < w0 ? 1 : 0);
    double s = pr->s0;                                     /* physical mode: the real SoC */
    double profit = 0.0;
    for (int32_t t = 1; t <= T; ++t) {
      uniforms(seed, path, t, &u1, &u2);
      const double* Wrow = W + (int64_t)(t - 1) * KS + (int64_t)k * S;
      int32_t a;
      if (mode == REF_SIM_PHYSICAL) {
        double sn;
        a = physical_action(pr, S, A, act, Wrow, t, k, s, &sn);
        if (a < 0) { err = REF_E_INTERNAL; break; }       /* the zero action is always feasible */
        s = sn;
      } else {
        int32_t nv, rep;
        rc = ref_bidcurve(pr, W, t, i, k, A, &nv, vert, q, price, &rep);
        if (rc) { err = rc; break; }
        a = vert[ref_clear(nv, price, pr->lambda[(int64_t)(t - 1) * K + k])];
      }
      profit = profit + payoff(pr, A, act, t, k, a);
      if (mode == REF_SIM_CLEAR_BIDS) i = i + off[a] + ((w[a] > 0.0 && u1 < w[a]) ? 1 : 0);
      if (t < T) {
        const double* qk = pr->P ? pr->P + ((int64_t)(t - 1) * K + k) * K : pr->pi + (int64_t)t * K;
        k = sample_cdf(qk, K, u2);
      }
    }
    per_path[path] = profit;
  }
  if (!err) {
    double sm = 0.0;
    for (int64_t p = 0; p < n_paths; ++p) sm += per_path[p];
    double m = sm / (double)n_paths;
    double ss = 0.0;
    for (int64_t p = 0; p < n_paths; ++p) ss += (per_path[p] - m) * (per_path[p] - m);
    *mean = m;
    *var = n_paths > 1 ? ss / (double)(n_paths - 1) : 0.0;
  }
  free(act); free(off); free(w); free(omw); free(ilo); free(ihi); free(vert); free(q); free(price);
  return err;
}

int ref_simulate_strategy(const ref_problem* pr, const double* W, int32_t mode, const int16_t* schedule,
                          int64_t n_paths, uint64_t seed, double* per_path, int16_t* actions) {
  int32_t S, A;
  int rc = ref_dims(pr, &S, &A);
  if (rc) return rc;
  if (n_paths < 1) return REF_E_STATE;
  if (mode != REF_SIM_PHYSICAL && mode != REF_SIM_SELF && mode != REF_SIM_FIXED) return REF_E_STATE;
  if ((mode != REF_SIM_FIXED && !W) || (mode == REF_SIM_FIXED && !schedule)) return REF_E_STATE;
  if (mode == REF_SIM_SELF && pr->payoff_kind == REF_PAYOFF_TABLE) return REF_E_STATE;
  const int32_t T = pr->T, K = pr->K;
  double* act = (double*)malloc(sizeof(double) * (size_t)A);
  ref_actions(pr, act);
  const int64_t KS = (int64_t)K * S;
  int err = REF_OK;
  for (int64_t path = 0; path < n_paths && !err; ++path) {
    double u1, u2;
    uniforms(seed, path, 0, &u1, &u2);
    int32_t k = sample_cdf(pr->pi, K, u1);
    int32_t k_prev = k;
    double s = pr->s0, profit = 0.0, lam_prev = pr->lambda[k];   /* stage 1's lag: its own price */
    for (int32_t t = 1; t <= T; ++t) {
      uniforms(seed, path, t, &u1, &u2);
      const double lam_t = pr->lambda[(int64_t)(t - 1) * K + k];
      int32_t a;
      if (mode == REF_SIM_FIXED) {
        a = schedule[t - 1];
      } else {
        const int32_t row = pr->P == NULL ? 0 : (mode == REF_SIM_SELF ? k_prev : k);
        const double* Wrow = W + (int64_t)(t - 1) * KS + (int64_t)row * S;
        double sn;
        a = physical_action_lam(pr, S, A, act, Wrow, t, k, mode == REF_SIM_SELF ? &lam_prev : NULL, s, &sn);
        if (a < 0) { err = REF_E_INTERNAL; break; }
        s = sn;
      }
      if (actions) actions[(int64_t)(t - 1) * n_paths + path] = (int16_t)a;
      profit = profit + payoff(pr, A, act, t, k, a);        /* settled at the realised price */
      lam_prev = lam_t;
      k_prev = k;
      if (t < T) {
        const double* qk = pr->P ? pr->P + ((int64_t)(t - 1) * K + k) * K : pr->pi + (int64_t)t * K;
        k = sample_cdf(qk, K, u2);
      }
    }
    per_path[path] = profit;
  }
  free(act);
  return err;
}
