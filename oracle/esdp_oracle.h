/*
 * esdp_oracle.h -- plain, slow, FP64 CPU oracle for the discretized storage-arbitrage DP.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 *  (the CUDA package at the repo root) never links, loads or calls it, and the two
 * share no code: no headers, no helpers, no tables.
 *
 * Every function follows /root/reference/PAPER.md ("P:NNN" = line NNN) step by step,
 * with the readings of SURVEY.md §8(c) / DESIGN.md §3 where the paper is silent or garbled.
 * Arithmetic is IEEE binary64, compiled with -O2 -ffp-contract=off (no FMA contraction);
 * the only fused operations are the explicit C99 fma() calls of the expectation
 * (canonical ascending-k' chain, reading R15).
 *
 * Array conventions (0-based, row-major, all host memory, caller-owned):
 *   stage t = 1..T (paper indexing) is stored at index t-1.
 *   lambda[T][K]      price level lambda_{t,k}                  (Markov states k)
 *   P[T-1][K][K]      P_t[k][k'] = Pr(k_{t+1}=k' | k_t=k), t=1..T-1 (north_star; NULL => rank-1)
 *   pi                Markov: pi[K] = distribution of k_1;  rank-1 (P==NULL): pi[T][K], row t-1 = pi_t
 *   V[T][K][S]        V_t(s_i, k): value after observing k at stage t, before acting (paper Q_hat_{t-1})
 *   W[T][K][S]        W_t = P_t V_{t+1}, W_T = 0 (paper V_hat_t)
 *   pol[T][K][S]      smallest maximizing action index (R8)
 */
#ifndef ESDP_ORACLE_H
#define ESDP_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { REF_OK = 0, REF_E_CONFIG = 1, REF_E_DATA = 2, REF_E_INTERNAL = 3, REF_E_STATE = 4 };
enum { REF_PAYOFF_LINEAR = 0, REF_PAYOFF_LINEAR_MINUS_G = 1, REF_PAYOFF_TABLE = 2 };

typedef struct {
  int32_t T, K;
  double pbar, sbar, s0;
  double eta_c, eta_d;     /* P:82-89 with separate charge / discharge efficiency */
  double delta;
  int32_t A;               /* 0 => paper action grid, Eq. 10 */
  const double* actions;   /* [A] when A > 0 */
  const double* lambda;    /* [T][K] */
  const double* P;         /* [T-1][K][K] or NULL */
  const double* pi;        /* [K] or [T][K] */
  int32_t payoff_kind;
  const double* g;         /* [A] (LINEAR_MINUS_G) or [T][K][A] (TABLE); ignored for LINEAR */
} ref_problem;

/* Grid sizes: S = sbar/delta + 1 and A (Eq. 10).  Validates the whole problem
 * (DESIGN.md §3 "validation"); returns REF_E_CONFIG / REF_E_DATA on invalid input. */
int ref_dims(const ref_problem* pr, int32_t* S, int32_t* A);

/* Action grid p_hat (Eq. 10) written to actions[A] (ascending). */
int ref_actions(const ref_problem* pr, double* actions);

/* Alg. 1 lines 2-5, reduced to per-action data: e_a = F(p_a)/delta,
 * o_a = floor (or round if integral), w_a = interpolation factor b, omw_a = 1 - w_a,
 * feasible row range [ilo_a, ihi_a] (Eq. 4 / Alg. 1 line 8). */
int ref_tables(const ref_problem* pr, int32_t* off, double* w, double* omw, int32_t* ilo, int32_t* ihi);

/* Backward induction (Alg. 1 lines 6-11; Markov form of Eqs. 5-6).
 * Computes stages t = T down to t_stop (1 <= t_stop <= T).  V, W: [T][K][S]; pol: [T][K][S]
 * (int16).  J (nullable) is written only when t_stop == 1 (Eq. 6 at t=0).
 * nthreads > 1 parallelises over independent (k, i) rows (OpenMP); results are
 * bit-identical for every nthreads. */
int ref_backward(const ref_problem* pr, int32_t t_stop, int32_t nthreads,
                 double* V, double* W, int16_t* pol, double* J);

/* One stage t for the price-state rows [k_lo, k_hi) only (the unit of the K-partitioned multi-GPU
 * schedule): Vnext = V_{t+1} [K][S] (all rows; NULL at t = T); Wt, Vt, polt are
 * [k_hi - k_lo][S].  ref_backward is exactly this over all rows, stage after stage. */
int ref_stage(const ref_problem* pr, int32_t t, int32_t k_lo, int32_t k_hi, int32_t nthreads, const double* Vnext,
              double* Wt, double* Vt, int16_t* polt);

/* J = sum_k pi_1[k] V_1(s0, k) (Eq. 6 at t = 0) from V_1 [K][S]. */
int ref_objective(const ref_problem* pr, const double* V1, double* J);

/* Bid curve for stage t (1..T), SoC index i, price state k, from W_t:
 * points (p_a, u_a = Wint_t(i,a,k) - g_a) over feasible a, upper concave hull
 * (monotone chain = Graham scan on x-sorted points), prices -du/dp (Eq. 12),
 * running-max repair (R20).  Outputs nvert, vert[nvert] (action indices),
 * q[nvert] (powers), price[nvert-1].  cap >= A required.  Not defined for TABLE payoffs. */
int ref_bidcurve(const ref_problem* pr, const double* W, int32_t t, int32_t i, int32_t k,
                 int32_t cap, int32_t* nvert, int16_t* vert, double* q, double* price,
                 int32_t* n_repairs);

/* Merit-order clearing of one curve at price lam: the vertex with the largest j such
 * that j == 0 or price[j-1] <= lam (ties to the larger quantity, R9). */
int32_t ref_clear(int32_t nvert, const double* price, double lam);

/* Philox4x32-10 (Salmon et al., SC'11), one block. */
void ref_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Forward simulation of the argmax policy, lottery semantics at off-grid endpoints
 * (R16/R17).  n paths; per_path[n] profits; mean/var over paths. */
int ref_simulate(const ref_problem* pr, const int16_t* pol, int64_t n_paths, uint64_t seed,
                 double* per_path, double* mean, double* var);

/* Simulation modes (SURVEY §8(a) a7 "take a = pol_t[k][i] (or clear the bid)"; §8(c) step 7 physical
 * mode; R25/R26), same random numbers as ref_simulate:
 *   REF_SIM_LOTTERY    = ref_simulate (pol; W unused);
 *   REF_SIM_PHYSICAL   real SoC s (starts at s0): at every stage re-optimise over all actions,
 *                      cand = payoff + W_t(s + F(p_a)) interpolated at the off-grid state, smallest
 *                      maximising index, then s <- s + F(p_a*) (snapped to the grid within 1e-9);
 *   REF_SIM_CLEAR_BIDS grid state i (lottery moves as in ref_simulate): the action is the bid curve
 *                      of (t, i, k) from W_t cleared at lambda_{t,k} (ref_bidcurve + ref_clear).
 * W: [T][K][S] (all stages; needed by the last two modes).  TABLE payoffs: CLEAR_BIDS -> REF_E_STATE. */
enum { REF_SIM_LOTTERY = 0, REF_SIM_PHYSICAL = 1, REF_SIM_CLEAR_BIDS = 2, REF_SIM_SELF = 3, REF_SIM_FIXED = 4 };
int ref_simulate_mode(const ref_problem* pr, const int16_t* pol, const double* W, int32_t mode, int64_t n_paths,
                      uint64_t seed, double* per_path, double* mean, double* var);

/* Dispatch strategies of the paper's Fig. 3 study (R27/R28),
 * on the same price paths (Philox draws) as the modes above, at the real SoC from s0:
 *   REF_SIM_PHYSICAL  as ref_simulate_mode (the "stochastic DP bid curves" dispatch: re-optimise at the
 *                     real SoC with the realised price, i.e. clear the stage's curve at it);
 *   REF_SIM_SELF      "self-scheduled": the decision uses the realised 1-stage-lagged price (stage 1: its
 *                     own price) and the continuation row of the last observed price state (persistence
 *                     forecast; stage 1: k_1), then settles at the realised price (R27);
 *   REF_SIM_FIXED     a fixed schedule of actions schedule[T] (e.g. the myopic plan on day-ahead prices),
 *                     settled at the realised prices (R28).
 * W: [T][K][S] (PHYSICAL, SELF).  actions (nullable): [T][n_paths] chosen action indices.  SELF rejects
 * TABLE payoffs (the price must enter linearly). */
int ref_simulate_strategy(const ref_problem* pr, const double* W, int32_t mode, const int16_t* schedule,
                          int64_t n_paths, uint64_t seed, double* per_path, int16_t* actions);

#ifdef __cplusplus
}
#endif
#endif
