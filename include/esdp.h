/*
 * esdp.h -- C ABI of libesdp.so, the B200 (sm_100a) backward induction for the discretized
 * multistage stochastic energy-storage arbitrage DP of arXiv 2511.15629
 * ("GPU-Accelerated Dynamic Programming for Multistage Stochastic Energy Storage Arbitrage").
 *
 * Citations "P:NNN" are lines of the paper source; "DESIGN §x" is DESIGN.md at the
 * repo root, which lists every reading of the paper this library adopts (R1..R24).
 *
 * Conventions for every entry point
 *   - Plain C types only.  Every call returns esdp_status; nothing throws across the ABI.
 *   - Host pointers unless the name ends in _dev.  Input arrays are deep-copied by the call
 *     that receives them; the caller may free them as soon as the call returns.
 *   - Output arrays are caller-allocated, sized from esdp_dims().
 *   - On error the outputs are left untouched and esdp_last_error(ctx) describes the failure
 *     (for esdp_create failures, esdp_last_error(NULL) holds the message for this thread).
 *   - One caller per context at a time; distinct contexts are independent.
 *   - All arithmetic is IEEE binary64.  Stage index t is 1-based (t = 1..T), SoC index
 *     i is 0-based (s_i = i * delta), price state k is 0-based.
 *   - Array layouts are row-major:  lambda[T][K], P[T-1][K][K], V/W[K][S] per stage,
 *     pol[K][S] per stage (int16 action index into the ascending action grid).
 */
#ifndef ESDP_H
#define ESDP_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct esdp_ctx esdp_ctx; /* opaque: owns device buffers, the CUDA graph, the stream */

typedef enum {
  ESDP_OK = 0,
  ESDP_E_CONFIG = 1,   /* bad grid / parameters: T, K < 1; K > 32767; pbar, sbar, delta <= 0; eta not in (0,1];
                          s0 not in [0, sbar]; sbar/delta not integral (no silent rounding);
                          actions not strictly ascending, without an exact 0, |p| > pbar; A > 8191 */
  ESDP_E_DATA = 2,     /* non-finite lambda or g; a row of P (or pi) is not a probability simplex
                          within 1e-9 */
  ESDP_E_INTERNAL = 3, /* an invariant failed (a row with every action infeasible; cannot happen
                          because the zero action is always feasible, Eq. 4) */
  ESDP_E_STATE = 4,    /* call order (query before esdp_backward), index out of range, or a
                          feature not defined for this problem (bid curves of TABLE payoffs) */
  ESDP_E_CUDA = 5,     /* a CUDA runtime error (message has the CUDA error string) */
  ESDP_E_NCCL = 6,     /* reserved for the multi-GPU communicator */
  ESDP_E_NOMEM = 7     /* device or host allocation failed */
} esdp_status;

/* Payoff of action p_a at price state k of stage t (Alg. 1 line 9; D3 in DESIGN §2):
 *   LINEAR          pay = lambda_{t,k} * p_a                       (the paper's payoff)
 *   LINEAR_MINUS_G  pay = lambda_{t,k} * p_a - g[a]                 (degradation / fixed costs;
 *                                                                    may be non-concave)
 *   TABLE           pay = g[t-1][k][a]                              (any payoff; no bid curves)
 * The candidate value is pay + Wint, rounded in that association (DESIGN R14). */
enum { ESDP_PAYOFF_LINEAR = 0, ESDP_PAYOFF_LINEAR_MINUS_G = 1, ESDP_PAYOFF_TABLE = 2 };

/* flags */
enum {
  ESDP_KEEP_VALUES = 1u,  /* keep V_t and W_t for every t on the device (needed by esdp_values
                             for t > 1 and by the bid-curve calls); otherwise only V_1 is kept */
  ESDP_PROFILE = 2u,      /* record CUDA events around the contraction and stencil launches of ~16
                             sampled stages inside the backward graph (esdp_kernel_times) */
  ESDP_FORCE_BRUTE = 4u,  /* always use the brute-force max-plus stencil (every (i, a) cell), even
                             where the exact sliding-window stencil applies (for testing) */
  ESDP_NO_PDL = 8u,       /* launch the per-stage kernels without programmatic dependent launch (PDL
                             with a late trigger is the default: ~3.5% faster chain) */
  ESDP_NO_DMMA = 16u,     /* expectation on FP64 CUDA cores (DFMA) instead of the FP64 tensor cores */
  ESDP_CONTRACT_OZAKI = 32u, /* batches (esdp_create_batch, flag of probs[0]) with K <= 128 and a zero
                             action of payoff >= 0 (so V >= 0): the expectation on the 5th-generation
                             tensor cores, Ozaki-sliced u8 tcgen05 products.  NOT
                             the canonical chain of R15: W within ~1e-14 relative of the exact product,
                             policies may differ at documented near-ties.  Ignored (the
                             DMMA path runs) where the conditions fail: esdp_batch_plan reports it. */
  ESDP_FLAGS_ALL = 63u    /* every defined flag; other bits -> ESDP_E_CONFIG.  Bit 64 once named a
                             path that measured slower on B200 and was removed. */
};

/* Environment variables read at context creation (measurement knobs; every setting gives the same bits):
 *   ESDP_DMMA3=0      expectation on the all-at-once staged DMMA kernel instead of the k'-pipelined one
 *   ESDP_WIN_OPT=1|2|4  output columns per thread of the window stencil (default: 1 for a latency-bound
 *                     grid, 4 for a large one and for batches)
 *   ESDP_WIN_GENERIC=1  window queries on the generic path even where the Eq. 10 fast path applies
 *   ESDP_WIN_FORCE_NONUNI=1  treat every window run table as non-unimodal (tests: the fallback paths)
 *   ESDP_GUIDE_RATIO=n  guide buckets per price state of the simulation's sampling rows (default 64)
 *   ESDP_GUIDE_BUDGET_MB=n  cap of the guide allocation per input slot (default 256, or the size of P)
 *   ESDP_FB_MODE=0|1|2  fused bid curves: side branches along the stage chain (0, default), the same batches
 *                     forked after stage 1 (1), one launch on the chain stream after stage 1 (2)
 *   ESDP_FB_BATCHES=n  fused bid curves in n stage batches per backward (default 8)
 *   ESDP_CARVEOUT=p   preferred shared-memory carveout (percent) of the stage-chain launches (default: the
 *                     maximum in the latency regime -- one output per thread in the window plan --, else none;
 *                     -1: none)
 *   ESDP_PRES=0       wide batch expectations (K <= 104, >= 4e6 outputs) on the block-tiled DMMA kernel
 *                     instead of the P-resident persistent one
 *   ESDP_HOST_THREADS=n  threads of the host pool (validation, slice hashing; default min(16, cores))
 *   ESDP_BATCH_GROUPS=G  a batch's instances in G groups with independent stage chains (default 2 from 128
 *                     instances on, else 1; window-plan instances with the DMMA or Ozaki expectation only)
 * DESIGN.md §5 and §7 record what each measured. */

typedef struct {
  int32_t T, K;          /* stages and Markov price states (north_star; the paper's R) */
  double pbar, sbar, s0; /* power cap, energy cap, initial SoC, energy-per-stage units */
  double eta_c, eta_d;   /* charge / discharge efficiency in (0,1]: F(p) = -p/eta_d (p >= 0),
                            -eta_c p (p < 0) (Eq. 2; single eta in the paper) */
  double delta;          /* SoC step; S = sbar/delta + 1 */
  int32_t A;             /* 0 => the paper's recombining grid, Eq. 10; else len(actions) */
  const double* actions; /* [A] strictly ascending, contains 0.0 exactly, |p| <= pbar (when A > 0) */
  const double* lambda;  /* [T][K] price levels lambda_{t,k} */
  const double* P;       /* [T-1][K][K], P[t-1][k][k'] = Pr(k_{t+1} = k' | k_t = k), t = 1..T-1;
                            NULL => stagewise independent (rank-1) prices, the paper's case */
  const double* pi;      /* Markov: [K] distribution of k_1.  Rank-1 (P == NULL): [T][K], row t-1 is
                            pi_t, the probabilities of the stage-t price levels */
  int32_t payoff_kind;   /* ESDP_PAYOFF_* */
  const double* g;       /* [A] for LINEAR_MINUS_G, [T][K][A] for TABLE, ignored for LINEAR */
  uint32_t flags;        /* ESDP_KEEP_* */
} esdp_problem;

/* Create a solver: validates the problem (same rules as the oracle), builds the state/action
 * grid and the per-action transition data (Alg. 1 lines 2-5), allocates device
 * memory on the current CUDA device and uploads the inputs.  *out receives the context. */
esdp_status esdp_create(const esdp_problem* prob, esdp_ctx** out);

/* Multi-GPU (north_star): one process per GPU, `world` ranks.  Rank r owns the price-
 * state rows [k_lo, k_lo + k_cnt) given by esdp_partition (blocks of kmax = ceil(K/world) rows).  Every
 * stage it computes W_t and V_t for its rows and all-gathers V_t over NCCL (in place, kmax rows per rank:
 * the only exchange on the stage chain, "only t is sequential"); the policy rows stay local and
 * are all-gathered once after stage 1 (one NCCL group of T all-gathers).  After esdp_backward every rank
 * holds all of V and the policy, bit-identical to a single GPU (an all-gather is a copy).  nccl_id: the
 * 128-byte ncclUniqueId made by esdp_nccl_unique_id on one rank and broadcast by the caller.  The current
 * CUDA device must be this rank's GPU.  W_t (and bid curves) are available only for the rank's own rows;
 * esdp_values with W != NULL -> ESDP_E_STATE.  Failure detection: the synchronous calls (esdp_backward,
 * esdp_objective) poll ncclCommGetAsyncError while they wait; an asynchronous NCCL error, or no completion
 * within ESDP_NCCL_TIMEOUT_S seconds (environment, default 120: a dead or hung peer), aborts the
 * communicator (ncclCommAbort) and returns ESDP_E_NCCL; the context then needs recreating. */
esdp_status esdp_create_dist(const esdp_problem* prob, int32_t world, int32_t rank, const void* nccl_id,
                             esdp_ctx** out);
esdp_status esdp_nccl_unique_id(void* id128);
/* world size and rank of a context, and the communicator's own rank count (ncclCommCount; 0 without a
 * communicator, -1 if the query failed): lets a launcher check that NCCL saw every rank. */
esdp_status esdp_dist_info(const esdp_ctx* ctx, int32_t* world, int32_t* rank, int32_t* nccl_nranks);
/* Row ownership of a rank (pure host function; no GPU needed). */
esdp_status esdp_partition(int32_t K, int32_t world, int32_t rank, int32_t* k_lo, int32_t* k_cnt, int32_t* kmax);

/* Grid sizes: T, S = sbar/delta + 1, A, K (any pointer may be NULL). */
esdp_status esdp_dims(const esdp_ctx* ctx, int32_t* T, int32_t* S, int32_t* A, int32_t* K);

/* The action grid p_hat[A] (ascending) the solver uses (Eq. 10 or the user's actions). */
esdp_status esdp_actions(const esdp_ctx* ctx, double* actions);

/* Re-upload the stochastic inputs from HOST memory (shapes as in esdp_problem; NULL keeps the
 * newest array).  Validated like esdp_create (on error nothing changes).  Used for end-to-end runs
 * where every solve brings new prices.  The inputs are double-buffered: a load fills the slot that
 * the last launched backward pass does not read, and the next esdp_backward* switches to it; until
 * then the results of the last backward (values, policy, bid curves, simulations) stay those of the
 * previous inputs. */
esdp_status esdp_load(esdp_ctx* ctx, const double* lambda, const double* P, const double* pi,
                      const double* g);

/* Same as esdp_load, but returns once the arrays are validated and their upload is enqueued (P in stage
 * chunks, highest stages first, on the context's copy stream, after the device has finished the
 * solve before last that read the target slot); the next backward pass waits for each chunk only
 * where it needs it, so the host-to-device copy overlaps the running solve (pipelined steps) and the
 * next one.  The host arrays must stay valid and unmodified until the next esdp_backward (or a
 * synchronizing call after esdp_backward_async) returns; pinned (page-locked) memory makes the
 * copies asynchronous. */
esdp_status esdp_load_async(esdp_ctx* ctx, const double* lambda, const double* P, const double* pi,
                            const double* g);

/* J of the last backward pass copied to J_host (pinned host memory for an asynchronous copy), enqueued
 * on stream after the solve (NULL = the context's own stream); the caller synchronizes. */
esdp_status esdp_objective_async(esdp_ctx* ctx, double* J_host, void* stream);

/* Backward induction, Alg. 1 lines 6-11 in Markov form (Eqs. 5-6):
 *   W_T = 0;  for t = T..1:  W_t = P_t V_{t+1} (t < T),
 *             V_t(i,k) = max_a pay(t,k,a) + Wint_t(i,a,k),  pol_t(i,k) = smallest argmax,
 * where Wint is the interpolated, infeasibility-masked continuation of Alg. 1 lines 7-8.
 * Then J = sum_k pi_1[k] V_1(s0, k) (Eq. 6 at t = 0).  Runs on `stream` (a cudaStream_t,
 * NULL = the context's own stream) and synchronizes it before returning.  J may be NULL. */
esdp_status esdp_backward(esdp_ctx* ctx, void* stream, double* J);

/* Enqueue the backward pass on `stream` without synchronizing (for timing harnesses); the J of the
 * run is available from esdp_objective after the stream completes. */
esdp_status esdp_backward_async(esdp_ctx* ctx, void* stream);
esdp_status esdp_objective(esdp_ctx* ctx, double* J);

/* Copy V_t [K][S] and (if W != NULL) W_t [K][S] to host memory.  t must be 1 unless the context
 * was created with ESDP_KEEP_VALUES. */
esdp_status esdp_values(const esdp_ctx* ctx, int32_t t, double* V, double* W);

/* Copy the policy pol_t [K][S] (int16 action indices) to host memory. */
esdp_status esdp_policy(const esdp_ctx* ctx, int32_t t, int16_t* pol);

/* Bid curves, one per request (t, i, k): points (p_a, u_a = Wint_t(i,a,k) - g_a) over the
 * feasible actions (Eq. 7), upper concave hull (Graham / monotone chain), monotone segment
 * prices price_j = -(u_{j+1} - u_j)/(p_{j+1} - p_j) (Eq. 12) with a running-max repair (DESIGN R20).
 *   req    [n][3] int32 (t, i, k), host
 *   cap    per-curve capacity, >= A
 *   nvert  [n] vertices per curve; vert [n][cap] action indices; q [n][cap] powers;
 *   price  [n][cap] segment prices (entries >= nvert-1 unused).  Requires ESDP_KEEP_VALUES. */
esdp_status esdp_bidcurves(esdp_ctx* ctx, int64_t n, const int32_t* req, int32_t cap,
                           int32_t* nvert, int16_t* vert, double* q, double* price);
/* Same, with DEVICE pointers for every array, enqueued on `stream` (no synchronization).  Output
 * layout is VERTEX-major, [cap][n] (entry j of curve r at j*n + r: coalesced stores); q_dev may be
 * NULL (the quantities are actions[vert]). */
esdp_status esdp_bidcurves_dev(esdp_ctx* ctx, int64_t n, const int32_t* req_dev, int32_t cap,
                               int32_t* nvert_dev, int16_t* vert_dev, double* q_dev, double* price_dev,
                               void* stream);

/* Register bid-curve requests that every following backward pass extracts INSIDE the stage chain: the
 * curves of stage t are built from W_t in a side branch of the backward graph as soon as W_t exists,
 * concurrently with the remaining (latency-bound) stages.  req: HOST [n][3] (t, i, k), copied; outputs:
 * DEVICE arrays in the layout of esdp_bidcurves_dev (vertex-major [cap][n]; q_dev may be NULL), written
 * by each backward pass.  n = 0 removes the requests.  Needs ESDP_KEEP_VALUES and the graph plan. */
esdp_status esdp_set_bid_requests(esdp_ctx* ctx, int64_t n, const int32_t* req, int32_t cap, int32_t* nvert_dev,
                                  int16_t* vert_dev, double* q_dev, double* price_dev);

/* Forward simulation of the argmax policy on n_paths sampled price paths:
 *   k_1 ~ pi_1; for t = 1..T: a = pol_t(i, k); profit += pay(t,k,a);
 *   i <- i + o_a (+1 with probability w_a at the interpolated endpoints: the lottery that the
 *   interpolation of Alg. 1 line 7 represents, DESIGN R16); k <- sample of P_t[k, :].
 * Random numbers: Philox4x32-10 (counter = (path, t, 'ESDP'), key = seed), DESIGN R17.
 * per_path [n_paths] (host, nullable), mean, var (sample variance) over paths. */
esdp_status esdp_simulate(esdp_ctx* ctx, int64_t n_paths, uint64_t seed, double* mean, double* var,
                          double* per_path);
/* Asynchronous variant for pipelined callers: the simulation and its deterministic reduction are
 * enqueued on stream (NULL = the context's own); stats_dev[2] (device) receives {mean, sample
 * variance}.  Nothing is synchronized. */
esdp_status esdp_simulate_async(esdp_ctx* ctx, int64_t n_paths, uint64_t seed, double* stats_dev, void* stream);
/* Device variant: per-path profits to per_path_dev, enqueued on stream. */
esdp_status esdp_simulate_dev(esdp_ctx* ctx, int64_t n_paths, uint64_t seed, double* per_path_dev,
                              void* stream);

/* Simulation modes (SURVEY §8(a) a7 "take a = pol_t[k][i] (or clear the bid)"; §8(c) step 7;
 * DESIGN.md R25/R26), with the same Philox draws as esdp_simulate:
 *   ESDP_SIM_LOTTERY     the argmax policy on the grid, lottery moves at off-grid endpoints (= esdp_simulate);
 *   ESDP_SIM_PHYSICAL    the real SoC s (from s0): every stage re-optimises over all actions with
 *                        payoff + W_t(s + F(p_a)) interpolated at the off-grid index (Alg. 1 line 7),
 *                        smallest maximising index; s <- s + F(p_a*) (snapped to the grid within 1e-9);
 *   ESDP_SIM_CLEAR_BIDS  grid states with lottery moves; the action is the stage's bid curve at (t, i, k)
 *                        cleared at the realised price lambda_{t,k} (merit order; ties to the
 *                        larger quantity, R9).
 * PHYSICAL and CLEAR_BIDS need ESDP_KEEP_VALUES and one GPU; CLEAR_BIDS rejects TABLE payoffs
 * (ESDP_E_STATE).  Host variant: mean, var (sample), per_path[n_paths] (nullable), synchronized. */
enum { ESDP_SIM_LOTTERY = 0, ESDP_SIM_PHYSICAL = 1, ESDP_SIM_CLEAR_BIDS = 2, ESDP_SIM_SELF = 3, ESDP_SIM_FIXED = 4 };
esdp_status esdp_simulate_mode(esdp_ctx* ctx, int64_t n_paths, uint64_t seed, int32_t mode, double* mean,
                               double* var, double* per_path);
esdp_status esdp_simulate_mode_dev(esdp_ctx* ctx, int64_t n_paths, uint64_t seed, int32_t mode,
                                   double* per_path_dev, void* stream);

/* The price paths of esdp_simulate(seed) for the inputs of the last solve: k_t and the realised price
 * lambda_{t,k_t} of every path, [T][n_paths] each (device; either output may be NULL).  Used to set up
 * perfect-foresight solves on the realised paths (the Fig. 3 upper bound). */
esdp_status esdp_price_paths_dev(esdp_ctx* ctx, int64_t n_paths, uint64_t seed, int16_t* kpath_dev,
                                 double* lambda_dev, void* stream);

/* Dispatch strategies of the paper's Fig. 3 study (R27/R28),
 * on the same price paths as esdp_simulate, from the real SoC s0:
 *   ESDP_SIM_PHYSICAL   "stochastic DP bid curves": the stage's curve cleared at the realised price
 *                       (= re-optimisation at the real SoC, as above);
 *   ESDP_SIM_SELF       "self-scheduled": decided at the realised one-stage-lagged price (stage 1: its own
 *                       price) with the continuation row of the last observed price state, settled at the
 *                       realised price;
 *   ESDP_SIM_FIXED      the fixed schedule schedule_dev[T] (device; e.g. the myopic plan recorded from a
 *                       day-ahead context of the same grid), settled at the realised prices.
 * actions_dev (nullable, device): [T][n_paths] chosen action indices (not for CLEAR_BIDS).  PHYSICAL and
 * SELF need ESDP_KEEP_VALUES and one GPU; SELF and CLEAR_BIDS reject TABLE payoffs. */
esdp_status esdp_simulate_strategy_dev(esdp_ctx* ctx, int64_t n_paths, uint64_t seed, int32_t mode,
                                       const int16_t* schedule_dev, int16_t* actions_dev, double* per_path_dev,
                                       void* stream);

/* Execution plan: bit 0 = stencil (1 = exact sliding-window for the recombining grid with a linear
 * payoff, 0 = brute force over every (i, a) cell); bit 1 = expectation on the FP64 tensor cores (DMMA,
 * wherever the shape allows: >= 8 rows or rank-1 with even K; 0 = DFMA on the CUDA cores); bit 2 = the DMMA bit-exactness probe run at context creation found a
 * DMMA result that differs from the canonical fma chain (R15), so the expectation fell back to DFMA.
 * All plans give bit-identical results. */
esdp_status esdp_stencil_kind(const esdp_ctx* ctx, int32_t* kind);

/* Number of (i, k) rows, summed over all stages and contexts since the last call, for which the
 * sliding-window stencil found a near tie and re-scanned every action canonically (then resets it). */
esdp_status esdp_window_fallbacks(esdp_ctx* ctx, int64_t* count);

/* Number of run tables (one charge and one discharge table per (stage, k, 256-column tile) item of the
 * sliding-window stencil), summed since the last call (then resets), whose packed keys were NOT
 * unimodal, so the sparse-table levels were built; a unimodal table is answered in O(1) from its peak
 * (DESIGN.md §5.3).  Either way the results are the same bits. */
esdp_status esdp_window_level_tables(esdp_ctx* ctx, int64_t* count);

/* Number of kernel launches one backward pass enqueues (for harness accounting). */
esdp_status esdp_launch_count(const esdp_ctx* ctx, int64_t* backward_launches);

/* Average device time (ms) of one expectation phase and of one stencil phase in the last completed
 * backward pass (requires ESDP_PROFILE; the caller has synchronized the stream): CUDA events recorded
 * inside the graph around the kernels of ~16 evenly spaced stages. */
esdp_status esdp_kernel_times(const esdp_ctx* ctx, double* contract_ms, double* stencil_ms);

/* Diagnostic micro-timing (not part of the solve): warm back-to-back launches of one kernel of stage
 * T-1 captured in a graph: what = 0 contraction, 1 the context's stencil, 2 brute-force stencil,
 * 3 objective kernel.  Needs a completed backward pass.  *us_per_launch = average device time. */
esdp_status esdp_debug_time(esdp_ctx* ctx, int32_t what, int32_t reps, double* us_per_launch);

void esdp_destroy(esdp_ctx* ctx);

/* Message of the last failing call on ctx (ctx == NULL: last esdp_create failure of this thread). */
const char* esdp_last_error(const esdp_ctx* ctx);

/* ---------------------------------------------------------------------------------------------
 * Batch contexts (SURVEY §8(b) esdp_create_batch; BASELINE cfg5: a sweep of storage configurations
 * over one price model).  n instances share T, K, sbar, delta (hence S), lambda, P and pi (the
 * price model of Eqs. 5-6) and each have their own pbar, eta_c, eta_d, s0, action grid
 * (Eq. 10) and payoff (LINEAR or LINEAR_MINUS_G; TABLE is rejected).  The backward pass
 * of all instances is one CUDA graph: per stage ONE expectation W_t = P_t V_{t+1} over the stacked
 * [K][n][ld] values (one [K] x [n ld] product) and ONE window-stencil launch over every instance on
 * the exact sliding-window plan (the others take a brute-force launch each).  Every instance's
 * values, policy and J are bit-identical to a context of its own.  Values are not kept per stage
 * (V_1 only); the policy of every stage is kept ([n][T][K][S] int16).
 * --------------------------------------------------------------------------------------------- */
typedef struct esdp_batch esdp_batch;

/* probs[0..n-1]: host descriptions as for esdp_create (deep-copied).  lambda, P and pi must be
 * identical in content across instances (else ESDP_E_CONFIG); they are validated once.  flags:
 * KEEP_VALUES / PROFILE are ignored.  Errors as esdp_create (message: esdp_batch_last_error(NULL)). */
esdp_status esdp_create_batch(const esdp_problem* probs, int32_t n, esdp_batch** out);
/* n, T, S, K and A[n] (each instance's action count; A may be NULL). */
esdp_status esdp_batch_dims(const esdp_batch* b, int32_t* n, int32_t* T, int32_t* S, int32_t* K, int32_t* A);
/* Backward pass of every instance on stream (NULL = the batch's own), synchronized; J[n] may be NULL. */
esdp_status esdp_batch_backward(esdp_batch* b, void* stream, double* J);
esdp_status esdp_batch_backward_async(esdp_batch* b, void* stream);
/* J of every instance ([n], host) after a completed backward pass. */
esdp_status esdp_batch_objective(esdp_batch* b, double* J);
/* Policy pol_t of instance m ([K][S] int16, host). */
esdp_status esdp_batch_policy(esdp_batch* b, int32_t m, int32_t t, int16_t* pol);
/* V_1 of instance m ([K][S] FP64, host). */
esdp_status esdp_batch_value1(esdp_batch* b, int32_t m, double* V1);
/* n_paths lottery-mode paths per instance (a7): instance m draws with Philox key seed + m, exactly the
 * paths of esdp_simulate_dev(seed + m) on a context of its own; per-path profits to
 * out_dev[m * n_paths + path] (device).  Enqueued on stream, not synchronized. */
esdp_status esdp_batch_simulate_dev(esdp_batch* b, int64_t n_paths, uint64_t seed, double* out_dev, void* stream);
/* Replace the shared price model (lambda [T][K]; P [T-1][K][K] or NULL in rank-1 mode; pi as in
 * esdp_problem) of every instance: validated on the host as esdp_create does (ESDP_E_DATA), then copied
 * host->device and the simulation's sampling tables rebuilt, all enqueued on stream (NULL = the batch's
 * own).  A later esdp_batch_backward_async on the same stream solves with the new inputs.  Pinned host
 * arrays must stay valid until the stream has passed the copies (pageable ones are staged at once).  A
 * new P may not have more distinct stage slices than the batch was created with (ESDP_E_STATE). */
esdp_status esdp_batch_load_async(esdp_batch* b, const double* lambda, const double* P, const double* pi, void* stream);
/* Kernel launches of one batch backward pass. */
esdp_status esdp_batch_launch_count(const esdp_batch* b, int64_t* n);
/* Diagnostic: microseconds per warm launch of stage T-1's batch expectation (what = 0), window-stencil
 * (1) or brute-force stencil (2) kernel, reps back-to-back launches in a CUDA graph (CUDA events on the
 * batch's stream).  Needs a completed backward pass (its buffers are the inputs). */
esdp_status esdp_batch_kernel_time(esdp_batch* b, int32_t what, int32_t reps, double* us_per_launch);
/* Plan of the batch's expectation: 0 FP64 DMMA (canonical chain), 1 DFMA (canonical chain), 2 Ozaki u8
 * tcgen05 (ESDP_CONTRACT_OZAKI granted). */
esdp_status esdp_batch_plan(const esdp_batch* b, int32_t* contraction);
/* The expectation alone (a2; Alg. 1 line 11; Eq. 6): W[m][n] = sum_k' P[m][k'] V[k'][n] for m < rows,
 * n < ncols, on DEVICE buffers: P [rows][K] (row stride K), V [K][ldv], W [rows][ldw]; enqueued on
 * stream (NULL: the legacy default stream), not synchronized.  method 0: the canonical ascending-k' fma
 * chain (R15) on the FP64 tensor cores (DMMA; DFMA for odd K or fewer than 8 rows), bit-identical to the
 * oracle; requires ldv == ldw.  method 1: the Ozaki-sliced u8 tcgen05 product (ozaki.cuh): requires
 * rows <= 128, K <= 128 and non-negative, finite P and V (not checked on the device: negative entries give
 * wrong results).  ESDP_E_CONFIG on bad sizes, strides or method; ESDP_E_CUDA on a launch failure. */
esdp_status esdp_expectation_dev(const double* P_dev, const double* V_dev, double* W_dev, int32_t rows, int32_t K,
                                 int64_t ncols, int64_t ldv, int64_t ldw, int32_t method, void* stream);
void esdp_batch_destroy(esdp_batch* b);
/* Message of the last failing call on b (b == NULL: last esdp_create_batch failure of this thread). */
const char* esdp_batch_last_error(const esdp_batch* b);

#ifdef __cplusplus
}
#endif
#endif
