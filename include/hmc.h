/*
 * hmc.h - C ABI of libhmc.so: the full-batch leapfrog hot path of VI-informed subset HMC
 * (Thiagarajan, Zaki, Shields, arXiv 2507.14652), built for NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = PAPER.md line n (LaTeX source of the paper); S:n = SPEC.md line n;
 * "Qn" = the readings of ambiguous passages listed in DESIGN.md §3.
 *
 * The operation (Algorithm 2): the parameters Theta of a network F_Theta are split
 * into an active subset Theta_s (k entries, flat indices idx) and a frozen subset Theta_~s fixed
 * at the VI means mu_~s.  HMC samples the conditional posterior
 * P(Theta_s | D, mu_~s) with Gaussian likelihood and a zero-mean Gaussian prior on
 * Theta_s (Table 5):
 *     log pi(theta_s) = -sum_n (y_n - F_n)^2 / (2 sigma^2) - sum_{i in s} theta_i^2 / (2 sigma_p^2)
 * (normalising constants dropped, Q7; hmc_logpost_const returns them).  Each HMC iteration draws
 * p ~ N(0, M), integrates Hamilton's equations with leapfrog (kick-drift-kick,
 * Q2), and applies the Metropolis test r > u (accept iff ln u < H0 - H*, strict,
 * non-finite rejects; Q4/Q5) with H = -log pi + 1/2 p^T M^-1 p (Q1), M diagonal (Q6).
 *
 * Conventions for every call:
 *  - All functions return an int status: HMC_OK (0) or one of HMC_E_* below.  A failing call
 *    leaves a message retrievable with hmc_last_error(ctx) (or hmc_last_error(NULL) for
 *    failures before a context exists).  Non-finite log pi or H is NOT an error: it is
 *    returned in the outputs and makes the proposal rejected.
 *  - Pointers may be host or device memory (detected per pointer with cudaPointerGetAttributes);
 *    host buffers are staged through pinned memory and the call synchronises the stream before
 *    returning.  With device pointers the call is asynchronous on `stream`.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - Flat parameter layout: per net, per linear layer W[out x in] row-major
 *    then b[out] (if the layer has a bias); for a DeepONet branch layers, trunk layers, then
 *    the scalar b0.  k-vectors are ordered by ascending flat index (idx order).
 *  - Chain-batched arrays are chain-major: theta[C x k], samples[C x S x k].
 *  - A context is bound to one CUDA device and is not thread-safe.
 */
#ifndef HMC_B200_H
#define HMC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------------- */
#define HMC_OK 0
#define HMC_E_CONFIG 1 /* bad shape, mask, sigma, argument or unsupported arch */
#define HMC_E_CUDA 3   /* a CUDA runtime / launch error */
#define HMC_E_NCCL 4   /* an NCCL error (data mode) */
#define HMC_E_OOM 5    /* device or pinned allocation failed */
#define HMC_E_STATE 6  /* call out of order (e.g. NULL context) */

/* ---- architecture ------------------------------------------------------------------------ */
enum { HMC_MLP = 0, HMC_DEEPONET = 1 };
enum { HMC_ACT_IDENTITY = 0, HMC_ACT_TANH = 1, HMC_ACT_SIN = 2 };
enum { HMC_MODE_SINGLE = 0, HMC_MODE_DATA = 1, HMC_MODE_CHAIN = 2 };
enum { HMC_SHARD_ROWS = 0, HMC_SHARD_POINTS_XB = 1, HMC_SHARD_POINTS_XC = 2 };

/* A feed-forward net with n_layers linear layers: widths[0] inputs ... widths[n_layers]
 * outputs; layer l applies act[l] to (W_l h + b_l).  Arrays are host memory, read at setup. */
typedef struct {
  int32_t n_layers;
  const int32_t* widths;   /* [n_layers + 1] */
  const int32_t* acts;     /* [n_layers] HMC_ACT_* */
  const int32_t* has_bias; /* [n_layers] 0/1 */
} hmc_net;

/* MLP: net[0] (output width must be 1).  DeepONet (Q14): net[0] = branch, net[1] = trunk,
 * equal output widths p; F(u, y) = sum_k B_k(u) T_k(y) + b0 (b0 present iff has_b0). */
typedef struct {
  int32_t kind;
  hmc_net net[2];
  int32_t has_b0;
} hmc_arch;

/* Training data D, fp32 row-major, host or device; copied in at setup, the caller may
 * free it on return.  MLP: x[n x d_in], y[n].  DeepONet (cartesian product layout, Q16):
 * u[n_c x m] branch inputs (function samples at the sensors), q[n_x x d_t] trunk inputs,
 * v[n_c x n_x] targets, pair (c, x) -> v[c * n_x + x].  q_per_pair = 1 selects the unaligned
 * DeepONet: every pair has its own query point, q[n_c x n_x x d_t]
 * (pair (c, x) -> row c * n_x + x), the trunk runs on all n_c * n_x points and the combine is a
 * row-wise dot (P:369 DeepONets).  In data mode these are this rank's
 * shard (a row block of x/y, or of u/v (and q when unaligned) for a DeepONet); n_global is the
 * sum over ranks. */
typedef struct {
  const float* x;
  const float* y;
  int64_t n;
  const float* u;
  const float* q;
  const float* v;
  int64_t n_c, n_x;
  int64_t n_global;
  int32_t q_per_pair; /* DeepONet: 0 = q[n_x x d_t] shared by all functions, 1 = q[n_c x n_x x d_t] */
} hmc_data;

typedef struct {
  const float* frozen;  /* [P] full flat mu; entries at idx are ignored (the state sets them) */
  const int32_t* idx;   /* [k] strictly ascending active flat indices, 1 <= k <= P */
  int64_t P, k;
  double noise_sigma;   /* likelihood sd sigma > 0 (Table 5 lists sigma^2, Q9) */
  double prior_sigma;   /* prior sd sigma_p > 0 on every active entry (Q8, Q10) */
  const float* inv_mass; /* [k] diagonal M^-1 (> 0) or NULL for identity (Q6) */
  uint64_t seed;        /* Philox key (Q23) */
  int32_t n_chains;     /* chains on this rank */
  const uint32_t* chain_ids; /* [n_chains] global chain ids keying Philox, or NULL = 0..C-1 */
  int32_t mode;         /* HMC_MODE_*; DATA needs world > 1 ranks sharing one chain set */
  int32_t rank, world;  /* this rank, number of ranks (1 for SINGLE / CHAIN) */
  int32_t shard;        /* DATA mode layout: HMC_SHARD_ROWS, or HMC_SHARD_POINTS_XB (DeepONet with
                           shared query points): this rank holds condition block r, u[n_c/world x m],
                           point block r, q[n_x x d_t], and v[n_c x n_x] for ALL n_c conditions and its
                           n_x points (hmc_data.n_c = all conditions, n_c % world == 0); the branch
                           outputs are all-gathered, dB reduce-scattered;
                           HMC_SHARD_POINTS_XC (DeepONet with shared query points): point block r of
                           q and v for the trunk and the combine, and the branch for chain block r
                           (n_chains / world chains) on ALL n_c conditions (u[n_c x m]; full-height
                           tiles at any world); the branch outputs of all chains are all-gathered,
                           dB reduce-scattered back to the chain owners */
  const uint8_t* nccl_id; /* [128] from hmc_comm_unique_id on rank 0 (DATA mode, world > 1) */
  int32_t exchange;     /* DATA mode: 0 = in-graph NCCL collectives (the product path); 1 = test hook,
                           no communicator: the context only runs hmc_debug_data_phase and the caller
                           performs the cross-rank steps (several ranks emulated on one GPU);
                           2 = timing stand-in, no communicator: the all-gather / reduce-scatter are
                           replaced by local copies of the same bytes and the all-reduce is skipped,
                           so one GPU can time one rank's share of a G-rank job (results are NOT
                           the data-mode posterior; scripts/project_scaling.py) */
} hmc_config;

typedef struct hmc_ctx hmc_ctx;

/* Rank 0 creates an NCCL unique id (128 bytes) to be broadcast to the other ranks. */
int hmc_comm_unique_id(uint8_t id_out[128]);

/* Validates arch/data/config (HMC_E_CONFIG with a message naming the field), uploads data,
 * frozen values and the mask, allocates all device workspace for n_chains chains, and (DATA
 * mode) creates the NCCL communicator.  Binds the context to the current CUDA device.
 * On success *out owns everything; release with hmc_destroy. */
int hmc_setup(const hmc_arch* arch, const hmc_data* data, const hmc_config* cfg, void* stream,
              hmc_ctx** out);

/* One full-batch gradient evaluation for every chain ("forward pass ... gradient
 * computation"): logp[c] = log pi(theta[c]) (constants dropped) in fp64 and
 * grad[c] = d log pi / d theta_s (ascent direction) in fp32.  theta [C x k] in, logp [C],
 * grad [C x k] out.  In DATA mode every rank receives identical values. */
int hmc_grad(hmc_ctx* ctx, const float* theta, double* logp, float* grad, void* stream);

/* Step-size adaptation ("the acceptance rate ... is fixed
 * at 80 % and the step size is computed using ... Algorithm 5 of" Hoffman & Gelman): n_adapt
 * trajectories (warm-up: the chain state theta / logp / grad advances exactly as in hmc_sample,
 * iter0 .. iter0 + n_adapt - 1), each chain running dual averaging on its own step size from
 * eps0 towards the acceptance statistic delta (gamma 0.05, t0 10, kappa 0.75; alpha =
 * min(1, exp(H0 - H*)), 0 for non-finite H*).  eps_bar [C] (host or device, fp64) receives
 * each chain's averaged step; the context keeps them, and hmc_trajectory / hmc_sample with
 * eps == 0 then use them per chain.  acc / dH [C x n_adapt] optional as in hmc_sample.
 * HMC_E_CONFIG if eps0 <= 0, delta outside (0, 1), n_adapt < 1. */
int hmc_adapt(hmc_ctx* ctx, float* theta, double* logp, float* grad, double eps0, int32_t L, int64_t iter0,
              int32_t n_adapt, double delta, double* eps_bar, uint8_t* acc, double* dH, void* stream);

/* Posterior predictive over the context's inputs (PAPER.md P:401 / P:480:
 * predictions "mean ± 3 standard deviations" over the HMC samples): for S samples of theta_s
 * (samples [S x k] fp32, host or device; the frozen entries stay at mu), mean[j] and var[j]
 * (population variance) of F(x_j) over the samples, fp64, for every datum j (MLP: the n rows;
 * DeepONet: the n_c x n_x pairs, row-major).  Predictions at new inputs: set up a context on
 * those inputs.  Runs the forward pass C samples at a time; synchronous.  HMC_E_CONFIG on NULL
 * arguments, S < 1 or a DATA-mode context. */
int hmc_predict(hmc_ctx* ctx, const float* samples, int64_t S, double* mean, double* var, void* stream);

/* Convergence diagnostics: split-R^ and effective sample
 * size per parameter (Gelman et al., BDA3 eqs. 11.3-11.8, on split chains: m = 2C half-chains of
 * n = S/2 draws; ESS truncated at the first odd lag T with rho_{T+1} + rho_{T+2} < 0).
 * samples [C x S x k] fp32 (host or device; the layout hmc_sample writes), rhat / ess [k] fp64
 * out (host or device).  Synchronous.  HMC_E_CONFIG unless 1 <= C <= 1024, S >= 4, k >= 1. */
int hmc_diagnostics(const float* samples, int32_t C, int64_t S, int64_t k, double* rhat, double* ess, void* stream);

/* Parameter sensitivities, the step before the hot path (Algorithm 2 "Compute: S_i^2",
 * PAPER.md eqn:sensitivities P:193-197):  S_i^2 = sigma_i^2 / N_d * sum_j (dF_mu(x_j)/dtheta_i)^2
 * for every flat parameter i (P = length of mu), gradients of the network OUTPUT at the VI mean
 * mu.  MLP: N_d = n rows; DeepONet: N_d = n_c * n_x pairs (u_c, y_x).
 * arch / data as for hmc_setup (data targets are not used); mu, sigma_vi [P] fp32 (host or
 * device, sigma_vi >= 0); s2 [P] fp64 out (host or device).  Synchronous: returns when s2 is
 * written.  Ranking and the tau threshold (eqn:threshold): hmc_partition.
 * HMC_E_CONFIG on invalid arguments (the same checks as hmc_setup), HMC_E_CUDA / HMC_E_OOM. */
int hmc_sensitivity(const hmc_arch* arch, const hmc_data* data, const float* mu, const float* sigma_vi,
                    double* s2, void* stream);

/* The tau-partition of the parameters by sensitivity (PAPER.md eqn:threshold P:200-204, §3.2
 * P:209-212): rank the P values s2 (>= 0) largest first, ties by ascending index, form the
 * cumulative fraction c_N of the ranked sum and pick N^ - rule 0 ("ge", the text's reading,
 * DESIGN.md §3): the smallest N with c_N >= tau (1e-15 relative slack); rule 1 ("le", the
 * equation as printed): the largest N with c_N <= tau.  N^ = 0 when sum s2 <= 0.  Writes the N^
 * selected flat indices in ascending order to active[0 .. N^) (host or device, capacity P; the
 * rest untouched) and N^ to *n_hat (host).  s2 [P] fp64 host or device.  Synchronous.
 * HMC_E_CONFIG unless 1 <= P < 2^31, 0 < tau <= 1, rule in {0, 1}; HMC_E_OOM / HMC_E_CUDA. */
int hmc_partition(const double* s2, int64_t P, double tau, int32_t rule, int32_t* active, int64_t* n_hat,
                  void* stream);

/* The dropped constant: -N log(sigma sqrt(2 pi)) - k log(sigma_p sqrt(2 pi)) (N = n_global or
 * n_c x n_x global), so logp + c is S:362's normalised value. */
int hmc_logpost_const(const hmc_ctx* ctx, double* c);

/* One Algorithm-2 iteration for every chain: momentum p ~ N(0, M) from Philox
 * (seed, tag 0, iter, chain_id) (Q23 / DESIGN §3), L kick-drift-kick steps of size eps with the
 * start gradient taken from `grad` (the cache), Metropolis test with u from Philox tag 1.
 * theta[C x k], logp[C], grad[C x k] are in/out: on accept they become the proposal's, on
 * reject they are unchanged.  acc[C] (0/1) and dH[C] = H* - H0 are outputs (either may be NULL).
 * L = 0 is the identity and always accepts.  eps must be finite and > 0 (or 0 after
 * hmc_adapt: each chain then uses its adapted step), L >= 0, 0 <= iter < 2^32. */
int hmc_trajectory(hmc_ctx* ctx, float* theta, double* logp, float* grad, double eps, int32_t L,
                   int64_t iter, uint8_t* acc, double* dH, void* stream);

/* Exactly S consecutive hmc_trajectory iterations iter0 .. iter0+S-1, replayed as one CUDA graph
 * per trajectory with no host round trip.  samples[C x S x k] (state after each iteration),
 * acc[C x S], dH[C x S] are outputs (acc / dH may be NULL).  Burn-in and thinning are the
 * caller's.  Resuming at iter0 + S with the returned state is bitwise identical to one call. */
int hmc_sample(hmc_ctx* ctx, float* theta, double* logp, float* grad, double eps, int32_t L,
               int64_t iter0, int32_t S, float* samples, uint8_t* acc, double* dH, void* stream);

/* Frees every resource of the context (NULL is a no-op). */
int hmc_destroy(hmc_ctx* ctx);

/* Context-owned message of the last failure (thread-local global when ctx == NULL). */
const char* hmc_last_error(const hmc_ctx* ctx);

/* ---- diagnostics used by tests and bench.py ---------------------------------------------- */

/* Counts of this library's kernel launches: per hmc_grad call, and per trajectory as
 * base + L * per_step. */
int hmc_launch_counts(const hmc_ctx* ctx, int64_t* per_grad, int64_t* per_traj_base,
                      int64_t* per_step);

/* Raw Philox4x32-10 words for counters (j, tag, iter, chain), j < nblocks, key from seed:
 * out[4 * j + w] (device or host pointer).  Used for the bitwise RNG agreement test. */
int hmc_philox_words(uint64_t seed, uint32_t tag, uint32_t iter, uint32_t chain, int64_t nblocks,
                     uint32_t* out, void* stream);

/* Momentum draw of `hmc_trajectory`: p[C x k] = sqrt(m) z for the given iter (fp32 out). */
int hmc_momentum(hmc_ctx* ctx, int64_t iter, float* p, void* stream);

/* Name of the GEMM engine used for each layer GEMM class ("simt" or "tcgen05"). */
const char* hmc_engine_info(const hmc_ctx* ctx);

/* Divergence diagnostic ("gradient explosion"; reading Q5): counts[c] (host or
 * device, uint32) = number of trajectories of chain c, since the context was created or last
 * reset, whose proposal energy was non-finite or had |H* - H0| > 1000 (SPEC S:445's threshold).
 * A flag only: such proposals are decided by the exact Metropolis test like any other (a
 * non-finite H* always rejects).  reset != 0 zeroes the counters after reading.  Synchronises
 * the context's stream.  HMC_E_CONFIG on NULL counts. */
int hmc_divergences(hmc_ctx* ctx, uint32_t* counts, int32_t reset);

/* Test hook: a DATA-mode gradient evaluation cut at its cross-rank steps, for contexts set up
 * with hmc_config.exchange = 1 (several ranks' contexts on ONE GPU, run one after another; the
 * caller does each collective on the host or with its own copies).  Device pointers; synchronous.
 *  phase 0: in = theta [C x k] f32.  ROWS: runs the rank's whole local evaluation, out = its
 *           likelihood gradient g_lik [C x k] f32, out2 = its sum of squared residuals [C] f64 (the
 *           all-reduce's inputs).  POINTS_XB: runs the forward of both nets, out = this rank's
 *           branch outputs [C x n_c/world x p] f32 (the all-gather's input).
 *  phase 1: POINTS_XB only: in = the all-gather result [world x C x n_c/world x p]; runs the
 *           combine / residual and the partial dB; out = the reduce-scatter input [world x C x
 *           n_c/world x p] (block r for rank r).
 *  phase 2: POINTS_XB only: in = this rank's reduce-scattered dB block [C x n_c/world x p]; runs
 *           dT and both nets' backward; out / out2 = g_lik / sum r^2 as in phase 0 (ROWS).
 *  phase 3: in / in2 = the all-reduced g_lik [C x k] / sum r^2 [C]; adds the prior once; out =
 *           grad [C x k] f32, out2 = log pi [C] f64 - what hmc_grad returns in DATA mode.
 * HMC_E_CONFIG on a context without exchange = 1, a bad phase or NULL buffers. */
int hmc_debug_data_phase(hmc_ctx* ctx, int32_t phase, const void* in, const void* in2, void* out, void* out2,
                         void* stream);
/* Test hook: the POINTS_XB permutations alone (device pointers, synchronous): dir 0 maps the
 * all-gather layout [rank][chain][i][k] to per-chain rows [chain][rank n_loc + i][k], dir 1 the
 * inverse (the reduce-scatter input).  HMC_E_CONFIG on bad arguments. */
int hmc_debug_xb_permute(int32_t dir, int32_t C, int32_t G, int64_t n_loc, int32_t p, const float* in, float* out,
                         void* stream);

/* Test hook, process-wide, read by hmc_setup: mode 0 = automatic (the narrow-network cluster
 * engine for MLPs that qualify, else tcgen05 wherever it takes the shape and SIMT elsewhere);
 * 1 = every GEMM on the per-layer SIMT FP32 engine; 2 = the per-layer dense engines only (no narrow
 * engine, no masked weight gradient); 3 = the narrow engine restricted to its cluster mode (no cooperative grid mode);
 * 4 = the per-layer engines with the masked weight gradient (sampled dense-dense kernel over the
 * mask's entries) on every hidden layer it takes, whatever the planner's cost model
 * would choose.  Returns HMC_E_CONFIG for any other mode.  Developer knobs of the tcgen05 engine (HMC_TC_* environment
 * variables: barrier profiles, timelines, A/B toggles) are compiled in only with -DHMC_DEV
 * (`make DEV=1`); the product library ignores the environment. */
int hmc_debug_set_engine(int32_t mode);

/* Live kernel timing.  hmc_profile(ctx, 1) makes the next trajectory graph capture CUDA event
 * nodes (cudaEventRecordExternal) around every kernel of the FIRST leapfrog step and around the
 * gradient-evaluation body of EVERY step; hmc_profile_read returns, for the most recently
 * replayed trajectory, one record per bracketed launch: kernel name, duration (ms), algorithmic
 * FLOPs and bytes of that launch, and the leapfrog step (-1 for begin / Metropolis).  Records
 * named "body" cover a whole gradient evaluation of step `step`.  Synchronises the context. */
typedef struct {
  char name[64];
  double ms;
  double flops;
  double bytes;
  int32_t step;
} hmc_prof_rec;
int hmc_profile(hmc_ctx* ctx, int32_t enable);

/* One chain-batched GEMM C[b] (M x N) = A[b] (M x K) . B[b] (K x N) on a chosen engine
 * (0 = SIMT FP32, 1 = tcgen05 3xTF32), no epilogue; device pointers, fp32 row-major with the
 * given leading dimensions and per-batch strides.  A(m,k) = A[m*lda+k] if a_kmajor else
 * A[k*lda+m]; B(k,n) = B[n*ldb+k] if b_kmajor else B[k*ldb+n].  HMC_E_CONFIG if the engine
 * does not take the shape.  Used by the engine unit tests. */
int hmc_debug_gemm(int32_t engine, int32_t a_kmajor, int32_t b_kmajor, int32_t M, int32_t N, int32_t K,
                   int32_t batch, const float* A, int64_t lda, int64_t sA, const float* B, int64_t ldb,
                   int64_t sB, float* C, int64_t ldc, int64_t sC, void* stream);
int hmc_profile_read(hmc_ctx* ctx, int32_t max_recs, hmc_prof_rec* out, int32_t* n_out);

/* Development diagnostics of the tcgen05 engine: with HMC_TC_PROF=1 in the environment at
 * hmc_setup time, every tensor-core GEMM adds, per CTA, the clock cycles each warp role spent
 * waiting on its pipeline barriers.  out[16 x 16] (host) receives the sums per kernel variant
 * (row = variant index of the engine's instantiation table; slot order: TMA waiting
 * for a free stage, MMA waiting for a free accumulator, MMA waiting for converted operands,
 * converter waiting for TMA, converter waiting for a free TMEM A slot, epilogue waiting for an
 * accumulator, epilogue waiting for prefetched tiles, epilogue output cycles, kernel cycles);
 * reset != 0 zeroes them.  Returns HMC_E_CUDA on a CUDA error. */
int hmc_debug_tc_profile(uint64_t* out, int32_t reset);
/* With HMC_TC_PROF=2: clock64 timeline of CTA 0 of the most recent tensor-core GEMM, out[24 x 256]
 * (host): per K block, MMA loop top / accumulator free / operands ready / issued, epilogue
 * partial ready / folded, converter A landed / operands published; rows 8-15: phases of converter
 * warp 0 (A split, slot free, TMEM store issued, B landed, B split, store done, fence, arrive);
 * rows 16-22: epilogue warp 0 (partial ready, folded, released, emitted; at the tile end: flushed,
 * biased / prefetch landed, parked). */
int hmc_debug_tc_timeline(uint64_t* out);
/* Developer build only (-DHMC_DEV, `make DEV=1`; HMC_E_STATE otherwise): clock cycles of CTA 0 of
 * the narrow-network engine per phase, out[10] (host): forward, output layer, push of the block
 * partials (+ the last input-gradient GEMM), cluster barrier 1, reduction + update, barrier 2,
 * tail, input gradients + loop overhead, weight gradients; reset != 0 zeroes them. */
int hmc_debug_nw_profile(uint64_t* out, int32_t reset);

#ifdef __cplusplus
}
#endif

#endif /* HMC_B200_H */
