/*
 * pssgp.h — C ABI of the B200-native parallel state-space GP hot path
 * (Corenflos, Zhao & Sarkka, "Temporal Gaussian Process Regression in
 * Logarithmic Time", arXiv:2102.09964).  Citations "PAPER.md:n" refer to the
 * paper text (main paper lines 1-249, supplement 249-480).
 *
 * The library computes, for a stationary GP written in state-space form
 * (Eq. (2)) on a SORTED time grid where test points are
 * MISSING observations (supplement PAPER.md:255):
 *   - the Kalman filter via the associative scan of filter elements
 *     (A, b, C, eta, J), including the paper's missing-measurement elements
 *     (Eqs. (6)-(8); Prop. 1),
 *   - the RTS smoother via the reverse associative scan of (E, g, L)
 *     (Prop. 2),
 *   - the negative log marginal likelihood (named PAPER.md:75, 144, 157;
 *     evaluated by the predictive decomposition, reading Z3 in DESIGN.md),
 *   - posterior mean/variance of the latent f = H x.
 * All arithmetic is IEEE fp64.  Every step runs in CUDA kernels for sm_100a;
 * there is no CPU fallback.
 *
 * Conventions for every call below:
 *   - Array pointers are CUDA DEVICE pointers owned by the caller unless the
 *     function name ends in _host.  Nothing is retained after the call.
 *   - t[N]: fp64, finite, NON-DECREASING (ties allowed: dt = 0 -> F = I,
 *     Q = 0; reading Z13).  Decreasing / non-finite t -> PSSGP_E_INPUT with
 *     the first failing index (pssgp_error_index).
 *   - mask[N]: uint8; nonzero = observed, 0 = missing (test point).
 *   - y[N]: fp64; read only where mask != 0 (NaN allowed elsewhere); an
 *     observed non-finite y -> PSSGP_E_INPUT.
 *   - Outputs mean[N], var[N]: fp64 posterior mean and variance of f at every
 *     grid point (observed and missing).  nll: ONE fp64 device scalar,
 *     sum over observed k of 0.5 (log(2 pi S_k) + v_k^2 / S_k).
 *   - Calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *     default stream).  Host-detectable errors are returned immediately;
 *     device-detected errors (non-finite data, S <= 0, non-PD predicted
 *     covariance) are latched in the handle and returned by pssgp_check().
 *   - A handle may be used by one stream at a time; distinct handles are
 *     independent.  Workspace grows on demand and is owned by the handle.
 */
#ifndef PSSGP_H
#define PSSGP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pssgp_model pssgp_model;   /* opaque */

typedef enum {
    PSSGP_OK = 0,
    PSSGP_E_ARG = 1,          /* bad argument (NULL, N < 0, noise_var <= 0, bad hyper-parameter) */
    PSSGP_E_INPUT = 2,        /* bad data: unsorted / non-finite t, non-finite observed y */
    PSSGP_E_NUMERIC = 3,      /* S <= 0, non-PD predicted covariance, non-finite intermediate */
    PSSGP_E_CUDA = 4,         /* CUDA runtime error (see pssgp_last_error) */
    PSSGP_E_NOMEM = 5,        /* device or host allocation failed */
    PSSGP_E_UNSUPPORTED = 6   /* kernel combination / state dim / irregular dt not supported */
} pssgp_status;

typedef enum {
    PSSGP_MATERN12 = 1,       /* d = 1, exact                                   */
    PSSGP_MATERN32 = 2,       /* d = 2, exact                                                  */
    PSSGP_MATERN52 = 3,       /* d = 3, exact                                                  */
    PSSGP_RBF_TAYLOR = 4,     /* d = order, Taylor approximation of 1/S(w) */
    PSSGP_PERIODIC = 5,       /* d = 2 (order + 1) harmonic oscillators        */
    PSSGP_QUASIPERIODIC = 6   /* periodic(order) x Matern-(mat_nu2/2): d = 2 (order + 1) m,
                                 m = (mat_nu2 + 1) / 2 (CO2 model) */
} pssgp_kind;

/* One additive component of the covariance (sum of components = block-diagonal
 * state).  variance = sigma^2 > 0, lengthscale > 0, period > 0
 * (periodic, quasi-periodic), order >= 1 (RBF Taylor order / periodic harmonics J).
 * Quasi-periodic only: mat_lengthscale > 0 and mat_nu2 in {1, 3, 5} describe the
 * Matern factor (unit variance; the product's variance is `variance`). */
typedef struct {
    int kind;                 /* pssgp_kind */
    double variance;
    double lengthscale;
    double period;
    int order;
    double mat_lengthscale;
    int mat_nu2;
} pssgp_component;

typedef struct {
    int balance;              /* 1 (default): Osborne balancing, Eq. (9) */
    int device;               /* CUDA device ordinal used for workspace (default: current) */
    double uniform_dt;        /* > 0: steps with |t[k]-t[k-1] - uniform_dt| <= 1e-12 uniform_dt
                                 (time-stamp rounding) use F, Q precomputed on the host (fp64
                                 result of an extended-precision Van Loan); 0 = none.
                                 Non-Matern models (no closed form):
                                   > 0 -> only dt = uniform_dt or 0 allowed, other steps fail
                                          with PSSGP_E_UNSUPPORTED (pure uniform grids);
                                   = 0 -> any dt: per-step F = expm(G dt) by scaling and
                                          squaring on the device and Q by the Taylor series
                                          of the Lyapunov ODE on the scaled step composed by
                                          doubling (north_star discretisation kernel; d > 3
                                          stores (F, Q) per step in a handle-owned buffer of
                                          N 2 d (d+1) doubles). */
    int64_t chain_len;        /* steps per thread chain (0 = automatic)                   */
    int blocks_per_sm;        /* CTAs per SM for the one-wave grid (0 = automatic)        */
} pssgp_options;

/* Build the continuous SSM (G, L, q, H, P_inf) of the summed kernel, balance it,
 * and (if opt->uniform_dt > 0) discretise it once.  Host only; no device work
 * until the first compute call.  opt may be NULL (defaults).  On success *out
 * receives a new handle.  Errors: PSSGP_E_ARG (bad hyper-parameters, n_comps < 1,
 * noise_var <= 0), PSSGP_E_UNSUPPORTED (state dimension > the compiled maximum),
 * PSSGP_E_NUMERIC (singular Lyapunov system). */
pssgp_status pssgp_create(const pssgp_component* comps, int n_comps, double noise_var,
                          const pssgp_options* opt, pssgp_model** out);

void pssgp_destroy(pssgp_model* m);

/* State dimension d = n_x. */
int pssgp_state_dim(const pssgp_model* m);

/* Filter + smoother + NLL over one grid (the hot path).  mean, var: device
 * arrays of N doubles (may both be NULL -> smoother skipped); nll: device
 * scalar or NULL.  N = 0 is allowed (nll = 0). */
pssgp_status pssgp_posterior(pssgp_model* m, int64_t N, const double* t, const double* y,
                             const uint8_t* mask, double* mean, double* var, double* nll,
                             void* stream);

/* NLL only: forward filter pass (no filtered state stored, no smoother). */
pssgp_status pssgp_nll(pssgp_model* m, int64_t N, const double* t, const double* y,
                       const uint8_t* mask, double* nll, void* stream);

/* Optional fp32 path (north_star "an optional fp32 path must match to 1e-3"):
 * the same filter / smoother / NLL as pssgp_posterior (Prop. 1-2) with
 * the state algebra (moments, aggregates, F, Q) and the filtered state in HBM in fp32.  Times,
 * observations, mean / var outputs and the NLL accumulation stay fp64 (fp32 ulp at t ~ 2048
 * exceeds the step).  Same arguments, layout, ownership and stream semantics as
 * pssgp_posterior; mean and var may both be NULL (NLL only: no filtered state stored, no
 * smoother).  Accuracy ~1e-4 relative on the Matern workloads (tests/test_gpu_f32.py, bar 1e-3).
 * Single Matern components only (fp32 misses 1e-3 for the d = 16 sum)
 * -> else PSSGP_E_UNSUPPORTED. */
pssgp_status pssgp_posterior_f32(pssgp_model* m, int64_t N, const double* t, const double* y,
                                 const uint8_t* mask, double* mean, double* var, double* nll, void* stream);

/* NLL and its exact gradient with respect to the log hyper-parameters theta (the gradient the
 * paper obtains by automatic differentiation of the parallel filter; its
 * L-BFGS / HMC workloads).  theta, in this order (pssgp_num_params entries):
 * for each component in the order given to pssgp_create
 *     Matern-nu, RBF-Taylor:  log variance, log lengthscale
 *     periodic:               log variance, log lengthscale, log period
 *     quasi-periodic:         log variance, log lengthscale, log period, log mat_lengthscale
 * then log noise_var.  The model basis (balancing matrix D, Eq. (9); the Matern lambda-scaling) is
 * treated as constant ("D treated as constant"), which leaves the gradient exact.
 *   - One Matern component (any grid): forward-mode tangents of the Kalman recursion (supplement
 *     PAPER.md:304-315) composed as affine maps per thread chain (pssgp_grad.cuh).
 *   - Any other model (sums, RBF, periodic, quasi-periodic products): reverse mode - the adjoint
 *     of the Kalman recursion is an affine backward recursion whose per-chain maps compose in
 *     closed form; forward rescan composing them, reverse scan, backward rescan, contraction with
 *     dF/dtheta, dQ/dtheta (exact Van Loan tangents at the uniform step) and dP_inf/dtheta
 *     (pssgp_wide.cuh).  Needs options.uniform_dt > 0 (every step of length
 *     uniform_dt or 0), else PSSGP_E_UNSUPPORTED.
 * nll: device scalar or NULL; grad: device array of pssgp_num_params(m) doubles.  N = 0 -> nll = 0,
 * grad = 0. */
pssgp_status pssgp_nll_grad(pssgp_model* m, int64_t N, const double* t, const double* y,
                            const uint8_t* mask, double* nll, double* grad, void* stream);

/* Number of hyper-parameters of the model (length of pssgp_nll_grad's grad; see its order). */
int pssgp_num_params(const pssgp_model* m);

/* End-to-end variant on HOST arrays (pinned memory recommended): copies the
 * inputs to handle-owned device buffers, runs pssgp_posterior, copies mean,
 * var (nullable) and *nll (nullable) back, and synchronises the stream.
 * Returns device-detected errors directly. */
pssgp_status pssgp_posterior_host(pssgp_model* m, int64_t N, const double* t, const double* y,
                                  const uint8_t* mask, double* mean, double* var, double* nll,
                                  void* stream);

/* Merge sorted training times t_train[n_train] (with y_train) and sorted test
 * times t_test[n_test] into one sorted grid (pipeline stage 4,
 * P:171; test points = missing observations, supplement P:255): t_out, y_out
 * (0 at test points), mask_out (1 train / 0 test) of n_train + n_test entries,
 * and test_index[j] = position of test time j in the grid.  Training first on
 * ties.  Device arrays, caller-owned.  Unsorted / non-finite times are reported
 * by pssgp_check as PSSGP_E_INPUT (index n_train + j for test time j). */
pssgp_status pssgp_merge_grid(pssgp_model* m, int64_t n_train, const double* t_train, const double* y_train,
                              int64_t n_test, const double* t_test, double* t_out, double* y_out,
                              uint8_t* mask_out, int64_t* test_index, void* stream);

/* mean_test[j] = mean[test_index[j]], var_test[j] = var[test_index[j]] (either
 * output may be NULL).  Device arrays. */
pssgp_status pssgp_gather(pssgp_model* m, int64_t n_test, const int64_t* test_index, const double* mean,
                          const double* var, double* mean_test, double* var_test, void* stream);

/* The paper's prediction pipeline in one call: merge (handle-
 * owned grid buffers), filter + smoother + NLL on the merged grid, gather the
 * test outputs.  nll (device scalar, nullable) is the training NLL (test points
 * are missing observations and do not contribute). */
pssgp_status pssgp_predict(pssgp_model* m, int64_t n_train, const double* t_train, const double* y_train,
                           int64_t n_test, const double* t_test, double* mean_test, double* var_test,
                           double* nll, void* stream);

/* Batched independent problems: nseg series concatenated
 * along the time axis, series b = steps [offsets[b], offsets[b+1]) (offsets: device
 * int64[nseg + 1], offsets[0] = 0, offsets[nseg] = N, non-decreasing; empty series
 * allowed).  Times must be non-decreasing within a series; each series restarts
 * from the stationary prior (its first element is Eq. (7)'s).  Per-series Matern
 * hyper-parameters variance[b], lengthscale[b], noise_var[b] (device fp64 arrays;
 * NULL = the model's value).  Outputs mean[N], var[N] (device) and nll[nseg]
 * (device, per-series NLL, fixed-order sums).  Only single-component Matern
 * models (closed-form discretisation) -> else PSSGP_E_UNSUPPORTED. */
pssgp_status pssgp_posterior_batched(pssgp_model* m, int nseg, const int64_t* offsets, const double* variance,
                                     const double* lengthscale, const double* noise_var, int64_t N,
                                     const double* t, const double* y, const uint8_t* mask, double* mean,
                                     double* var, double* nll, void* stream);

/* Batched NLL + gradient (NEXT rows f1 x f2: the paper's multi-start / HMC workloads,
 * PAPER.md:206-209, 224): the series and per-series hyper-parameters of
 * pssgp_posterior_batched; outputs nll[nseg] and grad[3 nseg] (device; grad[3b..3b+2] =
 * d NLL_b / d (log sigma_b^2, log ell_b, log sigma_n,b^2)).  The tangent aggregates restart
 * at every series start; series spanning several chains are composed from per-chain pieces
 * (pssgp_grad.cuh).  Only single-component Matern models -> else PSSGP_E_UNSUPPORTED. */
pssgp_status pssgp_nll_grad_batched(pssgp_model* m, int nseg, const int64_t* offsets, const double* variance,
                                    const double* lengthscale, const double* noise_var, int64_t N,
                                    const double* t, const double* y, const uint8_t* mask, double* nll,
                                    double* grad, void* stream);

/* Batched independent series with PER-SERIES log hyper-parameters for any sum of Matern,
 * periodic and quasi-periodic components on a uniform grid (SURVEY.md §8(f) row 2 widened: HMC
 * chains / multi-start fits on the paper's CO2 model).  The model m
 * gives the structure (components, orders, uniform_dt > 0); theta (device, nseg x
 * pssgp_num_params(m), row b = series b, the order of pssgp_nll_grad) replaces its
 * hyper-parameters per series.  Series b = steps [offsets[b], offsets[b+1]) (device int64[nseg+1],
 * non-decreasing, offsets[nseg] = N); each starts from its stationary prior; steps inside a series
 * are uniform_dt apart or ties (dt = 0), else PSSGP_E_UNSUPPORTED from pssgp_check.  The per-series
 * F, Q, P_inf and their theta-derivatives are closed forms built on the device
 * (pssgp_batch_theta.cuh); one warp runs each series' sequential Kalman filter and then the RTS
 * smoother in its solve-free adjoint form / the reverse-mode adjoint of the filter (series share
 * nothing, so no scan).  Outputs (device): mean[N], var[N]
 * (nullable), nll[nseg], grad[nseg x pssgp_num_params].  RBF components -> PSSGP_E_UNSUPPORTED. */
pssgp_status pssgp_posterior_batched_theta(pssgp_model* m, int nseg, const int64_t* offsets,
                                           const double* theta, int64_t N, const double* t,
                                           const double* y, const uint8_t* mask, double* mean,
                                           double* var, double* nll, void* stream);
pssgp_status pssgp_nll_grad_batched_theta(pssgp_model* m, int nseg, const int64_t* offsets,
                                          const double* theta, int64_t N, const double* t,
                                          const double* y, const uint8_t* mask, double* nll,
                                          double* grad, void* stream);

/* Synchronise the handle's last stream and return the first device-detected
 * error (PSSGP_E_INPUT / PSSGP_E_NUMERIC / PSSGP_E_UNSUPPORTED) since the last
 * pssgp_check, or PSSGP_OK.  Clears the latched error. */
pssgp_status pssgp_check(pssgp_model* m);

/* Index of the time step that caused the last error returned by pssgp_check
 * (or by a host-side check), -1 if none. */
int64_t pssgp_error_index(const pssgp_model* m);

/* Human-readable description of the last error (static storage of the handle). */
const char* pssgp_last_error(const pssgp_model* m);

/* Pipelined variant of pssgp_posterior_host for streams of problems: enqueues the host ->
 * device copies, pssgp_posterior and the device -> host copies on one of two handle-owned
 * streams (alternating per call) and returns immediately, so one call's device -> host copies
 * overlap the next call's host -> device copies (PCIe is full duplex); the computes run in call
 * order.  Host arrays must be PINNED and stay untouched until pssgp_sync returns; the two most
 * recent calls may be in flight.  Host-detectable errors are returned immediately. */
pssgp_status pssgp_posterior_host_async(pssgp_model* m, int64_t N, const double* t, const double* y,
                                        const uint8_t* mask, double* mean, double* var, double* nll);

/* Wait for every pssgp_posterior_host_async call of the handle; returns the first
 * device-detected error (as pssgp_check). */
pssgp_status pssgp_sync(pssgp_model* m);

/* Copy the host-side balanced model: G, W = L q L^T, P_inf (d*d row-major),
 * H (d), D (d, balancing diagonal; z = D^-1 x).  Any pointer may be NULL. */
pssgp_status pssgp_get_ssm(const pssgp_model* m, double* G, double* W, double* H,
                           double* Pinf, double* D);

/* The (F, Q) the device code uses for a step of length dt.  d <= 3: evaluated on
 * the host by the same __host__ __device__ function the kernels call (closed form
 * for Matern, the precomputed pair for dt == uniform_dt, the scaled-step series for
 * uniform_dt = 0).  d > 3 with uniform_dt = 0: ONE step of the device kernel
 * kw_discretize (needs a GPU).  F, Q: d*d row-major.  Test/introspection only;
 * returns PSSGP_E_UNSUPPORTED where the device would. */
pssgp_status pssgp_debug_discretize(const pssgp_model* m, double dt, double* F, double* Q);

/* Launch plan for N steps: steps per chain, number of chains, CTAs, threads/CTA. */
pssgp_status pssgp_plan(pssgp_model* m, int64_t N, int64_t* chain_len, int64_t* n_chains,
                        int* n_blocks, int* threads_per_block);
/* The same for pssgp_posterior_f32 (its kernels' occupancy); PSSGP_E_UNSUPPORTED for models
 * the fp32 path does not cover. */
pssgp_status pssgp_plan_f32(pssgp_model* m, int64_t N, int64_t* chain_len, int64_t* n_chains,
                            int* n_blocks, int* threads_per_block);

/* Optional per-kernel timing with CUDA events recorded on the launch stream.
 * pssgp_profile_enable(m, 1) starts recording; pssgp_profile_read synchronises
 * and returns, per kernel slot (see pssgp_profile_name), the summed elapsed
 * milliseconds and launch counts since the last read, then resets.
 * Returns the number of slots written (<= cap). */
void pssgp_profile_enable(pssgp_model* m, int on);
int pssgp_profile_read(pssgp_model* m, double* ms, int64_t* launches, int cap);
const char* pssgp_profile_name(int slot);

/* Measurement helper (the fp64 roofline denominator): DFMA throughput of the
 * handle's device in TFLOP/s (FMA = 2 flop), best of three runs each of two probe kernels (8
 * independent FMA chains per thread, 8 CTAs of 256 threads per SM; register or constant-bank
 * addend).  Synchronous (default stream); ~10 ms.  *tflops: host double. */
pssgp_status pssgp_measure_fp64_peak(pssgp_model* m, double* tflops);

/* ---- Time-sharded path (multi-GPU, one process per GPU).
 * Rank g owns the contiguous chunk [k0, k0 + n) of a global grid of N_global
 * steps.  t points at the chunk's first element and t[-1] (if k0 > 0) and
 * t[n] (if k0 + n < N_global) must be readable (one-point halo each side);
 * y, mask point at the chunk's first element.  Aggregates are opaque byte
 * blobs of pssgp_aggregate_bytes(m, which) bytes (which = 0 filter, 1
 * smoother + NLL partial) in DEVICE memory; the caller all-gathers them (e.g. NCCL) into
 * arrays ordered by rank.  The three calls must be made in order with the
 * same chunk arguments; the handle keeps the filtered state in between. */
size_t pssgp_aggregate_bytes(const pssgp_model* m, int which);

pssgp_status pssgp_shard_filter_reduce(pssgp_model* m, int64_t k0, int64_t n, int64_t N_global,
                                       const double* t, const double* y, const uint8_t* mask,
                                       void* filt_agg_out, void* stream);

/* all_filt_aggs: world filter aggregates; the carry into this chunk is the
 * ordered product of ranks 0..rank-1 (any grouping P:326).
 * Writes this chunk's smoother blob (pssgp_aggregate_bytes(m, 1) bytes: the chunk's
 * smoother aggregate followed by its NLL partial) and, if nll_partial != NULL, the
 * partial alone (device scalar). */
pssgp_status pssgp_shard_filter_apply(pssgp_model* m, int64_t k0, int64_t n, int64_t N_global,
                                      const double* t, const double* y, const uint8_t* mask,
                                      const void* all_filt_aggs, int rank, int world,
                                      void* smooth_agg_out, double* nll_partial, void* stream);

/* all_smooth_aggs: world smoother blobs in rank order; the carry into this chunk is
 * the ordered product of ranks rank+1..world-1.  Writes mean[n],
 * var[n] and, if nll != NULL, the TOTAL NLL of the global grid into the device scalar
 * *nll: the fixed-order sum over ranks 0..world-1 of the NLL partials carried in the
 * blobs (deterministic; identical on every rank). */
pssgp_status pssgp_shard_smoother_apply(pssgp_model* m, int64_t k0, int64_t n, int64_t N_global,
                                        const double* t, const void* all_smooth_aggs, int rank,
                                        int world, double* mean, double* var, double* nll,
                                        void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PSSGP_H */
