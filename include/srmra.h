/*
 * srmra.h — C ABI of libsrmra.so: B200-native (sm_100a) projected EM for 2-D super-resolution
 * multi-reference alignment (Shani, Giryes, Bendory, arXiv 2204.04754).
 *
 * The problem statement the arguments mirror (§I eq:model_1 and its explicit
 * form):   y_i[n1,n2] = x[(n1 K - s_i^1) mod L_high, (n2 K - s_i^2) mod L_high] + eps_i[n1,n2],
 *          i = 1..N, n in Z_{L_low}^2, K = L_high / L_low an integer, eps ~ N(0, sigma^2) i.i.d.,
 *          s^1 ~ rho1, s^2 ~ rho2 i.i.d..  theta = (x, rho1, rho2).
 *
 * One call of srmra_em_iter(ctx, 1) is one iteration of Algorithm 2:
 *   E-step  eq:weights_EM over all N observations and all L_high^2 shifts,
 *   M-step  eq:x_EM (P^{-1} read as P^T so A is diagonal) and eq:rho_EM
 *           (separable marginals: rho1'[s1] = sum_{s2} sum_i w^{i,s} / sum w),
 *   the log-likelihood eq:likelihood_EM ("up to a constant": the Gaussian
 *           normaliser is omitted) at the iteration's INPUT theta,
 *   and, every proj_every-th iteration, the projection x <- D(x) with the fixed
 *           stand-in denoiser D = 3x3 circular box filter followed by clamping to [-1, 1].
 * Shifts are s = (s1, s2) in Z_{L_high}^2, s1 acting on the first (row) index; flattened
 * row-major s = s1 * L_high + s2.  All arrays are row-major and C-contiguous.
 *
 * Ownership: the caller owns every host buffer passed in or out; srmra_init / srmra_load copy
 * their inputs into library-owned device memory, so the caller may free them on return.  The
 * context owns all device memory, its stream (unless one was supplied) and the NCCL
 * communicator until srmra_free.  A context is not thread-safe; separate contexts are
 * independent.  No C++ exception crosses this ABI.
 *
 * Errors: every int-returning call returns SRMRA_OK (0) or a negative SRMRA_ERR_* code and
 * records a message readable with srmra_last_error(ctx) (ctx == NULL: the calling thread's last
 * srmra_init failure).  After SRMRA_ERR_CUDA / SRMRA_ERR_NCCL the context is failed and every
 * later call returns SRMRA_ERR_STATE.
 */
#ifndef SRMRA_H_
#define SRMRA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SRMRA_API __attribute__((visibility("default")))
#else
#define SRMRA_API
#endif

#define SRMRA_OK 0
#define SRMRA_ERR_INVALID_ARG (-1) /* K*L_low != L_high, size <= 0, sigma <= 0 or non-finite, non-finite
                                      y/x0/rho, rho negative or |sum rho - 1| > 1e-6, bad option    */
#define SRMRA_ERR_UNSUPPORTED (-2) /* shape outside the compiled specialisations / no sm_100 device  */
#define SRMRA_ERR_CUDA (-3)
#define SRMRA_ERR_NCCL (-4)
#define SRMRA_ERR_OOM (-5)
#define SRMRA_ERR_STATE (-6)       /* call on a failed context, or em_iter after a rejected srmra_load */
#define SRMRA_ERR_NUMERIC (-7)     /* non-finite log-likelihood or estimate detected by finalize      */

/* E-step / M-step implementation ("path") */
#define SRMRA_PATH_AUTO 0   /* per-shape choice from measurement ("Path choice")        */
#define SRMRA_PATH_GEMM 1   /* S = Y T(x)^T and Z = W^T Y on tcgen05 tensor cores, 3xTF32             */
#define SRMRA_PATH_FFT 2    /* batched polyphase FFT correlation (K^2 correlations of L_low x L_low)  */
#define SRMRA_PATH_DIRECT 3 /* direct SIMT correlation (small shapes)                                 */

typedef struct srmra_ctx srmra_ctx; /* opaque, owned by the library */

/*
 * Exchange provider for world > 1 (a6 of SURVEY.md §8: the sums over i of eq:x_EM, eq:rho_EM and
 * eq:likelihood_EM, over the ranks' shards).  Called on the host in place
 * of ncclAllReduce(sum, float64) with the device buffer buf_dev (float64 [n], this rank's partial sums on
 * entry, the sum over all ranks on return) and the context stream (cudaStream_t): the input is complete
 * once the work enqueued on `stream` before the call has finished, and the result must be visible to the
 * work enqueued on `stream` after the hook returns (e.g. synchronise the stream, exchange, copy back and
 * synchronise again).  Every rank calls it the same number of times with the same n.  Return 0 on success;
 * non-zero fails the call with SRMRA_ERR_NCCL.  Use: host transports (gloo / MPI), tests that run several
 * ranks on one GPU.  With a provider set, the iteration is never captured in a CUDA graph.
 */
typedef int (*srmra_allreduce_fn)(double* buf_dev, uint64_t n, void* stream, void* user);

typedef struct {
    int32_t path;        /* SRMRA_PATH_*; default AUTO                                              */
    int32_t proj_every;  /* F: project after iteration t (0-based, counted over the context's life)
                            when (t+1) % F == 0; 0 = never; default 1                                */
    double floor_tau;    /* pixel p keeps x_t[p] when its coverage A[p] <= floor_tau;
                            < 0 selects the default 1e-12 * N_global                                 */
    int32_t device;      /* CUDA ordinal; < 0 = the calling thread's current device                 */
    int32_t rank;        /* this process's rank in [0, world)                                         */
    int32_t world;       /* number of ranks sharing the observations; 1 = no NCCL                     */
    const void* nccl_id; /* world > 1: the 128-byte ncclUniqueId from srmra_nccl_unique_id() on rank 0,
                            broadcast by the caller (e.g. torch.distributed); ignored if world == 1  */
    void* stream;        /* cudaStream_t to enqueue on, or NULL: the context creates its own          */
    int32_t trace_cap;   /* capacity of the on-device log-likelihood trace; default 4096              */
    srmra_allreduce_fn allreduce; /* world > 1: exchange provider used instead of NCCL (nccl_id is then
                            ignored); NULL = NCCL                                                     */
    void* allreduce_user; /* passed to `allreduce` unchanged                                           */
    int32_t grid_cap;    /* upper bound on the persistent E/M grid of the FFT path (CTAs; clusters at
                            L_low = 128), so that each CTA walks several observations even at small
                            n_local (test hook of the persistent loop); <= 0 = one per SM (default)    */
    int32_t nccl_timeout_ms; /* world > 1 with NCCL: a synchronising call that waits longer than this for
                            the stream while ncclCommGetAsyncError reports no error aborts the
                            communicator and fails with SRMRA_ERR_NCCL; <= 0 = wait without limit
                            (errors reported by NCCL still abort); default 0                          */
} srmra_options;

/* Fill *opt with the defaults above. */
SRMRA_API void srmra_default_options(srmra_options* opt);

/*
 * Create a context for this rank's shard of the observations and stage theta_0.
 *   y       host, float32 [n_local][L_low][L_low]: observations y_i of this rank (copied); or NULL:
 *           no observations yet — the context returns STATE from the iteration / moment calls until
 *           srmra_load or srmra_generate supplies them.
 *   n_local number of observations on this rank (>= 0; the global N is the sum over ranks).
 *   L_high, L_low, K   image side, observation side, K = L_high / L_low (must hold exactly).
 *   sigma   noise standard deviation (> 0, finite), known.
 *   x0      host, float32 [L_high][L_high]: initial image estimate (copied).
 *   rho1_0, rho2_0   host, float64 [L_high]: initial shift marginals (>= 0, each summing to 1
 *           within 1e-6; renormalised in float64).
 *   opt     NULL for defaults.
 * Errors: INVALID_ARG, UNSUPPORTED, CUDA, NCCL, OOM.  On error *out is NULL.
 */
SRMRA_API int srmra_init(srmra_ctx** out, const float* y, int32_t n_local, int32_t L_high, int32_t L_low,
               int32_t K, double sigma, const float* x0, const double* rho1_0, const double* rho2_0,
               const srmra_options* opt);

/* Replace the observations (same n_local and shape) and theta with new host data, reusing the
 * context's device memory; resets the iteration counter and the trace.  y is validated on the device
 * (finite): a rejected y returns INVALID_ARG and leaves the context requiring a successful srmra_load
 * before the next srmra_em_iter (which returns STATE until then). */
SRMRA_API int srmra_load(srmra_ctx* ctx, const float* y, const float* x0, const double* rho1_0,
               const double* rho2_0);

/* srmra_load followed by n_iters EM iterations (Algorithm 2's EM steps; eq:weights_EM,
 * eq:x_EM, eq:rho_EM), with the upload overlapped: on the FFT path with one rank and no
 * denoiser hook, the first iteration's E-step / M-step runs per observation range as soon as that range's
 * host->device copy has landed, while the next range is still being copied (pass y in pinned host memory for
 * an asynchronous copy).  Arguments and errors as srmra_load and srmra_em_iter; synchronous (returns after the
 * first iteration, with the later n_iters - 1 enqueued).  The result equals srmra_load + srmra_em_iter(n_iters)
 * up to the float32 rounding of the per-CTA partial sums (the partials are grouped by range).  Other paths /
 * world > 1 / a denoiser hook: exactly srmra_load + srmra_em_iter(n_iters). */
SRMRA_API int srmra_load_iterate(srmra_ctx* ctx, const float* y, const float* x0, const double* rho1_0,
               const double* rho2_0, int32_t n_iters);

/*
 * NEXT-4 device data generator: like srmra_load, but the n_local observations are drawn on the GPU from
 * the model of PAPER.md:37-38 (eq:model_1), y_j[n1, n2] = x[(n1 K - s^1) mod L_high, (n2 K - s^2) mod
 * L_high] + sigma z, for the global observation indices j = first_index .. first_index + n_local - 1
 * (ranks pass their offset, so the union over ranks equals the one-rank data set), sigma the context's.
 * Counter-based: Philox4x32-10 with key (seed mod 2^32, seed >> 32).  Shifts: counter (j mod 2^32,
 * j >> 32, 0, 0) -> words (u0, u1); s^1 = min{k : (u0 + 0.5) 2^-32 < C1[k]}, C1 the sequential float64
 * partial sums of rho1_true as given (clamped to the last k with positive mass), s^2 likewise from u1
 * and rho2_true.  Noise: counter (j mod 2^32, j >> 32, 1 + b, 0) -> (r0..r3), V = ((r >> 9) + 0.5) 2^-23 (exact in float32),
 * Box-Muller z = sqrt(-2 ln V0) (cos, sin)(2 pi V1), sqrt(-2 ln V2) (cos, sin)(2 pi V3) for pixels
 * 4b .. 4b+3 (row-major), evaluated in float32 (logf, sqrtf, sincospif).  synth/philox.py is the
 * reference.  x_true: host float32 [L_high][L_high]; rho*_true, rho*_0: host float64 [L_high] (>= 0,
 * sum 1 within 1e-6); x0 / rho*_0 the initial estimate as in srmra_load; shifts_out: host int32
 * [n_local][2] (s^1, s^2) or NULL.  Resets the iteration counter and trace.  Synchronises.
 * Errors: INVALID_ARG (NULL, first_index < 0, non-finite, bad pmf), STATE, CUDA.
 */
SRMRA_API int srmra_generate(srmra_ctx* ctx, const float* x_true, const double* rho1_true, const double* rho2_true,
                             uint64_t seed, int64_t first_index, const float* x0, const double* rho1_0,
                             const double* rho2_0, int32_t* shifts_out);

/* Test hook: copy observations first .. first + count - 1 of this rank (float32 [count][L_low][L_low],
 * caller-owned host buffer) as the device holds them (e.g. after srmra_generate).  Synchronises.
 * Errors: INVALID_ARG (range outside [0, n_local), NULL), STATE, CUDA. */
SRMRA_API int srmra_get_observations(srmra_ctx* ctx, int64_t first, int64_t count, float* y_out);

/* Enqueue n_iters >= 0 EM iterations on the context stream; asynchronous (no host sync).
 * With world > 1 each iteration performs one all-reduce (NCCL, or the options' exchange provider) of the
 * sufficient statistics: FFT path the compact float64 frequency-domain accumulators (+ the per-shift
 * posterior mass with a joint prior); GEMM / direct paths the packed b | class mass | marginals | LL
 * (+ the per-shift posterior mass with a joint prior).  FFT path with NCCL: one iteration (E/M kernel,
 * reduce, ncclAllReduce, fold / finalize / projection / prep) is captured once into a CUDA graph and
 * replayed. */
SRMRA_API int srmra_em_iter(srmra_ctx* ctx, int32_t n_iters);

/* NEXT-3: a joint (non-separable) shift prior rho[s1 L_high + s2] (host, float64, [L_high][L_high],
 * >= 0, summing to 1 within 1e-6; copied) replaces (rho1, rho2) in eq:weights_EM, and the M-step
 * becomes eq:rho_EM as written: rho'[s] = sum_i w^{i,s} / sum_i sum_s' w^{i,s'};
 * srmra_get_estimate then reports its marginals.  All paths except the FFT path at L_low = 128
 * (UNSUPPORTED there); on the FFT path the E/M kernel is re-planned with a per-CTA accumulator of every
 * shift's posterior mass (possibly fewer thread groups per SM).  Synchronises.  A later srmra_load /
 * srmra_generate / srmra_mom_run returns the context to a separable prior. */
SRMRA_API int srmra_set_joint_rho(srmra_ctx* ctx, const double* rho);
/* Copy the current joint prior [L_high][L_high] (STATE if none is set).  Synchronises. */
SRMRA_API int srmra_get_joint_rho(srmra_ctx* ctx, double* out);

/* Denoiser hook of Algorithm 2: called on the host for every projection
 * step with the device buffer of the estimate x (float64, [L_high][L_high], modified in place), the
 * schedule value sigma_t of eq:decaying_function and the context stream (cudaStream_t); work must be
 * enqueued on that stream.  Return 0 on success (non-zero aborts the run with SRMRA_ERR_NUMERIC). */
typedef int (*srmra_denoiser_fn)(double* x_dev, int32_t L_high, double sigma_t, void* stream, void* user);

/* Replace the built-in stand-in projection (3x3 circular box filter, clamp to [-1, 1]; north_star)
 * with `fn` (NULL restores the built-in one).  The context keeps `user` opaque. */
SRMRA_API int srmra_set_denoiser(srmra_ctx* ctx, srmra_denoiser_fn fn, void* user);

/*
 * Algorithm 2 (projected EM) run to convergence: up to max_iters EM iterations;
 * after iteration t the projection D(x, sigma_j) is applied when (t+1) % F == 0 (F = proj_every),
 * with sigma_j = 2^(-(j-1)/10) for the j-th projection of this run (eq:decaying_function,
 * PAPER.md:345-349; the built-in stand-in ignores it); the run stops after the first iteration
 * t >= 1 (t counted within this run) with |LL_t - LL_{t-1}| <= rel_tol |LL_t|, LL_t the
 * log-likelihood at the input of iteration t (rel_tol <= 0: run max_iters).
 * FFT path without a denoiser hook or an exchange provider (one rank, or NCCL: every rank records the
 * same all-reduced LL, so all take the same decision): asynchronous — the convergence test runs on the
 * device and the remaining enqueued iterations become no-ops; srmra_get_estimate reports the
 * iterations actually run.  Otherwise the host checks the log-likelihood after every iteration.
 * Errors: INVALID_ARG (max_iters < 0), STATE, CUDA, NCCL, NUMERIC (denoiser hook failure).
 */
SRMRA_API int srmra_run(srmra_ctx* ctx, int32_t max_iters, double rel_tol);

/* Evaluation (NEXT-4): error(x_hat) = min_s ||R_s x_hat - x_true||_F / ||x_true||_F over
 * all L_high^2 circular shifts s, for the context's current estimate x_hat (float64), with
 * (R_s z)[p] = z[(p - s) mod L_high] (Eq. (2) sign).  x_true: host float32 [L_high][L_high] (copied,
 * must be finite and non-zero); *err_out the error, (*s1_out, *s2_out) the minimising shift (ties:
 * the smallest s1 L_high + s2).  Any output may be NULL.  Synchronises.  The correlation over all
 * shifts runs on the device in float64 (L_high^4 products). */
SRMRA_API int srmra_relative_error(srmra_ctx* ctx, const float* x_true, double* err_out, int32_t* s1_out,
                                   int32_t* s2_out);

/*
 * NEXT-2, the data term of the projected method of moments (Algorithm 1): the
 * empirical moments of eq:empiric_MOM with D = 2 over ALL ranks' observations,
 *     m1[a]          = (1/N) sum_i y_i[a],
 *     m2[a L_low^2 + b] = (1/N) sum_i y_i[a] y_i[b],      a, b = p1 L_low + p2 (row-major y_i),
 * N the global number of observations.  m1: caller-owned float64 [L_low^2]; m2: float64
 * [L_low^2][L_low^2] (symmetric); either may be NULL (not both).  The sums run on the tensor cores
 * (3xTF32 tcgen05 GEMM of the transposed observations with themselves, float32 accumulation in
 * TMEM, float64 split-K combine) and are all-reduced in float64 when world > 1.  Uses
 * O(L_low^2 n_local) temporary device memory; independent of the EM state.  Synchronises.
 * Errors: INVALID_ARG (both NULL), STATE (failed context / rejected load), CUDA, NCCL.
 */
SRMRA_API int srmra_moments(srmra_ctx* ctx, double* m1, double* m2);

/*
 * NEXT-2, Algorithm 1 (projected method of moments).  L_low <= 64 (else UNSUPPORTED).
 *
 * srmra_mom_set_moments: the data term of eq:LS_SR.  m1 / m2 both NULL: the empirical moments of the
 * loaded observations (srmra_moments' computation, kept on the device); both non-NULL: caller moments,
 * host float64 m1 [L_low^2], m2 [L_low^2][L_low^2] (e.g. the perfect moments of the paper's Fig. 2
 * experiment), copied; the symmetric part of m2 is used.  Transforms them once to the Fourier domain
 * (F M2 F^H, F the L_low x L_low 2-D DFT; O(L_low^5) float64).  Allocates 2 L_low^4 complex doubles.
 * Errors: INVALID_ARG (exactly one NULL, non-finite), STATE (rejected load with NULL moments),
 * UNSUPPORTED, CUDA, NCCL.  Synchronises.
 */
SRMRA_API int srmra_mom_set_moments(srmra_ctx* ctx, const double* m1, const double* m2);

/*
 * The objective eq:LS_SR at theta = (x, rho1 rho2^T), sigma the context's:
 *     f = || P C_x D_rho C_x^T P^T + sigma^2 I - M2 ||_F^2 + lambda || P C_x rho - M1 ||_2^2,
 *     lambda = 1 / (L_high^2 (1 + sigma^2)),
 * and its gradient with respect to x [L_high][L_high], rho1 [L_high], rho2 [L_high] (float64, host;
 * outputs may be NULL).  Evaluated in the Fourier domain without forming C_x:
 * O(L_high^4) float64 work.  theta is not checked (any real values).  Errors: INVALID_ARG (NULL theta),
 * STATE (no moments set), CUDA.  Synchronises.
 */
SRMRA_API int srmra_mom_objective(srmra_ctx* ctx, const double* x, const double* rho1, const double* rho2,
                                  double* f, double* grad_x, double* grad_rho1, double* grad_rho2);

/*
 * Algorithm 1 from the context's current estimate (x, rho1, rho2): up to max_steps L-BFGS steps
 * (memory 10, Armijo backtracking) on eq:LS_SR over (x, a1, a2), rho_j = softmax(a_j); after every F-th
 * step (F = 0: never) the projection x <- D(x, sigma_j) (built-in stand-in or the srmra_set_denoiser
 * hook; sigma_j = 2^(-(j-1)/10), eq:decaying_function) and a memory reset.  Stops early when
 * ||grad||_inf <= gtol or the line search finds no decrease.  The result becomes the context's estimate
 * (srmra_get_estimate; EM iterations may follow; a joint prior is dropped); *f_out the final objective,
 * *steps_out the steps taken (either may be NULL).  Errors: INVALID_ARG (max_steps < 0, F < 0,
 * gtol < 0 or NaN), STATE (no moments set), NUMERIC (non-finite objective / hook failure), CUDA.
 */
SRMRA_API int srmra_mom_run(srmra_ctx* ctx, int32_t max_steps, int32_t F, double gtol, double* f_out,
                            int32_t* steps_out);

/*
 * Synchronise the stream and copy the current estimate to caller-owned host buffers (any may be
 * NULL): x_out float32 [L_high][L_high], rho1_out / rho2_out float64 [L_high], *loglik_out the
 * log-likelihood at the INPUT of the last iteration (NaN if none ran), *iters_done the number of
 * iterations run since init/load.  Returns SRMRA_ERR_NUMERIC if any iteration produced a
 * non-finite log-likelihood or estimate.
 */
SRMRA_API int srmra_get_estimate(srmra_ctx* ctx, float* x_out, double* rho1_out, double* rho2_out,
                       double* loglik_out, int32_t* iters_done);

/* Copy up to cap entries of the per-iteration log-likelihood trace (LL_0, LL_1, ...) into out;
 * *n receives the number of iterations recorded (may exceed cap). Synchronises. */
SRMRA_API int srmra_get_loglik_trace(srmra_ctx* ctx, double* out, int32_t cap, int32_t* n);

/* Test hook: the global (all-reduced) sufficient statistics of the last iteration, float64:
 * b [L_high^2] numerator of eq:x_EM, class_mass [K^2] (A[p] = class_mass[(-p1 mod K)*K + (-p2 mod K)]),
 * marg1 / marg2 [L_high] un-normalised marginals sum_i sum_{s2} w^{i,s} / sum_i sum_{s1} w^{i,s}.
 * Any pointer may be NULL.  Synchronises. */
SRMRA_API int srmra_get_stats(srmra_ctx* ctx, double* b, double* class_mass, double* marg1, double* marg2);

/* Test hook: per-observation log-likelihood terms log sum_s rho[s] exp(-||y_i - P R_s x||^2/(2 sigma^2))
 * of this rank's observations at the input of the last iteration, float64 [n_local]. */
SRMRA_API int srmra_get_obs_loglik(srmra_ctx* ctx, double* out);

/* Test hook: compute this rank's LOCAL (not all-reduced) packed statistics at the current theta
 * without updating it: out float64 [L_high^2 + K^2 + 2 L_high + 1] = b | class_mass | marg1 |
 * marg2 | LL.  Used to check that shard statistics sum to the full-data statistics. */
SRMRA_API int srmra_local_stats(srmra_ctx* ctx, double* out);

/* The path the context runs (SRMRA_PATH_GEMM / FFT / DIRECT), or a negative error code. */
SRMRA_API int srmra_get_path(const srmra_ctx* ctx);

/* Number of kernel launches one srmra_em_iter(ctx, 1) enqueues (for launch accounting). */
SRMRA_API int srmra_launches_per_iter(const srmra_ctx* ctx);

/* Profiling: enable != 0 opens a measuring window (clearing earlier records); 0 closes it.
 * FFT path: every E/M launch stamps its first-CTA start and last-CTA end with the GPU's globaltimer
 * (no event nodes in the CUDA graph: they cost ~9 % of a c1 iteration); GEMM / direct paths: CUDA
 * events on the context stream around each iteration and its E/M kernels. */
SRMRA_API int srmra_profile(srmra_ctx* ctx, int32_t enable);

/* Synchronise and return, over the iterations run since srmra_profile(ctx, 1) (or the previous
 * read): the summed duration of the dominant E/M kernel launches (*em_kernel_ms), of whole
 * iterations (*iter_ms; FFT path: from the spacing of consecutive E/M starts), and the number of
 * iterations (*n_iters).  Any pointer may be NULL.  Clears the records. */
SRMRA_API int srmra_profile_read(srmra_ctx* ctx, double* em_kernel_ms, double* iter_ms, int32_t* n_iters);

/* Debug hook: globaltimer stamps (ns) of the FFT path's tail-kernel phase boundaries of the last
 * iteration, out8[0..5] = start, fold, update, projection, prep, end (0 where a phase did not run),
 * out8[6] = earliest and out8[7] = latest start / end over all tail blocks since the previous call
 * (each call re-arms them).
 * Requires the environment variable SRMRA_TAIL_STAMPS to be set at srmra_init (else SRMRA_ERR_STATE). */
SRMRA_API int srmra_debug_timestamps(srmra_ctx* ctx, uint64_t* out8);

/* Write a fresh 128-byte ncclUniqueId into out (rank 0 calls this before srmra_init). */
SRMRA_API int srmra_nccl_unique_id(void* out128);

/* Release all device memory, the stream (if owned) and the NCCL communicator.  NULL is a no-op. */
SRMRA_API void srmra_free(srmra_ctx* ctx);

/* Last error message of ctx (or of the calling thread's last failed srmra_init when ctx is NULL). */
SRMRA_API const char* srmra_last_error(const srmra_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SRMRA_H_ */
