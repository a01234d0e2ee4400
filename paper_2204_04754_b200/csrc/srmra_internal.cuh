// srmra_internal.cuh — context layout, launch declarations and device helpers shared by the
// kernels of libsrmra.so.  Notation follows PAPER.md §I/§II-C and SURVEY.md §8(a):
//   L = L_high, Ll = L_low, K = L/Ll, s = (s1, s2) in Z_L^2 flattened s1*L + s2,
//   class r(s) = (s1 mod K, s2 mod K), low-res shift t(s) = (s1 / K, s2 / K), s = r + K t,
//   polyphase component x_r[m] = x[(K m1 - r1) mod L, (K m2 - r2) mod L]   (PAPER.md:127-131,
//   relabelled), so that (P R_s x)[n] = x_r[n - t] and ||P R_s x||^2 = E_r := ||x_r||^2.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "../../include/srmra.h"

namespace srmra {

// Per-iteration small parameters, written by k_prep and read by the E/M kernels.
// fp32 part (bias of the logits) and fp64 part (constants of the log-likelihood).
struct IterParams {
    // float32 (device), laid out contiguously: lr1[L] | lr2[L] | beta[K^2]
    float* f32;
    // float64 (device): E[K^2] | E_min | xm[K^2] (mean of x_r, fft path)
    double* f64;
};

struct MomState;  // NEXT-2 moment-objective state (k_mom_obj.cu)

struct PackLayout {  // packed statistics  b | class_mass | marg1 | marg2 | LL
    int64_t b, cmass, m1, m2, ll, total;
};

}  // namespace srmra

struct srmra_ctx {
    // shape
    int L = 0, Ll = 0, K = 0, KK = 0, L2 = 0, Ll2 = 0, Lh = 0;  // Lh = Ll/2+1 (rfft width)
    int64_t n_local = 0, n_global = 0;
    double sigma = 0, inv_s2 = 0, inv_2s2 = 0, tau = 0;
    srmra_options opt{};
    int path = 0;
    int device = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // H2D of y in chunks, overlapped with the init kernels
    cudaEvent_t copy_event = nullptr;
    bool own_stream = false;
    bool failed = false;
    bool needs_load = false;  // the last srmra_load was rejected (non-finite y found on the device)
    std::string err;

    // observation-side buffers (this rank's shard)
    float* d_y = nullptr;       // [n][Ll][Ll]             (direct / gemm paths)
    float2* d_yhat = nullptr;   // [n][Ll][Lh]             (fft path: rfft2 of y_i, float32)
    double* d_ynorm = nullptr;  // [n]  ||y_i||^2, float64
    double* d_ysum = nullptr;   // [n]  sum_n y_i[n], float64 (fft path: the DC term of the scores)
    double* d_llobs = nullptr;  // [n]  per-observation log-likelihood of the last iteration

    // theta
    double* d_x64 = nullptr;  // [L2]
    float* d_x32 = nullptr;   // [L2]
    double* d_rho = nullptr;  // [2L] rho1 | rho2
    double* d_rhoj = nullptr; // [L2] joint shift prior (NEXT-3, GEMM / direct paths), valid when `joint`
    float* d_lrj = nullptr;   // [L2] its natural log (float32), the per-shift logit bias
    bool joint = false;
    double* d_xtmp = nullptr; // [L2] finalize scratch

    // per-iteration
    srmra::IterParams par{};
    float2* d_xhat = nullptr;   // [KK][Ll][Lh] rfft2 of x_r (fft path)
    float4* d_xcoef = nullptr;  // L_low = 128: E-step product coefficients [2][NP][128][128] (k_fft128.cu)
    double* d_colsum = nullptr; // [L2] sum_i w^{i,s}
    double* d_bhat = nullptr;   // fft path, float64: Bhat [KK][Ll][Lh] complex | mass lines [KK][Ll+Lh] complex
    float2* d_part = nullptr;   // fft path: per-CTA float32 partials of the above [fft_grid][...]
    double* d_llpart = nullptr; // fft path: per-CTA log-likelihood partials [fft_grid]
    double* d_tw = nullptr;     // fft path: cos | sin (2 pi j / L_low), j < L_low, float64
    int fft_grid = 0, fft_groups = 0, fft_threads = 0;
    int fft_xs = 0;             // Xhat staged in shared memory by the E/M kernel (1) / as product coefficients (2)
    bool fft_tacc = false;      // E/M kernel keeps the M-step accumulators in tensor memory
    bool fft_joint = false;     // E/M kernel planned with the joint-prior accumulator (NEXT-3)
    int fft_part_cap = 0;       // CTAs the partial buffers were sized for (first plan)
    float2* d_ljp = nullptr;    // NEXT-3, FFT path: log2 joint prior per class pair [NP][Ll n2][Ll n1]
    float* d_jpart = nullptr;   // NEXT-3, FFT path: per-CTA posterior mass per shift [fft_part_cap][KK Ll^2]
    double* d_jacc = nullptr;   // NEXT-3, FFT path: its fixed-order float64 sum [KK Ll^2]
    int fft_tmem_cols = 0;      // tensor-memory columns per CTA (fft_tacc)
    // srmra_load_iterate (FFT path): the first iteration's E/M kernel runs per observation range as the range lands;
    // em_* select that range and its partial slots for launch_fft_em (em_n < 0: all observations, d_part / d_llpart),
    // tail_* the partial slots the tail reduces (tail_nparts 0: fft_grid slots of d_part / d_llpart)
    int64_t em_off = 0, em_n = -1;
    float2* em_part = nullptr;
    double* em_llpart = nullptr;
    float2* tail_part = nullptr;
    double* tail_llpart = nullptr;
    int tail_nparts = 0;
    float2* d_part_s = nullptr;   // [stream_chunks][fft_grid][PB] partial slots of the streamed first iteration
    double* d_llpart_s = nullptr; // [stream_chunks][fft_grid]
    int stream_chunks = 0;
    size_t fft_smem = 0;
    double* d_pack = nullptr;   // packed statistics, see PackLayout
    srmra::PackLayout pk{};
    double* d_trace = nullptr;  // [trace_cap]
    int* d_flag = nullptr;      // [1] numeric error flag
    unsigned* d_counter = nullptr;  // [1] grid "last block" counter of the fused fold + finalize
    int* d_iter = nullptr;          // [1] device iteration counter (FFT tail reads t from it)
    int* d_run = nullptr;           // [2] run control of srmra_run: stop flag, first iteration of the run
    double* d_rtol = nullptr;       // [1] convergence tolerance of the current run (0: none)
    srmra_denoiser_fn denoiser = nullptr;  // Algorithm 2 denoiser hook (NULL: built-in stand-in)
    void* denoiser_user = nullptr;
    int n_proj = 0;                 // projections applied in the current run (sigma schedule index)
    int h_run[2] = {0, 0};          // host staging of d_run / d_rtol
    double h_rtol = 0.0;
    cudaGraphExec_t graph = nullptr;  // captured FFT iteration (E/M kernel + tail), world == 1
    cudaGraphExec_t graph_prof = nullptr;  // same with 4 event-record nodes (profiling quadruple)
    cudaGraphNode_t prof_nodes[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaGraph_t graph_prof_src = nullptr;     // kept alive with graph_prof (exec-node updates need it)
    cudaEvent_t prof_ph[4] = {nullptr, nullptr, nullptr, nullptr};  // capture placeholders, same
    bool graph_failed = false;
    unsigned long long* d_stamps = nullptr;  // [8] tail-kernel phase timestamps (env SRMRA_TAIL_STAMPS)
    unsigned long long* d_emt = nullptr;     // [trace_cap][2] E/M kernel first-CTA start / last-CTA end (globaltimer ns)
    int prof_t0 = 0;                         // first iteration of the current profiling window
    int iters_done = 0;
    bool iters_stale = false;                // a device-loop run may have stopped early: sync_iters first

    // gemm path (k_gemm.cu): tf32 hi|lo splits, scores, transposed posterior, Z = W^T Y, rotated x copies
    float* g_yhl = nullptr;   // [2][n][Ll2]
    float* g_ythl = nullptr;  // [2][Ll2 + 16][ldw]  (row Ll2 = ones)
    float* g_s = nullptr;     // [n][L2]
    float* g_wthl = nullptr;  // [2][L2][ldw]
    float* g_z = nullptr;     // [L2][Ll2 + 16]
    float* g_xe = nullptr;    // [2][KK][4][Ll][2 Ll]
    float* g_cf = nullptr;    // [2][KK Ll Ll][Ll] circulant factor of the polyphase components (TMA mainloop)
    int64_t g_ldw = 0;        // n rounded up to a multiple of 4

    // NEXT-2: method of moments (k_mom_obj.cu), allocated by srmra_mom_set_moments
    srmra::MomState* mom = nullptr;

    // multi-GPU
    void* nccl_comm = nullptr;

    // profiling (srmra_profile): per-iteration event quadruples
    //   [iteration start, E/M kernel start, E/M kernel end, iteration end]
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    cudaEvent_t prof_event();
};

namespace srmra {

// ---------------------------------------------------------------- launches (k_common.cu)
cudaError_t launch_init_obs(srmra_ctx* c, int64_t first, int64_t count);  // ||y_i||^2 (+ finiteness flag)
cudaError_t launch_prep(srmra_ctx* c);          // theta -> IterParams (+ Xhat), zero accumulators
cudaError_t launch_pack(srmra_ctx* c);          // colsum (+ Bhat) -> packed b | cmass | marg | LL
cudaError_t launch_finalize(srmra_ctx* c, int t, int project);
cudaError_t launch_x32_from_x64(srmra_ctx* c);   // after a denoiser hook changed x
cudaError_t launch_shift_corr(srmra_ctx* c, const double* xref_dev, double* corr_dev);  // NEXT-4
cudaError_t launch_generate(srmra_ctx* c, const float* x_dev, const double* cdf_dev, int last1, int last2,
                            uint64_t seed, int64_t first, int* shifts_dev);  // NEXT-4 (k_synth.cu)
int moments(srmra_ctx* c, double* m1, double* m2, std::string& err);  // NEXT-2 (k_moments.cu)
int moments_dev(srmra_ctx* c, double* out_dev, std::string& err);     // same, left on the device
bool mom_supported(const srmra_ctx* c);                                // k_mom_obj.cu: L_low <= 64
void mom_free(srmra_ctx* c);
bool mom_ready(const srmra_ctx* c);                                    // moments set
int mom_set(srmra_ctx* c, const double* m1, const double* m2, std::string& err);
int mom_objective(srmra_ctx* c, const double* x, const double* r1, const double* r2, double* f, double* gx,
                  double* g1, double* g2, std::string& err);
int mom_run(srmra_ctx* c, int max_steps, int F, double gtol, double* f_out, int* steps_out, std::string& err);
// TMA 3xTF32 tcgen05 GEMM C = A B^T (k_gemm_tma.cu); c64 / kz / sym: see there
cudaError_t launch_gemm_tma(const float* a_hi, const float* a_lo, int64_t M, int64_t lda, const float* b_hi,
                            const float* b_lo, int64_t nb_rows, int64_t ldb, int N, int64_t Kdim, int circ, int Ll,
                            float* c, int64_t ldc, cudaStream_t st, double* c64 = nullptr, int kz = 0, int sym = 0);
// same product accumulated in float64 (TMEM chunks drained into registers; k_gemm_tma.cu)
cudaError_t launch_gemm_tma_acc64(const float* a_hi, const float* a_lo, int64_t M, int64_t lda, const float* b_hi,
                                  const float* b_lo, int64_t nb_rows, int64_t ldb, int N, int64_t Kdim, double* c,
                                  int64_t ldc, int sym, int num_sms, cudaStream_t st, int* zslices = nullptr);
int allreduce_doubles(srmra_ctx* c, double* buf, size_t n);           // NCCL sum, no-op for world 1
// ---------------------------------------------------------------- path kernels
cudaError_t launch_direct_em(srmra_ctx* c);     // k_direct.cu
bool direct_supported(int L, int Ll, int K);
cudaError_t launch_fft_em(srmra_ctx* c);        // k_fft.cu
bool fft_supported(int L, int Ll, int K);
cudaError_t launch_fft_init(srmra_ctx* c, int64_t first, int64_t count);  // Yhat_i, sum y_i
int fft_partial_bins(int KK, int Ll);  // per-CTA partial bins of the FFT E/M kernels (k_fft.cu)
// tcgen05 3xTF32 GEMM path (k_gemm.cu)
bool gemm_supported(int L, int Ll, int K);
size_t gemm_bytes(const srmra_ctx* c);
cudaError_t gemm_alloc(srmra_ctx* c);
void gemm_free(srmra_ctx* c);
cudaError_t launch_gemm_init(srmra_ctx* c);
cudaError_t launch_gemm_em(srmra_ctx* c, cudaEvent_t ev_em0, cudaEvent_t ev_em1);
// cooperative tail kernel of the FFT path (k_fft_tail.cu): phases selected by TAIL_* bits
enum { TAIL_REDUCE = 1, TAIL_FOLD = 2, TAIL_FINALIZE = 4, TAIL_PREP = 8 };
cudaError_t launch_fft_tail(srmra_ctx* c, int mode);
int fft_launches_per_iter(const srmra_ctx* c);
size_t fft_bhat_doubles(int KK, int Ll);  // Bhat [KK][Ll][Lh] complex + mass lines [KK][Ll+Lh] complex
size_t fft_yhat_stride(int Ll);           // float2 per observation in d_yhat (16-byte multiple)
cudaError_t fft_plan(srmra_ctx* c);       // grid / groups / smem of the E/M kernel for this shard
cudaError_t fft_plan_joint(srmra_ctx* c, bool joint);  // re-plan with / without the joint-prior accumulator
size_t fft_joint_bins(int KK, int Ll);
size_t fft_part_float2(const srmra_ctx* c);
size_t fft_xhat_float2(int KK, int Ll);   // pair-interleaved Xhat
size_t fft128_coef_float4(int KK);        // L_low = 128 product coefficients

// cudaFuncSetAttribute is per device: run a setup functor once per device ordinal (retried after a failure)
struct PerDeviceOnce {
    std::atomic<unsigned long long> mask{0};
    template <class F>
    cudaError_t run(F f) {
        int d = 0;
        cudaGetDevice(&d);
        const unsigned long long bit = 1ull << (d & 63);
        if (mask.load() & bit) return cudaSuccess;
        const cudaError_t e = f();
        if (e == cudaSuccess) mask.fetch_or(bit);
        return e;
    }
};

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ int imod(int a, int m) {
    int r = a % m;
    return r < 0 ? r + m : r;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide reductions; `scratch` must hold >= 32 elements of T; all threads get the result.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    T r = lane < nw ? scratch[lane] : T(0);
    r = warp_sum(r);
    return r;
}
template <typename T>
__device__ __forceinline__ T block_max(T v, T* scratch, T neg_inf) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    T r = lane < nw ? scratch[lane] : neg_inf;
    r = warp_max(r);
    return r;
}

}  // namespace srmra
