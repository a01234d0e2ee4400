// k_fft.cu — batched polyphase FFT-correlation E-step + M-step (SRMRA_PATH_FFT).
//
// Sub-image form of the likelihood (proof of thm:uniqueness): with the
// polyphase components x_r[m] = x[(K m1 - r1) mod L, (K m2 - r2) mod L] and s = r + K t,
//     (P R_s x)[n] = x_r[n - t],   so   S[i, r + K t] = <y_i, P R_s x> = sum_n y_i[n] x_r[n - t]
// is, for each observation i and class r, a circular cross-correlation on the L_low x L_low grid:
//     S_{i,r} = irfft2( Yhat_i . conj(Xhat_r) )                                   (E-step scores)
// and the adjoint gather of the M-step (eq:x_EM with P^{-1} := P^T),
//     b_r[m] = b[(K m1 - r1) mod L, (K m2 - r2) mod L] = sum_i sum_t w_{i,r}[t] y_i[m + t],
// is again a correlation, accumulated over i in the frequency domain:
//     Bhat_r += Yhat_i . conj(What_{i,r}),   What_{i,r} = rfft2(w_{i,r}),   b_r = irfft2(Bhat_r).
// The shift marginals only need the k2 = 0 column and the k1 = 0 row of sum_i What_{i,r}
// (row / column sums of the posterior mass of class r), so those two lines are accumulated too.
//
// Kernel layout (one persistent CTA per SM slot, G "groups" of threads per CTA, each group owns one
// observation at a time):  two classes (r, r') are packed into one complex L_low x L_low transform
// (real part r, imaginary part r').  Each 1-D FFT of length L_low is done by ONE thread entirely in
// registers (split radix, compile-time twiddles); the row/column transposes go through a padded shared
// buffer (row stride L_low + 2 float2: conflict-free for both row and column access).  The scores of
// the observation never leave registers: softmax (3 group reductions) runs on them, and the row
// thread immediately starts the forward transform of the posterior.  Yhat_i is prefetched with
// cp.async into a double buffer; Xhat (per-iteration, <= 70 KB) is read through the L1/read-only
// path; Bhat is accumulated per CTA in shared memory (float32) and added to the float64 global
// accumulator once at the end.
#include <math.h>
#include <stdlib.h>

#include <utility>

#include "regfft.cuh"
#include "srmra_internal.cuh"
#include "tcgen05.cuh"

namespace srmra {
namespace fftk {
using namespace regfft;

// ------------------------------------------------------------------ group sync / reductions
__device__ __forceinline__ void group_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <typename T, bool MAX>
__device__ __forceinline__ T group_reduce(T v, T* scratch, int gwarp, int nwarps, int lane, int bar_id, int gthreads) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T u = __shfl_xor_sync(0xffffffffu, v, o);
        v = MAX ? (u > v ? u : v) : v + u;
    }
    if (nwarps == 1) return v;
    if (lane == 0) scratch[gwarp] = v;
    group_bar(bar_id, gthreads);
    T r = scratch[0];
    for (int w = 1; w < nwarps; ++w) r = MAX ? (scratch[w] > r ? scratch[w] : r) : r + scratch[w];
    return r;
}

__device__ __forceinline__ float2 cmul_conj(float2 a, float2 b) {  // a * conj(b)
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ------------------------------------------------------------------ main E/M kernel
struct EmArgs {
    const float2* yhat;     // [n][ystride] rfft2(y_i), float32 (ystride = Ll*Lh rounded up to even)
    const double* ynorm;    // [n]
    const float4* xhat;     // [NP][Ll][Lh] pair-interleaved: (Xhat_{2q}, Xhat_{2q+1}) / Ll^2
    const float* par32;     // log2 units: lr1[L] | lr2[L] | beta[KK]
    const double* par64;    // E[KK] | (unused) | xm[KK]
    int64_t n;
    int L, K, KK, ystride, ybuf, groups;  // ybuf: shared-memory stride of a staged Yhat (ystride + wrap row)
    float c2;               // log2(e) / sigma^2
    double inv_s2, inv_2s2;
    float2* part;           // [gridDim.x][PB] per-CTA partials, see part_bins()
    double* llpart;         // [gridDim.x] per-CTA log-likelihood partials
    double* llobs;          // [n]
    int tmem_cols;          // TACC: tensor-memory columns allocated per CTA (power of two >= 32)
    const int* run;         // srmra_run stop flag ([0])
    unsigned long long* emt;  // [cap][2] first-CTA start / last-CTA end of this launch (globaltimer), slot *iter
    const int* iter;          // device iteration counter (slot index)
    int emt_cap;
    const float2* ljp;        // JOINT: log2 joint prior per pair [NP][LL n2][LL n1] = (class 2q, class 2q+1)
    float* jpart;             // JOINT: per-CTA posterior mass per shift [gridDim.x][KK][LL t1][LL t2]
};

template <int LL>
struct Geo {
    static constexpr int LH = LL / 2 + 1;
    // padded row stride of the transpose buffer (float2): even, so a row thread moves two elements per
    // 128-bit access; (LL + 2) * 8 B = 4 banks mod 32, so 8 lanes of a row access cover all 32 banks
    static constexpr int WS = LL + 2;
    // Yhat row stride (float2), = yrow_of(LL).  (Rows padded to 24 at LL = 32 — each 8-byte bank pair hit
    // exactly twice by a warp's E-column read — and the full mirrored LL x LL spectrum both measured no faster
    // at c3 and slower at c1 / c2: the extra staging bytes cost more than the bank conflicts.)
    static constexpr int YR = LH;
};

template <int LL>
__host__ __device__ constexpr int group_threads(int KK) {
    return ((((KK + 1) / 2) * LL + 31) / 32) * 32;
}

// Accumulators (float2) of one group / one CTA partial, NP = ceil(K^2 / 2) class pairs:
//   UV [NP][2][Ll][Lh]  U_q[k] = sum_i Yhat_i[k] conj(Z_{i,q}[k]),  V_q[k] = sum_i Yhat_i[k] Z_{i,q}[-k]
//                       (Z_{i,q} = What_{i,2q} + i What_{i,2q+1}: Bhat_{2q} = (U+V)/2, Bhat_{2q+1} = i(U-V)/2)
//   R  [KK][Ll]         spatial row sums of the posterior, sum_i sum_t2 w_{i,r}[t1, t2]  (real in .x)
//   CU [NP][Ll]         sum_i Z_{i,q}[0][k2]  (k1 = 0 row of the transformed posterior pair)
__host__ __device__ inline int part_bins(int KK, int LL) {
    const int NP = (KK + 1) / 2, LH = LL / 2 + 1;
    return 2 * NP * LL * LH + KK * LL + NP * LL;
}

// Shared memory of one group (16-B multiple): Yb [2][ystride] | Wk [NP][LL][WS] | Acc [part_bins] | red [32]
template <int LL>
__host__ __device__ inline size_t group_smem(int KK, int ystride) {
    using G = Geo<LL>;
    const int NP = (KK + 1) / 2;
    size_t b = sizeof(float2) * (2 * (size_t)ystride + (size_t)NP * LL * G::WS + (size_t)part_bins(KK, LL)) +
               sizeof(double) * 32;
    return (b + 15) & ~(size_t)15;
}
template <int LL>
__host__ __device__ inline size_t par_off_lrp(int KK) {  // logit-bias table lr1 | lr2 | beta, L = K LL <= 8 LL
    return ((size_t)(2 * 8 * LL + KK) * sizeof(float) + 15) & ~(size_t)15;
}
// ... followed by the per-pair lr2 table lrp [NP][LL] float2 = (lr2 of class 2q, lr2 of class 2q+1) at n2
template <int LL>
__host__ __device__ inline size_t par_bytes(int KK) {
    return par_off_lrp<LL>(KK) + sizeof(float2) * (size_t)((KK + 1) / 2) * LL;
}
template <int LL>
__host__ __device__ inline size_t smem_bytes(int KK, int groups, int ystride) {
    return group_smem<LL>(KK, ystride) * groups + par_bytes<LL>(KK);
}

// JOINT (NEXT-3, eq:rho_EM as written): one per-CTA accumulator of the posterior mass of every shift,
// JA [KK][LL][LL + 1] float (rows padded: the row threads of a warp add at the same n2 conflict-free)
template <int LL>
__host__ __device__ inline size_t joint_bytes(int KK) {
    return ((size_t)KK * LL * (LL + 1) * sizeof(float) + 15) & ~(size_t)15;
}

// TACC (L_low >= 32): the M-step accumulators U_q / V_q (and the Yhat values of pass 0) live in tensor memory instead of the group's
// shared memory, which leaves room for more groups (warps) per SM.  Group shared memory then holds
// Yb [2][ystride] | Wk [NP][LL][WS] | zc [NP][2][LL] | yc [NP][2][LL] | red [32]; at the end the group's
// partial (layout part_bins) is staged over Yb / Wk.
// OVL (TACC without the joint prior): the softmax reduction is split around the M-row transform — each warp
// publishes its (s, m, z) summary with an mbarrier arrive, transforms its rows of unnormalised weights, and
// only then waits and scales the transformed rows (the transform is linear), so the cross-warp wait overlaps
// the pass-2 FFT instead of idling at a barrier.  Yhat then needs a ring of three staged buffers: the
// prefetch of observation j + 1 is issued at the start of observation j into the buffer of j - 2, whose last
// reader (the deferred vex_update in j - 1's pass 0) is ordered by j - 1's summary mbarrier: a warp arrives
// on it after its passes 0 and 1 of j - 1, and no warp starts j before it has waited on it (DESIGN 6.1e;
// there is no group barrier per observation).
// L_low = 32 only: measured c3 3.342 -> 3.198 ms (3.057 ms without the group barriers), c1 83.4 -> 82.9 us;
// at L_low = 64 (c2) the third buffer (17 KB per group) costs a group, 0.832 -> 1.045 ms.
// SRMRA_FFT_NO_OVL builds the previous form (reduction barrier before the transform) for A/B.
template <int LL, bool TACC, bool JOINT>
__host__ __device__ constexpr bool ovl_mode() {
#ifdef SRMRA_FFT_NO_OVL
    return false;
#else
    return LL == 32 && TACC && !JOINT;
#endif
}
template <int LL>
__host__ __device__ inline size_t group_smem_t(int KK, int ystride, int nybuf = 2) {
    using G = Geo<LL>;
    const int NP = (KK + 1) / 2;
    size_t b = sizeof(float2) * ((size_t)nybuf * ystride + (size_t)NP * LL * G::WS + 4 * (size_t)NP * LL) +
               sizeof(double) * 32;
    return (b + 15) & ~(size_t)15;
}
template <int LL>
__host__ __device__ inline bool tacc_fits(int KK, int ystride) {  // the staged partial fits over Yb / Wk
    return part_bins(KK, LL) <= 2 * ystride + ((KK + 1) / 2) * LL * Geo<LL>::WS;
}

// Threads per CTA cap (register budget: one L_low-point complex line per thread lives in registers)
template <int LL, bool TACC = false>
__host__ __device__ constexpr int max_cta_threads() {
#ifndef SRMRA_FFT32_TACC_THREADS
#define SRMRA_FFT32_TACC_THREADS 384
#endif
    return LL >= 64 ? 256 : (LL >= 32 ? (TACC ? SRMRA_FFT32_TACC_THREADS : 320) : 512);
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// (max, scaled sum) pair reduction over the group: (m1, z1) + (m2, z2) = (M, z1 2^(m1-M) + z2 2^(m2-M))
__device__ __forceinline__ void ms_combine(float& m, float& z, float m2, float z2) {
    const float M = fmaxf(m, m2);
    if (M == -INFINITY) return;  // both empty
    z = z * ex2(m - M) + z2 * ex2(m2 - M);
    m = M;
}
__device__ __forceinline__ void group_reduce_ms(float& m, float& z, float2* scratch, int gwarp, int nwarps, int lane,
                                                int bar_id, int gthreads) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const float z2 = __shfl_xor_sync(0xffffffffu, z, o);
        ms_combine(m, z, m2, z2);
    }
    if (nwarps == 1) return;
    if (lane == 0) scratch[gwarp] = make_float2(m, z);
    group_bar(bar_id, gthreads);
    float M = scratch[0].x, Zs = scratch[0].y;
    for (int w = 1; w < nwarps; ++w) ms_combine(M, Zs, scratch[w].x, scratch[w].y);
    m = M;
    z = Zs;
}

// (s, m, z) triples: a set of unnormalised weights 2^(s c2 + v) with log2 maximum s c2 + m and scaled
// sum z = sum 2^(v - m); two sets combine through the difference of their maxima, (s - s') c2 + (m - m'),
// so every thread may use its own score reference s (no separate max reduction)
__device__ __forceinline__ void smz_combine(float& s, float& m, float& z, float s2, float m2, float z2, float c2) {
    // branchless (a data-dependent return costs BSSY / BSYNC / BRA per level): the other set empty
    // (m2 = -inf) gives e = 0 and d = +inf or NaN, so this set is kept unchanged; this set empty (m = -inf)
    // gives d = -inf, e = 0 and the other set is taken
    const float d = fmaf(s - s2, c2, m - m2);
    const bool keep = !(d < 0.f);
    const float e = m2 == -INFINITY ? 0.f : ex2(-fabsf(d));
    z = keep ? fmaf(z2, e, z) : fmaf(z, e, z2);
    s = keep ? s : s2;
    m = keep ? m : m2;
}
__device__ __forceinline__ void smz_cross(float& s, float& m, float& z, float c2, const float4* scratch, int nwarps,
                                          int pw, int lane);
__device__ __forceinline__ void smz_warp(float& s, float& m, float& z, float c2) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const float z2 = __shfl_xor_sync(0xffffffffu, z, o);
        smz_combine(s, m, z, s2, m2, z2, c2);
    }
}
__device__ __forceinline__ void mbar_arrive(uint32_t saddr) {  // release.cta: orders this thread's prior stores
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr) : "memory");
}
__device__ __forceinline__ void group_reduce_smz(float& s, float& m, float& z, float c2, float4* scratch, int gwarp,
                                                 int nwarps, int pw, int lane, int bar_id, int gthreads) {
    smz_warp(s, m, z, c2);
    if (nwarps == 1) return;
    if (lane == 0) scratch[gwarp] = make_float4(s, m, z, 0.f);
    group_bar(bar_id, gthreads);
    smz_cross(s, m, z, c2, scratch, nwarps, pw, lane);
}
// the cross-warp half of group_reduce_smz, once every warp's summary is in scratch:
// lane j takes warp (j mod pw)'s summary (pw = nwarps rounded up to a power of two, missing warps empty);
// a log2(pw)-deep shuffle tree then leaves the group result in every block of pw lanes, i.e. in every
// lane — instead of a serial walk over the warps
__device__ __forceinline__ void smz_cross(float& s, float& m, float& z, float c2, const float4* scratch, int nwarps,
                                          int pw, int lane) {
    const int wj = lane & (pw - 1);
    const float4 e = wj < nwarps ? scratch[wj] : make_float4(0.f, -INFINITY, 0.f, 0.f);
    s = e.x;
    m = e.y;
    z = e.z;
    for (int o = 1; o < pw; o <<= 1) {
        const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const float z2 = __shfl_xor_sync(0xffffffffu, z, o);
        smz_combine(s, m, z, s2, m2, z2, c2);
    }
}

// PAIRS = true when K^2 is even (every complex transform carries two classes); for odd K^2 the
// imaginary half of the last pair is empty.
// XS = 1: the pair-interleaved Xhat of this iteration is staged once per CTA in shared memory
// (ahead of the group areas) instead of being read through L1 in the E-step product.
// XS = 2: staged instead as the E-step product's coefficients: for a stored bin o of the pair (a, b) and
// the sign g = +1 (column k2 < LH, stored bin) or -1 (k2 >= LH, Hermitian mirror), the conjugated packed
// product v = conj(Yhat conj(Xhat_a) + i Yhat conj(Xhat_b)) (g = +1; its mirror form for g = -1) is
//     v.x = Y.x (xa.x + g xb.y) + Y.y (xa.y - g xb.x),   v.y = Y.x (g xa.y - xb.x) + Y.y (-g xa.x - xb.y),
// so one float4 per (bin, g) turns the two complex products and their combination (10 FP32
// instructions) into 2 FMUL + 2 FFMA.  Stored per (k1, k2 < LL) in the order the column threads read
// them (the mirror resolved at staging), so a warp's load is 32 consecutive float4.
// (Mode 2 stores two numbers per (k1, k2): (b, d) = (B, -A) for g = +1 and (-B, A) for g = -1 with (a, c) = (A, B),
// see the kernel.)
template <int LL>
__host__ __device__ inline size_t xs_bytes(int KK, int xs_mode = 1) {
    return (xs_mode == 2 ? sizeof(float2) : sizeof(float4)) * (size_t)((KK + 1) / 2) * LL * (xs_mode == 2 ? LL : LL / 2 + 1);
}

// MAXT: the launch bound (register budget).  L_low = 32 with a 256-thread group (K^2 >= 15) fits one group in the
// default 384 threads anyway; its own instantiation with MAXT = 256 gives ptxas 222 instead of 168 registers and no
// spills: c3 3.544 -> 3.482 ms
template <int LL, bool PAIRS, int XS, bool TACC, bool JOINT, int MAXT = max_cta_threads<LL, TACC>()>
__global__ void __launch_bounds__(MAXT, 1) k_fft_em(EmArgs a) {
    using G = Geo<LL>;
    constexpr int LH = G::LH, WS = G::WS, M = LL - 1, YR = G::YR;
    if (*reinterpret_cast<const volatile int*>(a.run)) return;  // converged srmra_run: no-op iteration
    // launch duration stamps (the profiling window of srmra_profile reads them; no event nodes in the graph)
    int emt_slot = -1;
    if (threadIdx.x == 0) {
        emt_slot = *reinterpret_cast<const volatile int*>(a.iter);
        if (emt_slot < a.emt_cap) {
            unsigned long long t0;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            atomicMin(a.emt + 2 * emt_slot, t0);
        }
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int KK = a.KK, K = a.K, L = a.L;
    const int NP = (KK + 1) / 2;
    const int GT = group_threads<LL>(KK);
    const int g = threadIdx.x / GT;        // group
    const int tg = threadIdx.x - g * GT;   // thread in group
    const int lane = threadIdx.x & 31;
    const int gwarp = tg >> 5, nwarps = GT >> 5;
    int pw = 1;  // nwarps rounded up to a power of two (the cross-warp shuffle tree of the softmax reduction)
    while (pw < nwarps) pw <<= 1;
    const int bar_id = 1 + g;

    // ---- shared layout: par table | [Xhat (XS)] | group 0 | group 1 | ...
    float* pars = reinterpret_cast<float*>(smem_raw);
    const size_t pb = par_bytes<LL>(KK);
    const size_t xsb = XS ? xs_bytes<LL>(KK, XS) : 0;
    unsigned char* gbase = smem_raw + pb + xsb;
    for (int k = threadIdx.x; k < 2 * L; k += blockDim.x) pars[k] = __ldg(a.par32 + k);
    // class bias beta_r = (E_min - E_r) log2(e) / (2 sigma^2) from E_r (float64, written by the tail)
    double emin = __ldg(a.par64);
    for (int r = 1; r < KK; ++r) emin = fmin(emin, __ldg(a.par64 + r));
    for (int r = threadIdx.x; r < KK; r += blockDim.x)
        pars[2 * L + r] = (float)((emin - __ldg(a.par64 + r)) * a.inv_2s2 * 1.4426950408889634074);
    {  // per-pair lr2 table: one 128-bit load gives two n2 of both classes in the softmax
        float2* lrp_w = reinterpret_cast<float2*>(smem_raw + par_off_lrp<LL>(KK));
        for (int k = threadIdx.x; k < NP * LL; k += blockDim.x) {
            const int qq = k / LL, n2 = k - qq * LL, rA = 2 * qq, rB = 2 * qq + 1;
            lrp_w[k] = make_float2(__ldg(a.par32 + L + rA % K + K * n2),
                                   rB < KK ? __ldg(a.par32 + L + rB % K + K * n2) : 0.f);
        }
    }
    if (XS == 1) {
        const float4* src = a.xhat;
        float4* dst = reinterpret_cast<float4*>(smem_raw + pb);
        for (int k = threadIdx.x; k < NP * LL * LH; k += blockDim.x) dst[k] = __ldg(src + k);
    } else if (XS == 2) {  // product coefficients in the order pass 0 reads them: [q][k1][k2], k2 < LL
        const float4* src = a.xhat;
        float2* dst = reinterpret_cast<float2*>(smem_raw + pb);
        for (int k = threadIdx.x; k < NP * LL * LL; k += blockDim.x) {
            const int qq = k / (LL * LL), rem = k - qq * LL * LL, k1 = rem / LL, k2 = rem - k1 * LL;
            const bool fl = k2 >= LH;  // Hermitian mirror of a stored bin, g = -1
            const int o = (fl ? ((LL - k1) & M) : k1) * LH + (fl ? LL - k2 : k2);
            const float4 x = __ldg(src + (size_t)qq * LL * LH + o);  // (xa, xb)
            // (a, c) = (A, B); v = Y.x (A, B) + Y.y (b, d) with (b, d) = (B, -A) (g = +1) or (-B, A) (g = -1)
            dst[k] = fl ? make_float2(x.x - x.w, -x.y - x.z) : make_float2(x.x + x.w, x.y - x.z);
        }
    }
    __shared__ uint32_t tmem_slot;
    if (TACC && threadIdx.x < 32) tc::tmem_alloc_n(&tmem_slot, a.tmem_cols);
    if (TACC) tc::fence_before();
    __syncthreads();
    if (TACC) tc::fence_after();
    constexpr bool OVL = ovl_mode<LL, TACC, JOINT>();
    constexpr int NYB = OVL ? 3 : 2;  // staged Yhat buffers
    const size_t per_g = TACC ? group_smem_t<LL>(KK, a.ybuf, NYB) : group_smem<LL>(KK, a.ybuf);
    const int PB = part_bins(KK, LL);
    float* JA = reinterpret_cast<float*>(gbase + per_g * a.groups);  // JOINT accumulator (after the groups)
    if (JOINT) {
        for (int k = threadIdx.x; k < KK * LL * (LL + 1); k += blockDim.x) JA[k] = 0.f;
        __syncthreads();
    }
    float2* Yb = reinterpret_cast<float2*>(gbase + per_g * g);          // [NYB][ybuf]
    float2* Wk = Yb + NYB * a.ybuf;                                     // [NP][LL][WS]
    // TACC: zc | yc | red after Wk, the partial staged over Yb (at the end); else Acc [PB] | red
    float2* Acc = TACC ? Yb : Wk + (size_t)NP * LL * WS;
    float2* zc = Wk + (size_t)NP * LL * WS;                             // [NP][2][LL] (TACC)
    float2* yc = zc + 2 * NP * LL;                                      // [NP][2][LL] (TACC)
    double* red = reinterpret_cast<double*>(TACC ? yc + 2 * NP * LL : Acc + PB);  // [32]
    float* redf = reinterpret_cast<float*>(red);
    float2* red2 = reinterpret_cast<float2*>(red);
    if (!TACC)
        for (int k = tg; k < 2 * NP * LL * LH; k += GT) Acc[k] = make_float2(0.f, 0.f);
    // TMEM: warp w reaches lanes 32 (w & 3); a thread's accumulator line (2 LL columns) starts at column
    // 2 LL (w >> 2) of its lane
    const int warp = threadIdx.x >> 5;
    // TMEM per thread: its accumulator line (2 LL columns) and the Yhat values its pass 0 read (2 LL
    // columns), which are exactly the ones its pass 3 needs (for a mirrored column c >= LH pass 0 reads
    // Yhat[-k1][LL - c], so index k1 carries V_q[-k1][LL - c] and Z[k1] needs no reflection)
    const uint32_t tacc = TACC ? tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 4 * LL) : 0u;
    const uint32_t tys = tacc + 2 * LL;
    if (TACC) {
        float z[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) z[j] = 0.f;
#pragma unroll
        for (int ch = 0; ch < 2 * LL / 16; ++ch) tc::tmem_st16(tacc + 16 * ch, z);
        tc::tmem_wait_st();
    }

    const float* lr1 = pars;
    const float* lr2 = pars + L;
    const float* beta = pars + 2 * L;

    // line owned by this thread in every pass: pair q, index idx (column k2 / row n1 / column c)
    const bool line_ok = tg < NP * LL;
    const int q = line_ok ? tg / LL : 0;
    const int idx = line_ok ? tg - q * LL : 0;
    const int ra = 2 * q, rb = 2 * q + 1;
    const bool has_b = PAIRS || rb < KK;
    const float4* XP = (XS ? reinterpret_cast<const float4*>(smem_raw + pb) : a.xhat) + (size_t)q * LL * LH;
    const float2* XP2 = reinterpret_cast<const float2*>(smem_raw + pb) + (size_t)q * LL * LL;  // XS = 2
    float2* Wq = Wk + (size_t)q * LL * WS;
    float2* Uq = Acc + (size_t)(2 * q) * LL * LH;
    float2* Vq = Uq + (size_t)LL * LH;
    const int ra2 = ra % K, rb2 = rb % K;
    // logit bias (log2 units) of this thread's row n1 = idx, per class
    // (JOINT: the class bias only; the whole log prior comes from the per-shift table ljp)
    const float biasA = line_ok ? (JOINT ? 0.f : lr1[ra / K + K * idx]) + beta[ra] : 0.f;
    const float biasB = (line_ok && has_b) ? (JOINT ? 0.f : lr1[rb / K + K * idx]) + beta[rb] : 0.f;

    // per-thread accumulators over this group's observations
    float rsumA = 0.f, rsumB = 0.f;     // row sums of w (class ra / rb, row idx)
    float2 cu = make_float2(0.f, 0.f);  // sum_i Z_{i,q}[0][idx]
    __shared__ double llg[16];          // per-group log-likelihood accumulators (tg == 0)
    __shared__ double emin_g[16];       // E_min of this iteration (the LL constant), written and read by tg == 0
    if (tg == 0) {
        llg[g] = 0.0;
        emin_g[g] = emin;
    }
    // TACC roles in the M-column pass (column c = idx of pair q): c < LH accumulates U_q[., c], c >= LH
    // accumulates V_q[., LL - c]; the V columns 0 and LL/2 (from c = 0, LL/2) go through zc [NP][2 LL + 2]
    // (the second column at offset LL + 1: the two writer lanes of a warp hit different banks) into vex0 /
    // vexh, owned by thread (q, k1 = idx); their Yhat factors are read from the previous observation's
    // staged Yhat (vex_update runs before the prefetch overwrites that buffer)
    const bool role_u = idx < LH;
    const float su = role_u ? -1.f : 1.f;
    const bool vsrc = line_ok && (idx == 0 || idx == LL / 2);
    float2 vex0 = make_float2(0.f, 0.f), vexh = make_float2(0.f, 0.f);
    auto vex_update = [&](const float2* Yp) {
        if (line_ok) {
            const float2* zq = zc + q * (2 * LL + 2);
            const int mk = (LL - idx) & M;
            float2 yv = Yp[idx * YR], z = zq[mk];
            vex0.x += yv.x * z.x - yv.y * z.y;
            vex0.y += yv.y * z.x + yv.x * z.y;
            yv = Yp[idx * YR + LL / 2];
            z = zq[LL + 1 + mk];
            vexh.x += yv.x * z.x - yv.y * z.y;
            vexh.y += yv.y * z.x + yv.x * z.y;
        }
    };
    bool vex_pending = false;

    const int n = (int)a.n;  // n_local is an int32 at the ABI
    const int gstride = gridDim.x * a.groups;
    int i = blockIdx.x * a.groups + g;
    int buf = 0;
    auto nxt = [](int b) { return OVL ? (b == 2 ? 0 : b + 1) : (b ^ 1); };  // next / previous staged buffer
    auto prv = [](int b) { return OVL ? (b == 0 ? 2 : b - 1) : (b ^ 1); };
    // OVL: one mbarrier per group, one arrival per warp and observation (its softmax summary is in scratch)
    __shared__ __align__(8) unsigned long long ovl_mbar[16];
    const uint32_t ovl_mb = (uint32_t)__cvta_generic_to_shared(ovl_mbar + g);
    uint32_t ovl_ph = 0;
    if (OVL && tg == 0) {
        tc::mbar_init(ovl_mb, (uint32_t)nwarps);
        tc::fence_mbar_init();
    }
    // OVL: two summary slots by observation parity (a warp can be one observation ahead of a slower one
    // still combining: the pass-2 transpose is warp-local at L_low = 32, so no group barrier separates them)
    float4* const smz_scratch0 = reinterpret_cast<float4*>(red2) + 8;
    // OVL: one "staged" mbarrier per Yhat buffer: every thread's cp.async of a prefetch arrives on it
    // (cp.async.mbarrier.arrive.noinc), and pass 0 waits on it instead of a group barrier after the copies
    __shared__ __align__(8) unsigned long long ovl_full[16][3];
    const uint32_t ovl_full0 = (uint32_t)__cvta_generic_to_shared(&ovl_full[g][0]);
    uint32_t ovl_fph = 0;  // per-buffer phase parity bits
    int ovl_j = 0;         // this group's observation count
    if (OVL && tg == 0) {
        for (int b = 0; b < 3; ++b) tc::mbar_init(ovl_full0 + 8 * b, (uint32_t)GT);
        tc::fence_mbar_init();
    }
    __syncthreads();  // the mbarriers are initialised before any cp.async arrives on them
    // a staged Yhat carries a copy of its first row after its last (row LL): the mirrored E-column reads
    // Yhat[(LL - k1) mod LL] then walk a constant stride
    auto prefetch = [&](int obs, int b) {
        if (obs < n) {
            const float2* src = a.yhat + (int64_t)obs * a.ystride;
            float2* dst = Yb + b * a.ybuf;
            for (int c = tg; c < a.ybuf / 2; c += GT) {
                const int cs = c < a.ystride / 2 ? c : c - a.ystride / 2;
                cp_async16(dst + 2 * c, src + 2 * cs);
            }
        }
        cp_async_commit();
        if constexpr (OVL)
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(ovl_full0 + 8 * b) : "memory");
    };
    prefetch(i, 0);
    if constexpr (!OVL) {
        cp_async_wait0();
        group_bar(bar_id, GT);
    }
    const bool flip0 = idx >= LH;  // pass 0: column k2 = idx beyond the stored half spectrum
    const int ybase = flip0 ? LL * YR + (LL - idx) : idx;
    const int ystep = flip0 ? -YR : YR;
    for (; i < n; i += gstride) {
        const float2* Y = Yb + buf * a.ybuf;
        float4* const smz_scratch = OVL ? reinterpret_cast<float4*>(red2) + 8 * (ovl_j & 1) : smz_scratch0;
        if constexpr (OVL) {
            prefetch(i + gstride, nxt(buf));
            tc::mbar_wait(ovl_full0 + 8 * buf, (ovl_fph >> buf) & 1u);  // this observation's Yhat has landed
            ovl_fph ^= 1u << buf;
            ++ovl_j;
        }
        float row_s = 0.f, row_m = -INFINITY, row_za = 0.f, row_zb = 0.f;  // OVL: this row's softmax summary

        float2 v[LL];
        float sref = 0.f, mall = 0.f, zall = 1.f;
        // Four 1-D transform passes share ONE register FFT (forward); the two inverse passes use
        // ifft(z) = conj(fft(conj(z))), with the conjugations folded into the loads / score read-out.
        // The four passes as four code bodies (pass-specific addressing and control resolved at compile time):
        // measured c3 4.57 -> 3.69 ms, c1 0.0947 -> 0.0860 ms against one shared body selected per pass
        // (SRMRA_FFT_PASS_ROLLED builds the shared-body variant for A/B).
#ifdef SRMRA_FFT_PASS_ROLLED
#pragma unroll 1
#else
#pragma unroll
#endif
        for (int pass = 0; pass < 4; ++pass) {
            if (line_ok || (TACC && pass == 3)) {  // tcgen05.ld/st are warp-collective
                if (pass == 0) {
                    // E-step along k1 (column k2 = idx): conj of Z = Yhat conj(Xhat_ra) + i Yhat conj(Xhat_rb);
                    // columns k2 >= LH by Hermitian symmetry from the stored half
                    const int k2 = idx;
                    const bool flip = k2 >= LH;
                    const int sk2 = flip ? LL - k2 : k2;
                    const float sgn = flip ? -1.f : 1.f;
                    // all of this column's Yhat reads first (LL loads in flight), the TMEM stash, then the
                    // products in place; at LL <= 32 with the XS = 2 table its coefficient reads are issued first too
                    constexpr bool CF_FIRST = XS == 2 && LL <= 32;
                    float2 cfv[CF_FIRST ? LL : 1];
                    if constexpr (CF_FIRST) {
#pragma unroll
                        for (int k1 = 0; k1 < LL; ++k1) cfv[k1] = XP2[k1 * LL + idx];
                    }
#pragma unroll
                    for (int k1 = 0; k1 < LL; ++k1) v[k1] = Y[ybase + k1 * ystep];
                    if constexpr (TACC) {
#pragma unroll
                        for (int c8 = 0; c8 < LL; c8 += 8) {
                            float ys[16];
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                ys[2 * e] = v[c8 + e].x;
                                ys[2 * e + 1] = v[c8 + e].y;
                            }
                            tc::tmem_st16(tys + 2 * c8, ys);
                        }
                    }
#pragma unroll
                    for (int c8 = 0; c8 < LL; c8 += 8) {
#pragma unroll
                        for (int e = 0; e < 8 && c8 + e < LL; ++e) {
                            const int k1 = c8 + e;
                            const int sk1 = flip ? ((LL - k1) & M) : k1;
                            const int o = sk1 * LH + sk2;
                            const float2 yv = v[k1];
                            if constexpr (XS == 2) {
                                // (A, B), lane-contiguous; Y.y (b, d) = (-g Y.y) (-B, A): the pair as the first operand makes
                                // (-B, A) a free FFMA2 operand modifier (half the table of the (a, c, b, d) form: 8 B per bin)
                                float2 cf;
                                if constexpr (CF_FIRST) cf = cfv[k1];
                                else cf = XP2[k1 * LL + idx];
                                v[k1] = px::fma(cf, px::bc(yv.x), px::mul(make_float2(-cf.y, cf.x), px::bc(-sgn * yv.y)));
                            } else {
                                const float4 xv = XS ? XP[o] : __ldg(XP + o);
                                const float2 A = cmul_conj(yv, make_float2(xv.x, xv.y));
                                const float2 B = cmul_conj(yv, make_float2(xv.z, xv.w));
                                v[k1] = make_float2(A.x - sgn * B.y, -sgn * A.y - B.x);
                            }
                        }
                    }
                } else if (pass == 1) {
                    // E-step along k2 (row n1 = idx) of the conjugated column result
#pragma unroll
                    for (int k2 = 0; k2 < LL; k2 += 2) {
                        const float4 t = *reinterpret_cast<const float4*>(Wq + idx * WS + k2);
                        v[k2] = make_float2(t.x, t.y);
                        v[k2 + 1] = make_float2(t.z, t.w);
                    }
                } else if (pass == 3) {
                    // M-step along n1 (column c = idx)
#pragma unroll
                    for (int r = 0; r < LL; ++r) v[r] = Wq[r * WS + idx];
                }
                // pass 2: v holds the posterior row w of the pair (forward transform along n2)
                fft_sr2<LL, -1>(v);  // split radix, packed FP32x2 arithmetic
                if (OVL && pass == 2) {
                    // the cross-warp half of the softmax reduction, then w = e 2^((sref_t - Sref) c2 + mt - M) / Z
                    // applied to the transformed row (OVL implies L_low >= 32: every thread owns a line, so the
                    // whole warp is here for the shuffles)
                    if (nwarps > 1) {
                        tc::mbar_wait(ovl_mb, ovl_ph);
                        ovl_ph ^= 1;
                        smz_cross(sref, mall, zall, a.c2, smz_scratch, nwarps, pw, lane);
                    }
                    const float f = row_m == -INFINITY ? 0.f : ex2(fmaf(row_s - sref, a.c2, row_m - mall)) / zall;
                    rsumA = fmaf(row_za, f, rsumA);
                    rsumB = fmaf(row_zb, f, rsumB);
#pragma unroll
                    for (int n2 = 0; n2 < LL; ++n2) v[n2] = px::mul(v[n2], px::bc(f));
                }
                if (pass == 0) {
#pragma unroll
                    for (int k1 = 0; k1 < LL; ++k1) Wq[k1 * WS + idx] = v[k1];
                } else if (pass == 2) {
#pragma unroll
                    for (int k2 = 0; k2 < LL; k2 += 2)
                        *reinterpret_cast<float4*>(Wq + idx * WS + k2) = make_float4(v[k2].x, v[k2].y, v[k2 + 1].x, v[k2 + 1].y);
                } else if (pass == 3 && TACC) {
                    // U_q[k1][c] += Yhat[k1][c] conj(Z[k1]) (c < LH) | V_q[k1][LL-c] += Yhat[k1][LL-c] Z[-k1]
#pragma unroll
                    for (int ch = 0; ch < 2 * LL / 16; ++ch) {
                        float ac[16], ys[16];
                        tc::tmem_ld16x2(tys + 16 * ch, ys, tacc + 16 * ch, ac);
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const int k1 = 8 * ch + e;
                            const float2 z = v[k1];
                            const float zy = su * z.y;
                            // packed: (-y.y, y.x) is a free operand modifier of FFMA2 (swapped halves, one negated)
                            const float2 yy = make_float2(ys[2 * e], ys[2 * e + 1]);
                            const float2 r = px::fma(yy, px::bc(z.x),
                                                     px::fma(make_float2(-yy.y, yy.x), px::bc(zy), make_float2(ac[2 * e], ac[2 * e + 1])));
                            ac[2 * e] = r.x;
                            ac[2 * e + 1] = r.y;
                            if (vsrc) zc[q * (2 * LL + 2) + (idx == 0 ? 0 : LL + 1) + k1] = z;
                        }
                        tc::tmem_st16(tacc + 16 * ch, ac);
                    }
                    tc::tmem_wait_st();
                    cu.x += v[0].x;
                    cu.y += v[0].y;
                } else if (pass == 3) {
                    // v[k1] = Z[k1][c]: accumulate U (c < LH), V at column k2 = -c (c == 0 or c >= LL/2)
                    const int c = idx;
                    if (c < LH) {
#pragma unroll
                        for (int k1 = 0; k1 < LL; ++k1) {
                            const float2 yv = Y[k1 * YR + c];
                            const float2 u = cmul_conj(yv, v[k1]);
                            Uq[k1 * LH + c] = make_float2(Uq[k1 * LH + c].x + u.x, Uq[k1 * LH + c].y + u.y);
                        }
                    }
                    if (c == 0 || 2 * c >= LL) {
                        const int k2 = (LL - c) & M;
#pragma unroll
                        for (int k1 = 0; k1 < LL; ++k1) {
                            const float2 yv = Y[k1 * YR + k2];
                            const float2 z = v[(LL - k1) & M];
                            const float2 w = make_float2(fmaf(yv.x, z.x, -yv.y * z.y), fmaf(yv.x, z.y, yv.y * z.x));
                            Vq[k1 * LH + k2] = make_float2(Vq[k1 * LH + k2].x + w.x, Vq[k1 * LH + k2].y + w.y);
                        }
                    }
                    cu.x += v[0].x;
                    cu.y += v[0].y;
                }
            }
            if (pass == 1) {
                // ---- scores S_ra = Re, S_rb = -Im (inverse via conjugation); this row's reference
                float lmax = 0.f;
                if (line_ok) {
                    lmax = -INFINITY;
#pragma unroll
                    for (int n2 = 0; n2 < LL; ++n2) {
                        v[n2].y = -v[n2].y;
                        lmax = fmaxf(lmax, has_b ? fmaxf(v[n2].x, v[n2].y) : v[n2].x);
                    }
                }
                const float sref_t = lmax;
                // ---- posterior (eq:weights_EM) in log2 units: v2 = (S - sref_t) log2e/sigma^2 + bias
                float mt = -INFINITY, za = 0.f, zb = 0.f;
                const float2 biasAB = make_float2(biasA, biasB);
                if (line_ok) {
                    const float4* lq = reinterpret_cast<const float4*>(smem_raw + par_off_lrp<LL>(KK)) + q * (LL / 2);
#pragma unroll
                    for (int n2 = 0; n2 < LL; ++n2) {
                        float2 b2;
                        if constexpr (JOINT) {
                            b2 = __ldg(a.ljp + ((size_t)q * LL + n2) * LL + idx);
                        } else {
                            const float4 l4 = lq[n2 >> 1];
                            b2 = (n2 & 1) ? make_float2(l4.z, l4.w) : make_float2(l4.x, l4.y);
                        }
                        // (va, vb) = (S - sref_t) c2 + bias, both classes in packed FP32x2 (same rounding)
                        float2 vab = px::fma(px::sub(v[n2], px::bc(sref_t)), px::bc(a.c2), px::add(biasAB, b2));
                        if (!has_b) vab.y = -INFINITY;
                        v[n2] = vab;
                        mt = fmaxf(mt, fmaxf(vab.x, vab.y));
                    }
                    // a row whose shifts all have zero prior mass has mt = -inf: its weights are exactly 0
                    const float mref = mt == -INFINITY ? 0.f : mt;
                    float2 zab = make_float2(0.f, 0.f);
#pragma unroll
                    for (int n2 = 0; n2 < LL; ++n2) {
                        const float2 dm = px::sub(v[n2], px::bc(mref));
                        const float ea = ex2(dm.x);
                        const float eb = has_b ? ex2(dm.y) : 0.f;
                        v[n2] = make_float2(ea, eb);
                        zab = px::add(zab, v[n2]);
                    }
                    za = zab.x;
                    zb = zab.y;
                }
                sref = sref_t;
                mall = mt;
                zall = za + zb;
                if constexpr (OVL) {
                    // publish this warp's summary; the rows are transformed before the wait (pass 2)
                    row_s = sref_t;
                    row_m = mt;
                    row_za = za;
                    row_zb = zb;
                    smz_warp(sref, mall, zall, a.c2);
                    if (nwarps > 1 && lane == 0) {
                        smz_scratch[gwarp] = make_float4(sref, mall, zall, 0.f);
                        mbar_arrive(ovl_mb);
                    }
                } else {
                group_reduce_smz(sref, mall, zall, a.c2, smz_scratch, gwarp, nwarps, pw, lane, bar_id, GT);
                if (TACC) {
                    // the next observation's Yhat goes into the buffer vex_update read in pass 0: every thread of
                    // the group has passed the reduction's barrier, so none still reads it
                    if (nwarps == 1) __syncwarp();
                    prefetch(i + gstride, nxt(buf));
                }
                if (line_ok) {
                    // w = e 2^((sref_t - Sref) c2 + mt - M) / Z
                    const float f = mt == -INFINITY ? 0.f : ex2(fmaf(sref_t - sref, a.c2, mt - mall)) / zall;
                    rsumA = fmaf(za, f, rsumA);
                    rsumB = fmaf(zb, f, rsumB);
#pragma unroll
                    for (int n2 = 0; n2 < LL; ++n2) v[n2] = px::mul(v[n2], px::bc(f));
                    if constexpr (JOINT) {  // posterior mass of the shifts (ra | rb, t1 = idx, t2 = n2)
                        float* ja = JA + ((size_t)ra * LL + idx) * (LL + 1);
                        float* jb = JA + ((size_t)rb * LL + idx) * (LL + 1);
#pragma unroll
                        for (int n2 = 0; n2 < LL; ++n2) {
                            atomicAdd(ja + n2, v[n2].x);
                            if (has_b) atomicAdd(jb + n2, v[n2].y);
                        }
                    }
                }
                }  // !OVL
            }
            if (pass == 0) {
                // at LL = 32 a class pair's lines are exactly one warp: its transpose buffer, its zc rows and its
                // vex entries are warp-local, so the column -> row transpose needs only a warp barrier (the Yhat
                // buffers are ordered by the reduction and pass-2 group barriers)
                if constexpr (TACC && LL == 32) __syncwarp();
                else group_bar(bar_id, GT);
                if (TACC && vex_pending) vex_update(Yb + prv(buf) * a.ybuf);  // the previous observation's pass 3
                if (!TACC) prefetch(i + gstride, nxt(buf));
            } else if (pass == 2) {
                if constexpr (OVL) {
                    __syncwarp();  // the pair's transpose is warp-local at L_low = 32
                } else {
                    cp_async_wait0();
                    group_bar(bar_id, GT);
                }
            }
        }
        if (tg == 0) {
            const double lse = 0.69314718055994530942 * ((double)mall + (double)log2f(zall)) +
                               (double)sref * a.inv_s2 - (emin_g[g] + a.ynorm[i]) * a.inv_2s2;
            llg[g] += lse;
            if (a.llobs) a.llobs[i] = lse;
        }
        buf = nxt(buf);
        vex_pending = true;
    }
    cp_async_wait0();
    group_bar(bar_id, GT);
    if (TACC) {
        if (vex_pending) vex_update(Yb + prv(buf) * a.ybuf);
        // stage the TMEM accumulator lines and the V columns 0 / LL/2 as this group's partial (over Yb / Wk;
        // every thread of the group is past its last use of them)
        group_bar(bar_id, GT);
        float2* Uq = Acc + (size_t)(2 * q) * LL * LH;
        float2* Vq = Uq + (size_t)LL * LH;
#pragma unroll
        for (int ch = 0; ch < 2 * LL / 16; ++ch) {
            float ac[16];
            tc::tmem_ld16(tacc + 16 * ch, ac);
            if (line_ok) {
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int k1 = 8 * ch + e;
                    const float2 val = make_float2(ac[2 * e], ac[2 * e + 1]);
                    if (role_u) Uq[k1 * LH + idx] = val;
                    else Vq[((LL - k1) & M) * LH + (LL - idx)] = val;
                }
            }
        }
        if (line_ok) {
            Vq[idx * LH] = vex0;
            Vq[idx * LH + LL / 2] = vexh;
        }
    }
    // register accumulators -> this group's R / CU regions
    float2* R = Acc + 2 * NP * LL * LH;   // [KK][LL]
    float2* CU = R + KK * LL;             // [NP][LL]
    if (line_ok) {
        R[ra * LL + idx] = make_float2(rsumA, 0.f);
        if (has_b) R[rb * LL + idx] = make_float2(rsumB, 0.f);
        CU[q * LL + idx] = cu;
    }
    __syncthreads();
    // CTA partial (sum over groups in a fixed order) -> global slot of this CTA; the reduce kernel sums
    // the slots in a fixed order (deterministic, no atomics)
    float2* dst = a.part + (size_t)blockIdx.x * PB;
    const size_t acc_off = TACC ? 0 : 2 * (size_t)a.ybuf + (size_t)NP * LL * WS;  // float2 within a group
    for (int k = threadIdx.x; k < PB; k += blockDim.x) {
        float2 s = make_float2(0.f, 0.f);
        for (int gg = 0; gg < a.groups; ++gg) {
            const float2* A0 = reinterpret_cast<const float2*>(gbase + per_g * gg) + acc_off;
            s.x += A0[k].x;
            s.y += A0[k].y;
        }
        dst[k] = s;
    }
    if (JOINT) {
        float* jd = a.jpart + (size_t)blockIdx.x * KK * LL * LL;
        for (int k = threadIdx.x; k < KK * LL * LL; k += blockDim.x) {
            const int row = k / LL, c = k - row * LL;
            jd[k] = JA[row * (LL + 1) + c];
        }
    }
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int gg = 0; gg < a.groups; ++gg) s += llg[gg];
        a.llpart[blockIdx.x] = s;
    }
    if (TACC) {
        tc::fence_before();
        __syncthreads();
        if (threadIdx.x < 32) tc::tmem_dealloc_n(tmem_slot, a.tmem_cols);
    }
    // the last CTA to finish marks the launch's end
    __syncthreads();
    if (threadIdx.x == 0 && emt_slot >= 0 && emt_slot < a.emt_cap) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        atomicMax(a.emt + 2 * emt_slot + 1, t1);
    }
}

}  // namespace fftk

// ==================================================================== host side
using namespace fftk;

// Yhat row stride (float2): the stored half spectrum Lh = Ll/2 + 1; at Ll = 128 the rows are padded to
// 72 so that the staged copy is bank-conflict-free for the thread-pair access of k_fft128.cu
int yrow_of(int Ll) { return Ll == 128 ? 72 : Ll / 2 + 1; }

int ystride_of(int Ll) {
    const int n = Ll * yrow_of(Ll);
    return (n + 1) & ~1;  // even number of float2 -> 16-byte rows for cp.async / bulk copies
}
// shared-memory stride of one staged Yhat in k_fft_em: + a copy of row 0 (even number of float2)
int ybuf_of(int Ll) { return ystride_of(Ll) + ((yrow_of(Ll) + 1) & ~1); }

bool fft128_supported(int K);
cudaError_t fft128_plan(srmra_ctx* c);
cudaError_t launch_fft_em128(srmra_ctx* c);

bool fft_supported(int L, int Ll, int K) {
    if (Ll == 128) return fft128_supported(K);  // k_fft128.cu: class pairs on a CTA cluster
    if (Ll < 2 || Ll > 64 || (Ll & (Ll - 1))) return false;
    if (K * K > 64) return false;
    return true;
}

template <int LL, bool TACC, bool JOINT, int MAXT>
static auto em_kernel_m(int KK, int xs) {
    if (KK % 2 == 0)
        return xs == 2 ? k_fft_em<LL, true, 2, TACC, JOINT, MAXT>
                       : (xs == 1 ? k_fft_em<LL, true, 1, TACC, JOINT, MAXT> : k_fft_em<LL, true, 0, TACC, JOINT, MAXT>);
    return xs == 2 ? k_fft_em<LL, false, 2, TACC, JOINT, MAXT>
                   : (xs == 1 ? k_fft_em<LL, false, 1, TACC, JOINT, MAXT> : k_fft_em<LL, false, 0, TACC, JOINT, MAXT>);
}
// one 256-thread group per CTA at L_low = 32 (TACC): the MAXT = 256 instantiation (more registers per thread)
template <int LL, bool TACC>
constexpr bool big_group_variant() { return LL == 32 && TACC; }
template <int LL, bool TACC>
static bool use_big(int KK) { return big_group_variant<LL, TACC>() && 2 * group_threads<LL>(KK) > max_cta_threads<LL, TACC>(); }
template <int LL, bool TACC, bool JOINT>
static auto em_kernel(int KK, int xs) {
    if constexpr (big_group_variant<LL, TACC>()) {
        if (use_big<LL, TACC>(KK)) return em_kernel_m<LL, TACC, JOINT, 256>(KK, xs);
    }
    return em_kernel_m<LL, TACC, JOINT, max_cta_threads<LL, TACC>()>(KK, xs);
}

template <int LL, bool TACC, bool JOINT>
static cudaError_t plan_em_tt(srmra_ctx* c) {
    const int KK = c->KK;
    const int GT = group_threads<LL>(KK);
    const int ys = ybuf_of(LL);
    const int MAXT = use_big<LL, TACC>(KK) ? 256 : max_cta_threads<LL, TACC>();
    if (GT > MAXT) return cudaErrorInvalidConfiguration;
    const size_t jb = JOINT ? joint_bytes<LL>(KK) : 0;
    constexpr int NYB = ovl_mode<LL, TACC, JOINT>() ? 3 : 2;
    auto gsm = [&](int g) { return (TACC ? group_smem_t<LL>(KK, ys, NYB) : group_smem<LL>(KK, ys)) * g + par_bytes<LL>(KK) + jb; };
    int groups = MAXT / GT;
    if (groups > 15) groups = 15;
    const char* eg = getenv("SRMRA_FFT_GROUPS");  // tuning override
    if (eg && atoi(eg) > 0 && atoi(eg) < groups) groups = atoi(eg);
    // Xhat staged in shared memory unless that costs a group (SRMRA_FFT_XS=0/1/2 overrides): as the
    // product coefficients (mode 2) when they cost no group more than the plain staging (mode 1)
    const size_t xsb1 = xs_bytes<LL>(KK, 1), xsb2 = xs_bytes<LL>(KK, 2);
    int g_plain = groups, g_xs = groups, g_xs2 = groups;
    while (g_plain > 1 && gsm(g_plain) > 227 * 1024) --g_plain;
    while (g_xs > 1 && gsm(g_xs) + xsb1 > 227 * 1024) --g_xs;
    while (g_xs2 > 1 && gsm(g_xs2) + xsb2 > 227 * 1024) --g_xs2;
    // measured on B200 (tools/em_sweep.py, tools/path_timing.py): Xhat in shared memory with one group
    // fewer beat Xhat through L1 with the extra group at c1 (164 vs 177 us, 7 vs 6 groups), but at c2
    // staging halves the warps (1 group instead of 2) and costs 43 % (1.697 vs 1.184 ms): stage only when
    // it costs no group, or one group out of four or more
    int xs = (gsm(g_xs) + xsb1 <= 227 * 1024 && (g_xs == g_plain || (g_xs >= 4 && g_xs + 1 >= g_plain))) ? 1 : 0;
    if (xs && g_xs2 == g_xs && gsm(g_xs2) + xsb2 <= 227 * 1024) xs = 2;
    const char* ex = getenv("SRMRA_FFT_XS");
    if (ex) {
        xs = atoi(ex);
        if (xs < 0 || xs > 2 || gsm(1) + xs_bytes<LL>(KK, xs ? xs : 1) * (xs ? 1 : 0) > 227 * 1024) xs = 0;
    }
    const size_t xsb = xs ? xs_bytes<LL>(KK, xs) : 0;
    groups = xs == 2 ? g_xs2 : (xs == 1 ? g_xs : g_plain);
    while (groups > 1 && gsm(groups) + xsb > 227 * 1024) --groups;
    // keep enough CTAs for all SMs when N is small
    const int64_t need = (c->n_local + c->num_sms - 1) / c->num_sms;
    if (need < groups) groups = (int)(need < 1 ? 1 : need);
    const size_t smem = gsm(groups) + xsb;
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    auto kern = em_kernel<LL, TACC, JOINT>(KK, xs);
    c->fft_xs = xs;
    c->fft_tacc = TACC;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // = the tail's
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, GT * groups, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    // TACC: tensor-memory columns per CTA (one 2 LL-column line per thread, 4 warps share the 128 lanes);
    // the CTAs resident on one SM must fit the 512 columns together
    int cols = 32;
    while (cols < ((GT * groups / 32 + 3) / 4) * 4 * LL) cols *= 2;  // accumulator + Yhat stash lines
    if (TACC && cols > 512) return cudaErrorInvalidConfiguration;
    if (TACC && per_sm * cols > 512) per_sm = 512 / cols;
    c->fft_tmem_cols = TACC ? cols : 0;
    int64_t grid = (int64_t)c->num_sms * per_sm;
    const int64_t max_grid = (c->n_local + groups - 1) / groups;
    if (grid > max_grid) grid = max_grid;
    if (c->opt.grid_cap > 0 && grid > c->opt.grid_cap) grid = c->opt.grid_cap;  // test hook: several obs per CTA
    if (c->fft_part_cap > 0 && grid > c->fft_part_cap) grid = c->fft_part_cap;  // partial buffers of the first plan
    if (grid < 1) grid = 1;
    c->fft_grid = (int)grid;
    c->fft_joint = JOINT;
    c->fft_groups = groups;
    c->fft_threads = GT * groups;
    c->fft_smem = smem;
    return cudaSuccess;
}

template <int LL, bool JOINT>
static cudaError_t plan_em_tj(srmra_ctx* c) {
    // tensor-memory accumulators where the staged partial fits (L_low >= 32); SRMRA_FFT_TACC=0 disables
    const char* et = getenv("SRMRA_FFT_TACC");
    const bool tacc_ok = LL >= 32 && tacc_fits<LL>(c->KK, ybuf_of(LL)) && !(et && atoi(et) == 0);
    if constexpr (LL >= 32) {
        if (tacc_ok && plan_em_tt<LL, true, JOINT>(c) == cudaSuccess) return cudaSuccess;
        cudaGetLastError();
    }
    return plan_em_tt<LL, false, JOINT>(c);
}
template <int LL>
static cudaError_t plan_em_t(srmra_ctx* c) {
    return c->fft_joint ? plan_em_tj<LL, true>(c) : plan_em_tj<LL, false>(c);
}

template <int LL>
static cudaError_t launch_em_t(srmra_ctx* c) {
    EmArgs a;
    const int64_t off = c->em_n >= 0 ? c->em_off : 0;  // srmra_load_iterate: one observation range
    a.yhat = c->d_yhat + off * ystride_of(LL);
    a.ynorm = c->d_ynorm + off;
    a.xhat = reinterpret_cast<const float4*>(c->d_xhat);
    a.par32 = c->par.f32;
    a.par64 = c->par.f64;
    a.n = c->em_n >= 0 ? c->em_n : c->n_local;
    a.L = c->L;
    a.K = c->K;
    a.KK = c->KK;
    a.ystride = ystride_of(LL);
    a.ybuf = ybuf_of(LL);
    a.groups = c->fft_groups;
    a.c2 = (float)(1.4426950408889634074 * c->inv_s2);
    a.inv_s2 = c->inv_s2;
    a.inv_2s2 = c->inv_2s2;
    a.part = c->em_n >= 0 ? c->em_part : c->d_part;
    a.llpart = c->em_n >= 0 ? c->em_llpart : c->d_llpart;
    a.llobs = c->d_llobs ? c->d_llobs + off : nullptr;
    a.tmem_cols = c->fft_tmem_cols;
    a.run = c->d_run;
    a.emt = c->d_emt;
    a.iter = c->d_iter;
    a.emt_cap = c->opt.trace_cap;
    a.ljp = c->d_ljp;
    a.jpart = c->d_jpart;
#define SRMRA_EM_LAUNCH(T, J)                                                                                        \
    em_kernel<LL, T, J>(c->KK, c->fft_xs)<<<(unsigned)c->fft_grid, c->fft_threads, c->fft_smem, c->stream>>>(a); \
    return cudaGetLastError()
    if constexpr (LL >= 32) {
        if (c->fft_tacc) {
            if (c->fft_joint) { SRMRA_EM_LAUNCH(true, true); }
            SRMRA_EM_LAUNCH(true, false);
        }
    }
    if (c->fft_joint) { SRMRA_EM_LAUNCH(false, true); }
    SRMRA_EM_LAUNCH(false, false);
#undef SRMRA_EM_LAUNCH
}

int fft_partial_bins(int KK, int Ll) { return part_bins(KK, Ll); }
// hi plane | lo plane (x_hat = hi + lo, both float32; the lo plane is read by k_fft128.cu)
size_t fft_xhat_float2(int KK, int Ll) { return (size_t)4 * ((KK + 1) / 2) * Ll * (Ll / 2 + 1); }
size_t fft_bhat_doubles(int KK, int Ll) { return (size_t)2 * fft_partial_bins(KK, Ll) + 1; }  // + LL
size_t fft_yhat_stride(int Ll) { return (size_t)ystride_of(Ll); }
size_t fft_part_float2(const srmra_ctx* c) { return (size_t)c->fft_grid * fft_partial_bins(c->KK, c->Ll); }

#define SRMRA_LL_DISPATCH(FN, c)                 \
    switch ((c)->Ll) {                           \
        case 2: return FN<2>(c);                 \
        case 4: return FN<4>(c);                 \
        case 8: return FN<8>(c);                 \
        case 16: return FN<16>(c);               \
        case 32: return FN<32>(c);               \
        case 64: return FN<64>(c);               \
        default: return cudaErrorInvalidValue;   \
    }

static cudaError_t fft_plan_ll(srmra_ctx* c) { SRMRA_LL_DISPATCH(plan_em_t, c) }

cudaError_t fft_plan(srmra_ctx* c) {
    if (c->Ll == 128) return fft128_plan(c);
    const cudaError_t e = fft_plan_ll(c);
    if (e == cudaSuccess && c->fft_part_cap == 0) c->fft_part_cap = c->fft_grid;
    return e;
}

// NEXT-3 on the FFT path (L_low <= 64): re-plan the E/M kernel with / without the joint-prior accumulator
// (fewer groups may fit; the grid stays within the partial buffers of the first plan)
cudaError_t fft_plan_joint(srmra_ctx* c, bool joint) {
    if (c->Ll == 128) return cudaErrorNotSupported;
    const bool old = c->fft_joint;
    c->fft_joint = joint;
    const cudaError_t e = fft_plan_ll(c);
    if (e != cudaSuccess) {
        cudaGetLastError();
        c->fft_joint = old;
        fft_plan_ll(c);
    }
    return e;
}
size_t fft_joint_bins(int KK, int Ll) { return (size_t)KK * Ll * Ll; }

cudaError_t launch_fft_em(srmra_ctx* c) {
    if (c->n_local == 0) return cudaSuccess;
    if (c->Ll == 128) return launch_fft_em128(c);
    SRMRA_LL_DISPATCH(launch_em_t, c)
}

// prep, em, reduce, fold
// E/M kernel (if the shard is non-empty) + tail (+ a separate reduce-only tail when world > 1)
int fft_launches_per_iter(const srmra_ctx* c) {
    const int em = c->n_local > 0 ? (c->Ll == 128 ? 2 : 1) : 0;  // L_low = 128: + the product-coefficient kernel
    return em + 1 + (c->opt.world > 1 ? 1 : 0);
}
// (with world > 1 the NCCL all-reduce kernel between the two tails is NCCL's, not counted here)

}  // namespace srmra
