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
// registers (radix-2, compile-time twiddles); the row/column transposes go through a padded shared
// buffer (row stride L_low + 1 float2: conflict-free for both row and column access).  The scores of
// the observation never leave registers: softmax (3 group reductions) runs on them, and the row
// thread immediately starts the forward transform of the posterior.  Yhat_i is prefetched with
// cp.async into a double buffer; Xhat (per-iteration, <= 70 KB) is read through the L1/read-only
// path; Bhat is accumulated per CTA in shared memory (float32) and added to the float64 global
// accumulator once at the end.
#include <math.h>

#include <utility>

#include "srmra_internal.cuh"

namespace srmra {
namespace fftk {

// ------------------------------------------------------------------ compile-time twiddles
constexpr double kPi = 3.14159265358979323846264338327950288;

constexpr double sin_series(double x) {
    double t = x, s = x;
    for (int n = 1; n < 20; ++n) {
        t *= -x * x / ((2.0 * n) * (2.0 * n + 1.0));
        s += t;
    }
    return s;
}
constexpr double cos_series(double x) {
    double t = 1.0, s = 1.0;
    for (int n = 1; n < 20; ++n) {
        t *= -x * x / ((2.0 * n - 1.0) * (2.0 * n));
        s += t;
    }
    return s;
}
// cos(2 pi k / n) and sin(2 pi k / n), exact at multiples of pi/2
constexpr double cos2pi(int k, int n) {
    k %= n;
    if (k < 0) k += n;
    if (k == 0) return 1.0;
    if (2 * k == n) return -1.0;
    if (4 * k == n || 4 * k == 3 * n) return 0.0;
    return cos_series(2.0 * kPi * k / n);
}
constexpr double sin2pi(int k, int n) {
    k %= n;
    if (k < 0) k += n;
    if (k == 0 || 2 * k == n) return 0.0;
    if (4 * k == n) return 1.0;
    if (4 * k == 3 * n) return -1.0;
    return sin_series(2.0 * kPi * k / n);
}
constexpr int bitrev(int i, int n) {
    int r = 0;
    for (int b = 1; b < n; b <<= 1) {
        r = (r << 1) | (i & 1);
        i >>= 1;
    }
    return r;
}

// ------------------------------------------------------------------ register FFT (radix 2)
// In place, natural order in and out, unnormalised; SIGN = -1 forward, +1 inverse.
template <int N, int SIGN, int LEN, int I, int J>
__device__ __forceinline__ void bfly(float2* t) {
    constexpr int TK = J * (N / LEN);
    const float2 a = t[I + J], b = t[I + J + LEN / 2];
    float2 bw;
    if constexpr (TK == 0) {
        bw = b;
    } else if constexpr (4 * TK == N) {
        if constexpr (SIGN > 0) bw = make_float2(-b.y, b.x);   // b * (+i)
        else bw = make_float2(b.y, -b.x);                      // b * (-i)
    } else {
        constexpr float c = (float)cos2pi(TK, N);
        constexpr float s = (float)(SIGN * sin2pi(TK, N));
        bw = make_float2(fmaf(b.x, c, -b.y * s), fmaf(b.x, s, b.y * c));
    }
    t[I + J] = make_float2(a.x + bw.x, a.y + bw.y);
    t[I + J + LEN / 2] = make_float2(a.x - bw.x, a.y - bw.y);
}
template <int N, int SIGN, int LEN, int I, int... Js>
__device__ __forceinline__ void bfly_block(float2* t, std::integer_sequence<int, Js...>) {
    (bfly<N, SIGN, LEN, I, Js>(t), ...);
}
template <int N, int SIGN, int LEN, int... Bs>
__device__ __forceinline__ void fft_stage(float2* t, std::integer_sequence<int, Bs...>) {
    (bfly_block<N, SIGN, LEN, Bs * LEN>(t, std::make_integer_sequence<int, LEN / 2>{}), ...);
}
template <int N, int SIGN, int... Ls>
__device__ __forceinline__ void fft_stages(float2* t, std::integer_sequence<int, Ls...>) {
    (fft_stage<N, SIGN, (2 << Ls)>(t, std::make_integer_sequence<int, N / (2 << Ls)>{}), ...);
}
constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }
template <int N, int... Is>
__device__ __forceinline__ void bitrev_copy(float2* t, const float2* v, std::integer_sequence<int, Is...>) {
    ((t[Is] = v[bitrev(Is, N)]), ...);
}
template <int N, int SIGN>
__device__ __forceinline__ void fft(float2 (&v)[N]) {
    float2 t[N];
    bitrev_copy<N>(t, v, std::make_integer_sequence<int, N>{});
    fft_stages<N, SIGN>(t, std::make_integer_sequence<int, ilog2(N)>{});
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = t[i];
}

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
    group_bar(bar_id, gthreads);  // scratch reusable
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
    const float2* xhat;     // [KK][Ll][Lh] rfft2(x_r) / Ll^2
    const float* par32;     // lr1[L] | lr2[L] | beta[KK]
    const double* par64;    // E[KK] | E_min
    int64_t n;
    int L, K, KK, ystride, groups;
    float inv_s2f;
    double inv_s2, inv_2s2;
    float2* part;           // [gridDim.x][PB] per-CTA partials: Bhat [KK][Ll][Lh] | mass lines [KK][Ll+Lh]
    double* llpart;         // [gridDim.x] per-CTA log-likelihood partials
    double* llobs;          // [n]
};

template <int LL>
struct Geo {
    static constexpr int LH = LL / 2 + 1;
    static constexpr int WS = LL + 1;  // padded row stride of the transpose buffer (float2)
};

template <int LL>
__host__ __device__ constexpr int group_threads(int KK) {
    return ((((KK + 1) / 2) * LL + 31) / 32) * 32;
}

// Shared memory of one group (16-B multiple):
//   Yb [2][ystride] | Wk [NP][LL][WS] | Bs [KK][LL][LH] | Cs [KK][LL+LH] (float2) | red [32] (double)
// Every group owns its own Bhat / mass-line accumulators, so the bin pass needs no atomics.
template <int LL>
__host__ __device__ inline size_t group_smem(int KK, int ystride) {
    using G = Geo<LL>;
    const int NP = (KK + 1) / 2;
    size_t b = sizeof(float2) * (2 * (size_t)ystride + (size_t)NP * LL * G::WS + (size_t)KK * LL * G::LH +
                                 (size_t)KK * (LL + G::LH)) + sizeof(double) * 32;
    return (b + 15) & ~(size_t)15;
}
template <int LL>
__host__ __device__ inline size_t smem_bytes(int KK, int groups, int ystride) {
    return group_smem<LL>(KK, ystride) * groups;
}

// Threads per CTA cap (register budget: one L_low-point complex line per thread lives in registers)
template <int LL>
__host__ __device__ constexpr int max_cta_threads() {
    return LL >= 64 ? 256 : (LL >= 32 ? 384 : (LL >= 16 ? 512 : 1024));
}

template <int LL>
__global__ void __launch_bounds__(max_cta_threads<LL>(), 1) k_fft_em(EmArgs a) {
    using G = Geo<LL>;
    constexpr int LH = G::LH, WS = G::WS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int KK = a.KK, K = a.K, L = a.L;
    const int NP = (KK + 1) / 2;
    const int GT = group_threads<LL>(KK);
    const int g = threadIdx.x / GT;        // group
    const int tg = threadIdx.x - g * GT;   // thread in group
    const int lane = threadIdx.x & 31;
    const int gwarp = tg >> 5, nwarps = GT >> 5;
    const int bar_id = 1 + g;

    // ---- shared layout
    const size_t per_g = group_smem<LL>(KK, a.ystride);
    float2* Yb = reinterpret_cast<float2*>(smem_raw + per_g * g);      // [2][ystride]
    float2* Wk = Yb + 2 * a.ystride;                                    // [NP][LL][WS]
    float2* Bs = Wk + (size_t)NP * LL * WS;                             // [KK][LL][LH]
    float2* Cs = Bs + (size_t)KK * LL * LH;                             // [KK][LL + LH]
    double* red = reinterpret_cast<double*>(Cs + (size_t)KK * (LL + LH));  // [32]
    float* redf = reinterpret_cast<float*>(red);

    for (int k = tg; k < KK * LL * LH; k += GT) Bs[k] = make_float2(0.f, 0.f);
    for (int k = tg; k < KK * (LL + LH); k += GT) Cs[k] = make_float2(0.f, 0.f);
    group_bar(bar_id, GT);

    const float* lr1 = a.par32;
    const float* lr2 = a.par32 + L;
    const float* beta = a.par32 + 2 * L;
    const double emin = a.par64[KK];

    // line owned by this thread in the row / column passes: pair q, index idx
    const bool line_ok = tg < NP * LL;
    const int q = line_ok ? tg / LL : 0;
    const int idx = line_ok ? tg - q * LL : 0;
    const int ra = 2 * q, rb = 2 * q + 1;
    const bool has_b = rb < KK;
    const float2* XA = a.xhat + (size_t)ra * LL * LH;
    const float2* XB = a.xhat + (size_t)(has_b ? rb : ra) * LL * LH;
    float2* Wq = Wk + (size_t)q * LL * WS;

    double ll_acc = 0.0;
    const int64_t gstride = (int64_t)gridDim.x * a.groups;
    int64_t i = (int64_t)blockIdx.x * a.groups + g;
    int buf = 0;
    auto prefetch = [&](int64_t obs, int b) {
        if (obs < a.n) {
            const float2* src = a.yhat + obs * a.ystride;
            float2* dst = Yb + b * a.ystride;
            for (int c = tg; c < a.ystride / 2; c += GT) cp_async16(dst + 2 * c, src + 2 * c);
        }
        cp_async_commit();
    };
    prefetch(i, 0);

    for (; i < a.n; i += gstride) {
        prefetch(i + gstride, buf ^ 1);
        cp_async_wait1();
        group_bar(bar_id, GT);
        const float2* Y = Yb + buf * a.ystride;

        float2 v[LL];
        // ================= E-step, pass 1: product + inverse FFT along k1 (column k2 = idx)
        if (line_ok) {
            const int k2 = idx;
            // columns k2 >= LH come from the stored half by Hermitian symmetry: A[k] = conj(A[-k])
            const bool flip = k2 >= LH;
            const int sk2 = flip ? LL - k2 : k2;
            const float sgn = flip ? -1.f : 1.f;
#pragma unroll
            for (int k1 = 0; k1 < LL; ++k1) {
                const int sk1 = flip ? ((LL - k1) & (LL - 1)) : k1;
                const int o = sk1 * LH + sk2;
                const float2 yv = Y[o];
                const float2 A = cmul_conj(yv, __ldg(XA + o));
                float2 B = make_float2(0.f, 0.f);
                if (has_b) B = cmul_conj(yv, __ldg(XB + o));
                // Z = A + i B with A, B conjugated on the mirrored half
                v[k1] = make_float2(A.x - sgn * B.y, sgn * A.y + B.x);
            }
            fft<LL, +1>(v);
#pragma unroll
            for (int n1 = 0; n1 < LL; ++n1) Wq[n1 * WS + k2] = v[n1];
        }
        group_bar(bar_id, GT);
        // ================= E-step, pass 2: inverse FFT along k2 (row n1 = idx) -> scores
        const int n1 = idx;
        float lmax = -INFINITY;
        if (line_ok) {
#pragma unroll
            for (int k2 = 0; k2 < LL; ++k2) v[k2] = Wq[n1 * WS + k2];
            fft<LL, +1>(v);   // v[n2] = (S_ra[n1][n2], S_rb[n1][n2])
#pragma unroll
            for (int n2 = 0; n2 < LL; ++n2) lmax = fmaxf(lmax, has_b ? fmaxf(v[n2].x, v[n2].y) : v[n2].x);
        }
        const float sref = group_reduce<float, true>(lmax, redf, gwarp, nwarps, lane, bar_id, GT);
        // ================= posterior (eq:weights_EM), logits in the form of k_common.cu
        const int ra1 = ra / K, ra2 = ra - ra1 * K;
        const int rb1 = rb / K, rb2 = rb - rb1 * K;
        float vmax = -INFINITY;
        if (line_ok) {
            const float biasA = lr1[ra1 + K * n1] + beta[ra];
            const float biasB = has_b ? lr1[rb1 + K * n1] + beta[rb] : -INFINITY;
#pragma unroll
            for (int n2 = 0; n2 < LL; ++n2) {
                const float va = fmaf(v[n2].x - sref, a.inv_s2f, biasA + lr2[ra2 + K * n2]);
                const float vb = has_b ? fmaf(v[n2].y - sref, a.inv_s2f, biasB + lr2[rb2 + K * n2]) : -INFINITY;
                v[n2] = make_float2(va, vb);
                vmax = fmaxf(vmax, fmaxf(va, vb));
            }
        }
        const float m = group_reduce<float, true>(vmax, redf, gwarp, nwarps, lane, bar_id, GT);
        float zs = 0.f;
        if (line_ok) {
#pragma unroll
            for (int n2 = 0; n2 < LL; ++n2) {
                const float ea = __expf(v[n2].x - m);
                const float eb = has_b ? __expf(v[n2].y - m) : 0.f;
                v[n2] = make_float2(ea, eb);
                zs += ea + eb;
            }
        }
        const double Z = group_reduce<double, false>((double)zs, red, gwarp, nwarps, lane, bar_id, GT);
        if (tg == 0) {
            const double lse = (double)sref * a.inv_s2 + (double)m + log(Z) - (emin + a.ynorm[i]) * a.inv_2s2;
            ll_acc += lse;
            if (a.llobs) a.llobs[i] = lse;
        }
        const float invZ = (float)(1.0 / Z);
        // ================= M-step, pass 1: forward FFT of the posterior rows (n1 = idx)
        if (line_ok) {
#pragma unroll
            for (int n2 = 0; n2 < LL; ++n2) v[n2] = make_float2(v[n2].x * invZ, v[n2].y * invZ);
            fft<LL, -1>(v);
#pragma unroll
            for (int k2 = 0; k2 < LL; ++k2) Wq[n1 * WS + k2] = v[k2];
        }
        group_bar(bar_id, GT);
        // ================= M-step, pass 2: forward FFT along n1 (column k2 = idx)
        if (line_ok) {
            const int k2 = idx;
#pragma unroll
            for (int r = 0; r < LL; ++r) v[r] = Wq[r * WS + k2];
            fft<LL, -1>(v);
#pragma unroll
            for (int k1 = 0; k1 < LL; ++k1) Wq[k1 * WS + k2] = v[k1];
        }
        group_bar(bar_id, GT);
        // ================= M-step, pass 3: separate the pair, accumulate Bhat and the mass lines
        for (int bin = tg; bin < NP * LL * LH; bin += GT) {
            const int qq = bin / (LL * LH);
            const int rem = bin - qq * LL * LH;
            const int k1 = rem / LH, k2 = rem - (rem / LH) * LH;
            const float2* W = Wk + (size_t)qq * LL * WS;
            const float2 za = W[k1 * WS + k2];
            const float2 zb = W[((LL - k1) & (LL - 1)) * WS + ((LL - k2) & (LL - 1))];
            const float2 wa = make_float2(0.5f * (za.x + zb.x), 0.5f * (za.y - zb.y));   // (Z + conj Z-)/2
            const float2 wb = make_float2(0.5f * (za.y + zb.y), 0.5f * (zb.x - za.x));   // (Z - conj Z-)/2i
            const float2 yv = Y[k1 * LH + k2];
            // each bin of this group is owned by exactly one of its threads: plain read-modify-write
            const int rA = 2 * qq, rB = 2 * qq + 1;
            const float2 ba = cmul_conj(yv, wa);
            float2* BA = Bs + (size_t)rA * LL * LH + rem;
            *BA = make_float2(BA->x + ba.x, BA->y + ba.y);
            float2* CA = Cs + (size_t)rA * (LL + LH);
            if (k2 == 0) CA[k1] = make_float2(CA[k1].x + wa.x, CA[k1].y + wa.y);
            if (k1 == 0) CA[LL + k2] = make_float2(CA[LL + k2].x + wa.x, CA[LL + k2].y + wa.y);
            if (rB < KK) {
                const float2 bb = cmul_conj(yv, wb);
                float2* BB = Bs + (size_t)rB * LL * LH + rem;
                *BB = make_float2(BB->x + bb.x, BB->y + bb.y);
                float2* CB = Cs + (size_t)rB * (LL + LH);
                if (k2 == 0) CB[k1] = make_float2(CB[k1].x + wb.x, CB[k1].y + wb.y);
                if (k1 == 0) CB[LL + k2] = make_float2(CB[LL + k2].x + wb.x, CB[LL + k2].y + wb.y);
            }
        }
        group_bar(bar_id, GT);
        buf ^= 1;
    }
    cp_async_wait0();
    if (tg == 0) red[31] = ll_acc;
    __syncthreads();
    // CTA partial (sum over groups in a fixed order) -> global partial slot of this CTA; the reduce
    // kernel sums the slots in a fixed order (deterministic, no atomics)
    const int PB = KK * LL * LH + KK * (LL + LH);
    float2* dst = a.part + (size_t)blockIdx.x * PB;
    for (int k = threadIdx.x; k < PB; k += blockDim.x) {
        float2 s = make_float2(0.f, 0.f);
        for (int gg = 0; gg < a.groups; ++gg) {
            const float2* B0 = reinterpret_cast<const float2*>(smem_raw + per_g * gg) + 2 * a.ystride + (size_t)NP * LL * WS;
            s.x += B0[k].x;
            s.y += B0[k].y;
        }
        dst[k] = s;
    }
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int gg = 0; gg < a.groups; ++gg) {
            const float2* B0 = reinterpret_cast<const float2*>(smem_raw + per_g * gg) + 2 * a.ystride + (size_t)NP * LL * WS;
            s += reinterpret_cast<const double*>(B0 + PB)[31];
        }
        a.llpart[blockIdx.x] = s;
    }
}

}  // namespace fftk

// ==================================================================== host side
using namespace fftk;

int ystride_of(int Ll) {
    const int n = Ll * (Ll / 2 + 1);
    return (n + 1) & ~1;  // even number of float2 -> 16-byte rows for cp.async
}

bool fft_supported(int L, int Ll, int K) {
    if (Ll < 2 || Ll > 64 || (Ll & (Ll - 1))) return false;
    if (K * K > 64) return false;
    return true;
}

template <int LL>
static cudaError_t plan_em_t(srmra_ctx* c) {
    const int KK = c->KK;
    const int GT = group_threads<LL>(KK);
    const int ys = ystride_of(LL);
    if (GT > max_cta_threads<LL>()) return cudaErrorInvalidConfiguration;
    int groups = max_cta_threads<LL>() / GT;
    if (groups > 15) groups = 15;
    // shared-memory budget: 227 KB per CTA
    while (groups > 1 && smem_bytes<LL>(KK, groups, ys) > 227 * 1024) --groups;
    // keep enough CTAs for all SMs when N is small
    const int64_t need = (c->n_local + c->num_sms - 1) / c->num_sms;
    if (need < groups) groups = (int)(need < 1 ? 1 : need);
    const size_t smem = smem_bytes<LL>(KK, groups, ys);
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(k_fft_em<LL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fft_em<LL>, GT * groups, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t grid = (int64_t)c->num_sms * per_sm;
    const int64_t max_grid = (c->n_local + groups - 1) / groups;
    if (grid > max_grid) grid = max_grid;
    if (grid < 1) grid = 1;
    c->fft_grid = (int)grid;
    c->fft_groups = groups;
    c->fft_threads = GT * groups;
    c->fft_smem = smem;
    return cudaSuccess;
}

template <int LL>
static cudaError_t launch_em_t(srmra_ctx* c) {
    EmArgs a;
    a.yhat = c->d_yhat;
    a.ynorm = c->d_ynorm;
    a.xhat = c->d_xhat;
    a.par32 = c->par.f32;
    a.par64 = c->par.f64;
    a.n = c->n_local;
    a.L = c->L;
    a.K = c->K;
    a.KK = c->KK;
    a.ystride = ystride_of(LL);
    a.groups = c->fft_groups;
    a.inv_s2f = (float)c->inv_s2;
    a.inv_s2 = c->inv_s2;
    a.inv_2s2 = c->inv_2s2;
    a.part = c->d_part;
    a.llpart = c->d_llpart;
    a.llobs = c->d_llobs;
    k_fft_em<LL><<<(unsigned)c->fft_grid, c->fft_threads, c->fft_smem, c->stream>>>(a);
    return cudaGetLastError();
}

int fft_partial_bins(int KK, int Ll) { return KK * Ll * (Ll / 2 + 1) + KK * (Ll + Ll / 2 + 1); }
size_t fft_bhat_doubles(int KK, int Ll) { return (size_t)2 * fft_partial_bins(KK, Ll); }
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

cudaError_t fft_plan(srmra_ctx* c) { SRMRA_LL_DISPATCH(plan_em_t, c) }

cudaError_t launch_fft_em(srmra_ctx* c) {
    if (c->n_local == 0) return cudaSuccess;
    SRMRA_LL_DISPATCH(launch_em_t, c)
}

// prep, em, reduce, fold
int fft_launches_per_iter(const srmra_ctx* c) { return 2 + (c->n_local > 0 ? 2 : 0); }

}  // namespace srmra
