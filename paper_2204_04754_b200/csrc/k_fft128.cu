// k_fft128.cu — FFT-path E-step + M-step for L_low = 128 (configs[4]: L_high = 256, K = 2).
//
// Same mathematics as k_fft.cu (sub-image form of the likelihood; eq:weights_EM,
// eq:x_EM with P^{-1} := P^T, eq:rho_EM): for observation i and class pair q = (2q, 2q+1)
//     S_{i,2q} + i S_{i,2q+1} = ifft2( Yhat_i conj(Xhat_2q) + i Yhat_i conj(Xhat_2q+1) )   (E-step scores)
//     U_q += Yhat_i conj(Z_{i,q}),  V_q += Yhat_i Z_{i,q}(-k),  Z_{i,q} = fft2(w_{i,2q} + i w_{i,2q+1})
// but at L_low = 128 one pair's 128 x 128 complex working transform (128 KB) and its M-step
// accumulators (133 KB) no longer fit next to each other in one SM, so the layout changes:
//
//  * one CTA per class pair; the K^2/2 pairs of an observation run on the CTAs of ONE thread-block
//    cluster, which exchange their softmax partials (max reference, max, scaled sum) through
//    distributed shared memory once per observation (the log-sum-exp over all L_high^2 shifts);
//  * 256 threads, a thread PAIR per 128-point line: each thread does a 64-point register FFT and
//    the radix-2 stage across the pair goes through warp shuffles (DIT for the inverse passes:
//    parity-split input, half-split output; DIF for the forward passes: half-split input,
//    parity-split output — so the E-row output feeds the M-row input in registers, and the M-col
//    output keeps k1 and -k1 in the same thread);
//  * the transpose buffer is an XOR-swizzled 128 x 128 float2 array (conflict-free for all four
//    access patterns, no padding);
//  * Yhat_i (row stride 72 float2) is brought into shared memory by ONE bulk copy per observation
//    (cp.async.bulk + mbarrier), issued as soon as the previous observation's E-column pass is done;
//  * the M-step accumulators U_q / V_q live in TENSOR MEMORY (256 KB per SM): each thread owns one
//    TMEM lane segment of 128 columns for its accumulator line and 128 columns for the Yhat values
//    it read in the E-column pass (exactly the ones its M-column pass needs), tcgen05.ld/st move
//    them; the two columns (0 and 64) that need both U and V add V through a small shared stage.
#include <math.h>
#include <stdlib.h>

#include "regfft.cuh"
#include "srmra_internal.cuh"
#include "tcgen05.cuh"

namespace srmra {

int ystride_of(int Ll);
int fft_partial_bins(int KK, int Ll);

namespace fft128 {
using namespace regfft;

constexpr int LL = 128, LH = 65, YR = 72, NT = 256, MAXNP = 8;
constexpr uint32_t YBYTES = LL * YR * 8;  // one observation's staged spectrum, 73,728 B

// dynamic shared memory layout (bytes)
constexpr int WSP = 130;                      // transpose-buffer row stride (float2), = 2 (mod 16)
constexpr int OFF_W = 0;                      // float2 transpose buffer, 128 rows of WSP (+ gaps, wofs)
constexpr int OFF_Y = OFF_W + (LL * WSP + 16) * 8;  // float2 [128][72]  Yhat_i
constexpr int OFF_PAR = OFF_Y + (int)YBYTES;  // float [2L + KK] logit bias (log2 units), L <= 512
constexpr int OFF_ZC = OFF_PAR + 4224;        // float2 [2][128]  Z columns 0 and 64 (V extra)
constexpr int OFF_YC = OFF_ZC + 2048;         // float2 [2][128]  Yhat columns 0 and 64
constexpr int OFF_RED = OFF_YC + 2048;        // float2 [16]      block reductions
constexpr int OFF_XCH = OFF_RED + 128;        // float4 [2][MAXNP] cluster softmax exchange
constexpr int OFF_LRP = OFF_XCH + 32 * MAXNP;    // float2 [2][65] lr2 table per (half, element)
constexpr int OFF_MBAR = OFF_LRP + 8 * 2 * 65 + 16;
constexpr int OFF_TSLOT = OFF_MBAR + 8;
constexpr int OFF_MBAR2 = OFF_TSLOT + 8;      // OVL: the CTA softmax summary barrier (one arrival per warp)
constexpr int SMEM = OFF_MBAR2 + 8;
// OVL: the CTA softmax reduction is split around the pass-2 (M-row) transform — each warp publishes its
// (s, m, z) summary with an mbarrier arrive, transforms its rows of weights relative to its own reference,
// then waits, combines, publishes the pair's (g_q, z_q) to the cluster and scales the transformed rows (the
// transform is linear), instead of idling at a CTA barrier before the transform.  SRMRA_FFT128_NO_OVL builds
// the previous form for A/B.
#ifdef SRMRA_FFT128_NO_OVL
constexpr bool OVL = false;
#else
constexpr bool OVL = true;
#endif

// element (r, c) of the transpose buffer: rows 32 apart and the two parities of a column land in
// different 8-byte bank groups for both row-wise and column-wise thread-pair access
// Element (r, c) lives at r WSP + c + 8 (bit 5 of r) + 8 (bit 6 of r): every thread's four access patterns are
// a thread-constant base plus compile-time offsets (no per-element address arithmetic, unlike an XOR swizzle),
// rows never overlap (the bit-6 gap after row 63), and the accesses are conflict-free — row passes (row l,
// columns 2m + h): bank pair 2 l + h + const over 8 rows x 2 halves; column passes (rows 32 h + j (+ 64),
// column l): l + 8 h + const
__device__ __forceinline__ int wofs(int r, int c) { return r * WSP + c + (((r >> 5) & 1) << 3) + ((r >> 6) << 3); }

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float2 cmul_conj(float2 a, float2 b) {  // a * conj(b)
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
// a * conj(bh + bl) with the small product first (one rounding at the size of the result)
__device__ __forceinline__ float2 cmul_conj_acc(float2 a, float2 bh, float2 bl) {
    const float lx = fmaf(a.x, bl.x, a.y * bl.y), ly = fmaf(a.y, bl.x, -a.x * bl.y);
    return make_float2(fmaf(a.x, bh.x, fmaf(a.y, bh.y, lx)), fmaf(a.y, bh.x, fmaf(-a.x, bh.y, ly)));
}
// the float64 log2 maximum g_q a cluster peer stored in the (lo, hi, z, -) slot of its exchange float4
__device__ __forceinline__ double xch_g(float4 e) {
    return __longlong_as_double((long long)(((unsigned long long)__float_as_uint(e.y) << 32) | __float_as_uint(e.x)));
}
__device__ __forceinline__ float2 shfl_pair(float2 v) {
    return make_float2(__shfl_xor_sync(0xffffffffu, v.x, 1), __shfl_xor_sync(0xffffffffu, v.y, 1));
}

// ---------------------------------------------------------------- cluster / bulk copy / TMEM
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_cluster_f4(uint32_t local, uint32_t rank, float4 v) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
    asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(remote), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}
// ---------------------------------------------------------------- 128-point FFT over a thread pair
// w = exp(SIGN 2 pi i / 128).  DIT: in v[m] = x[2m + h]; 64-point FFT F_h; G_1[k] = w^k F_1[k];
// X[k] = G_0[k] + G_1[k], X[k + 64] = G_0[k] - G_1[k].  Thread h keeps k in [32h, 32h + 32).
// out v[j] = X[32h + j], v[32 + j] = X[64 + 32h + j].
template <int SIGN, int J>
__device__ __forceinline__ void dit_x1(float2 (&v)[64], bool hb, float sh) {
    constexpr float c0 = (float)cos2pi(J, 128), s0 = (float)(SIGN * sin2pi(J, 128));
    constexpr float c1 = (float)cos2pi(J + 32, 128), s1 = (float)(SIGN * sin2pi(J + 32, 128));
    float2 a = v[J], b = v[J + 32];
#ifdef SRMRA_FFT128_X_SCALAR
    if (hb) {
        a = make_float2(fmaf(a.x, c0, -a.y * s0), fmaf(a.x, s0, a.y * c0));
        b = make_float2(fmaf(b.x, c1, -b.y * s1), fmaf(b.x, s1, b.y * c1));
    }
    const float2 own = hb ? b : a, snd = hb ? a : b;
    const float2 rcv = shfl_pair(snd);
    v[J] = make_float2(own.x + rcv.x, own.y + rcv.y);
    v[J + 32] = make_float2(sh * (own.x - rcv.x), sh * (own.y - rcv.y));
#else
    // packed: a w = c a + s (i a) with scalar immediates and (-a.y, a.x) a free operand modifier (pair first)
    if (hb) {
        a = px::fma(make_float2(-a.y, a.x), px::bc(s0), px::mul(a, px::bc(c0)));
        b = px::fma(make_float2(-b.y, b.x), px::bc(s1), px::mul(b, px::bc(c1)));
    }
    const float2 own = hb ? b : a, snd = hb ? a : b;
    const float2 rcv = shfl_pair(snd);
    v[J] = px::add(own, rcv);
    v[J + 32] = px::mul(px::sub(own, rcv), px::bc(sh));
#endif
}
template <int SIGN, int... Js>
__device__ __forceinline__ void dit_xall(float2 (&v)[64], bool hb, float sh, std::integer_sequence<int, Js...>) {
    (dit_x1<SIGN, Js>(v, hb, sh), ...);
}
// DIF: in v[j] = x[32h + j], v[32 + j] = x[64 + 32h + j]; a[n] = x[n] + x[n+64],
// b[n] = (x[n] - x[n+64]) w^n; thread 0 transforms a (X[2k]), thread 1 transforms b (X[2k+1]).
// out v[k] = X[2k + h].
template <int SIGN, int J>
__device__ __forceinline__ void dif_x1(float2 (&v)[64], bool hb) {
    constexpr float c = (float)cos2pi(J, 128), s = (float)(SIGN * sin2pi(J, 128));
    const float2 x0 = v[J], x1 = v[J + 32];
#ifdef SRMRA_FFT128_X_SCALAR
    const float2 a = make_float2(x0.x + x1.x, x0.y + x1.y);
    const float2 d = make_float2(x0.x - x1.x, x0.y - x1.y);
    float2 b = make_float2(fmaf(d.x, c, -d.y * s), fmaf(d.x, s, d.y * c));
#else
    const float2 a = px::add(x0, x1);
    const float2 d = px::sub(x0, x1);
    float2 b = px::fma(make_float2(-d.y, d.x), px::bc(s), px::mul(d, px::bc(c)));
#endif
    if (hb) b = SIGN > 0 ? make_float2(-b.y, b.x) : make_float2(b.y, -b.x);  // w^32 = SIGN i
    const float2 own = hb ? b : a, snd = hb ? a : b;
    const float2 rcv = shfl_pair(snd);
    v[J] = hb ? rcv : own;
    v[J + 32] = hb ? own : rcv;
}
template <int SIGN, int... Js>
__device__ __forceinline__ void dif_xall(float2 (&v)[64], bool hb, std::integer_sequence<int, Js...>) {
    (dif_x1<SIGN, Js>(v, hb), ...);
}
// ---------------------------------------------------------------- block reductions (8 warps)
__device__ __forceinline__ float cta_max(float v, float2* red, int lane, int warp) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[warp].x = v;
    __syncthreads();
    float r = red[0].x;
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) r = fmaxf(r, red[w].x);
    return r;
}
__device__ __forceinline__ void ms_combine(float& m, float& z, float m2, float z2) {
    const float M = fmaxf(m, m2);
    if (M == -INFINITY) return;
    z = z * ex2(m - M) + z2 * ex2(m2 - M);
    m = M;
}
// (s, m, z): log2 maximum s c2 + m and scaled sum z of a set of unnormalised weights; sets with different
// score references s combine through (s - s') c2 + (m - m') (see k_fft.cu)
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
__device__ __forceinline__ void smz_warp(float& s, float& m, float& z, float c2) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float s2 = __shfl_xor_sync(0xffffffffu, s, o), m2 = __shfl_xor_sync(0xffffffffu, m, o),
                    z2 = __shfl_xor_sync(0xffffffffu, z, o);
        smz_combine(s, m, z, s2, m2, z2, c2);
    }
}
__device__ __forceinline__ void cta_smz(float& s, float& m, float& z, float c2, float4* red4, int lane, int warp) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float s2 = __shfl_xor_sync(0xffffffffu, s, o), m2 = __shfl_xor_sync(0xffffffffu, m, o),
                    z2 = __shfl_xor_sync(0xffffffffu, z, o);
        smz_combine(s, m, z, s2, m2, z2, c2);
    }
    if (lane == 0) red4[warp] = make_float4(s, m, z, 0.f);
    __syncthreads();
    float S = red4[0].x, Mx = red4[0].y, Z = red4[0].z;
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) smz_combine(S, Mx, Z, red4[w].x, red4[w].y, red4[w].z, c2);
    s = S;
    m = Mx;
    z = Z;
}
__device__ __forceinline__ void cta_ms(float& m, float& z, float2* red, int lane, int warp) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o), z2 = __shfl_xor_sync(0xffffffffu, z, o);
        ms_combine(m, z, m2, z2);
    }
    if (lane == 0) red[8 + warp] = make_float2(m, z);
    __syncthreads();
    float M = red[8].x, Z = red[8].y;
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) ms_combine(M, Z, red[8 + w].x, red[8 + w].y);
    m = M;
    z = Z;
}

struct Em128Args {
    const float2* yhat;   // [n][128][72] rfft2(y_i), float32
    const double* ynorm;  // [n]
    const double* ysum;   // [n] sum_n y_i[n] (the DC bin Yhat_i[0][0], float64)
    const float4* xhat;   // [2 (hi | lo)][NP][128][65] pair-interleaved (Xhat_2q, Xhat_2q+1) / L_low^2
    const float2* coef;   // COEF: [2 (hi | lo)][NP][128 k1][128 k2] E-step product coefficients (A, B) (k_fft128_coef)
    const float* par32;   // log2 units: lr1[L] | lr2[L] | beta[KK]
    const double* par64;  // E[KK] | (unused) | xm[KK] (mean of x_r)
    int64_t n;
    int L, K, KK, NP, PB;
    float c2;             // log2(e) / sigma^2
    double c2d, inv_2s2;
    float2* part;         // [clusters][PB] per-cluster partials (layout of k_fft.cu part_bins)
    double* llpart;       // [clusters]
    double* llobs;        // [n]
    const int* run;       // srmra_run stop flag ([0])
    unsigned long long* emt;  // [cap][2] first-CTA start / last-CTA end of this launch (globaltimer), slot *iter
    const int* iter;          // device iteration counter (slot index)
    int emt_cap;
};

// E-step product coefficients (COEF variant): for column k2 of pair q and row k1 the conjugated packed product
// v = conj(Yhat conj(Xhat_a) + i Yhat conj(Xhat_b)) of pass 0 is, with the true spectrum values Y (k2 >= 65: the
// conjugate of the stored mirror),  v = Y.x (A, B) + Y.y (B, -A),  A = Xa.x + Xb.y, B = Xa.y - Xb.x  (k_fft.cu XS = 2
// stores the same as four numbers (A, B, B, -A) / (A, B, -B, A)).  Two numbers per (k1, k2), formed in float64 from
// Xhat = hi + lo and stored as float32 hi + lo planes: 16 B per element where the four-number form streamed 32 B
// from L2 into pass 0 (whose loads were the kernel's largest latency stall); the kernel forms
// Y.y (B, -A) = (-Y.y) (-B, A) with (-B, A) a free FFMA2 operand modifier and -Y.y (conjugation of a mirrored
// stored value included) one FMUL.  (hi and lo interleaved as one float4 per element — one 16-B load instead of two
// 8-B loads — measured slower: 19.63 vs 19.17 ms.)
__global__ void k_fft128_coef(const float4* __restrict__ xhat, int NP, float2* __restrict__ coef) {
    const int total = NP * LL * LL;
    const float4* xlo = xhat + (size_t)NP * LL * LH;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
        const int q = k / (LL * LL), rem = k - q * LL * LL, k1 = rem / LL, k2 = rem - k1 * LL;
        const bool fl = k2 >= LH;
        const int o = q * LL * LH + (fl ? ((LL - k1) & (LL - 1)) : k1) * LH + (fl ? LL - k2 : k2);
        const float4 h = xhat[o], l = xlo[o];
        const double ax = (double)h.x + l.x, ay = (double)h.y + l.y, bx = (double)h.z + l.z, by = (double)h.w + l.w;
        // true values of a mirrored column: Xa = conj(stored), Xb = conj(stored)
        const double A = fl ? ax - by : ax + by, B = fl ? -ay - bx : ay - bx;
        const float2 hi = make_float2((float)A, (float)B);
        coef[k] = hi;
#ifndef SRMRA_FFT128_LO_F32
        // lo plane as bfloat16 pairs (round to nearest): |lo| <= 2^-24 |A|, kept to 2^-9 of itself, i.e. the
        // coefficients to ~2^-33 instead of float32's 2^-24 (the systematic error of DESIGN 6.5 scales with it)
        const unsigned lo_a = __float_as_uint((float)(A - hi.x)), lo_b = __float_as_uint((float)(B - hi.y));
        const unsigned ra = (lo_a + 0x7fffu + ((lo_a >> 16) & 1u)) >> 16, rb = (lo_b + 0x7fffu + ((lo_b >> 16) & 1u)) >> 16;
        reinterpret_cast<unsigned*>(coef + total)[k] = (rb << 16) | (ra & 0xffffu);
#else
        coef[(size_t)total + k] = make_float2((float)(A - hi.x), (float)(B - hi.y));
#endif
    }
}

template <bool PAIRS, bool COEF>
__global__ void __launch_bounds__(NT, 1) k_fft_em128(Em128Args a) {
    extern __shared__ __align__(1024) unsigned char sm[];
    float2* W = reinterpret_cast<float2*>(sm + OFF_W);
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
    float2* Ys = reinterpret_cast<float2*>(sm + OFF_Y);
    float* pars = reinterpret_cast<float*>(sm + OFF_PAR);
    float2* zc = reinterpret_cast<float2*>(sm + OFF_ZC);
    float2* yc = reinterpret_cast<float2*>(sm + OFF_YC);
    float2* red = reinterpret_cast<float2*>(sm + OFF_RED);
    float4* xch = reinterpret_cast<float4*>(sm + OFF_XCH);
    float2* lrp = reinterpret_cast<float2*>(sm + OFF_LRP);
    const uint32_t mbar = tc::smem_u32(sm + OFF_MBAR);
    const uint32_t mbar2 = tc::smem_u32(sm + OFF_MBAR2);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + OFF_TSLOT);

    const int t = threadIdx.x, h = t & 1, l = t >> 1, lane = t & 31, warp = t >> 5;
    const int NP = a.NP, K = a.K, L = a.L, KK = a.KK;
    const int q = NP > 1 ? (int)cluster_rank() : 0;
    const int cl = blockIdx.x / NP, ncl = gridDim.x / NP;
    const int n = (int)a.n;  // n_local is an int32 at the ABI
    const int ra = 2 * q, rb = 2 * q + 1;
    const bool has_b = PAIRS || rb < KK;

    for (int k = t; k < 2 * L; k += NT) pars[k] = __ldg(a.par32 + k);
    // class bias beta_r = (E_min - E_r) log2(e) / (2 sigma^2) from E_r (float64, written by the tail)
    double emin = __ldg(a.par64);
    for (int r = 1; r < KK; ++r) emin = fmin(emin, __ldg(a.par64 + r));
    for (int r = t; r < KK; r += NT) pars[2 * L + r] = (float)((emin - __ldg(a.par64 + r)) * a.inv_2s2 * 1.4426950408889634074);
    __shared__ double emin_cta;
    if (t == 0) emin_cta = emin;
    if (t == 0) {
        tc::mbar_init(mbar, 1);
        if (OVL) tc::mbar_init(mbar2, NT / 32);
        tc::fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc<512>(tslot);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    // TMEM: lane = t & 127 (warp w reaches lanes 32 (w & 3) ..); columns [256 (t >> 7), +128) hold the
    // Yhat values of this thread's line, the next 128 its accumulator line (U or V)
    const uint32_t trow = *tslot + ((uint32_t)(32 * (warp & 3)) << 16);
    const uint32_t ty = trow + (uint32_t)((t >> 7) * 256), tacc = ty + 128;
    {
        float z[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) z[j] = 0.f;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) tc::tmem_st16(tacc + 16 * ch, z);
        tc::tmem_wait_st();
    }
    int i = cl;
    if (t == 0 && i < n) {
        mbar_expect_tx(mbar, YBYTES);
        bulk_g2s(tc::smem_u32(Ys), a.yhat + (int64_t)i * (LL * YR), YBYTES, mbar);
    }

    // this thread's line: column l (passes 0, 3) / row l (passes 1, 2), half / parity h
    const int wrow = wofs(l, h);            // row passes: element (l, 2m + h) at wrow + 2m
    const int wcol = wofs(32 * h, l);       // column passes: (32 h + j, l) at wcol + j WSP, (64 + 32 h + j, l) + 64 WSP + 8
    const bool flip = l >= LH;             // column beyond the stored half spectrum (Hermitian mirror)
    const bool role_u = l < LH;            // accumulates U_q[., l]; otherwise V_q[., 128 - l]
    const bool both = (l == 0 || l == LL / 2);  // columns that also need V (added via zc / yc)
    const float su = role_u ? -1.f : 1.f;  // U: Yhat conj(Z); V: Yhat Z
    const int sk2 = flip ? LL - l : l;
    const float sg = flip ? -1.f : 1.f;
    const float4* XP = a.xhat + (size_t)q * LL * LH;
    const float4* XPL = XP + (size_t)NP * LL * LH;  // lo plane
    const float2* CH = a.coef + (size_t)q * LL * LL + l;            // COEF: hi coefficients of column l
    const float2* CL = CH + (size_t)NP * LL * LL;                   // lo (float32 pairs, SRMRA_FFT128_LO_F32)
    const unsigned* CLB = reinterpret_cast<const unsigned*>(a.coef + (size_t)NP * LL * LL) + (size_t)q * LL * LL + l;  // lo (bf16 pairs)
    const float ysg = flip ? 1.f : -1.f;                            // -Y.y = ysg * (stored Y).y
    const float* lr1 = pars;
    const float* lr2 = pars + L;
    const float* beta = pars + 2 * L;
    const int ra2 = ra % K, rb2 = rb % K;
    const float biasA = lr1[ra / K + K * l] + beta[ra];
    const float biasB = has_b ? lr1[rb / K + K * l] + beta[rb] : 0.f;
    // (the class means xm[ra], xm[rb] and E_min are re-read when needed: fewer live registers)

    // lr2 of (class ra, class rb) at the n2 of (half h, element j): n2 = 32h + j + 32 (j >= 32); rows
    // padded to 65 so the two halves of a warp read different banks
    for (int k = t; k < 2 * 65; k += NT) {
        const int hh = k / 65, j = k - hh * 65;
        const int n2 = 32 * hh + j + ((j >> 5) << 5);
        lrp[k] = j < 64 ? make_float2(lr2[ra2 + K * n2], has_b ? lr2[rb2 + K * n2] : 0.f) : make_float2(0.f, 0.f);
    }
    __syncthreads();
    float rsumA = 0.f, rsumB = 0.f;        // row sums of the posterior (row l, this half), classes ra / rb
    float2 cu = make_float2(0.f, 0.f);     // sum_i Z_{i,q}[0][l]
    float2 vex = make_float2(0.f, 0.f);    // V_q[t & 127][64 (t >> 7)] (columns 0 / 64)
    __shared__ double ll_acc;  // t == 0 of the q == 0 CTA accumulates the observations' log-likelihood terms
    if (t == 0) ll_acc = 0.0;
    uint32_t phase = 0, phase2 = 0;
    int it = 0;
    auto vex_update = [&]() {
        const int col = t >> 7, k1 = t & (LL - 1);
        const float2 yv = yc[col * LL + k1], z = zc[col * LL + ((LL - k1) & (LL - 1))];
        vex.x += yv.x * z.x - yv.y * z.y;
        vex.y += yv.y * z.x + yv.x * z.y;
    };

    // One forward 64-point FFT body serves all four passes (the kernel is otherwise instruction-fetch
    // bound): the two inverse passes use ifft(z) = conj(fft(conj z)) — the conjugation is folded into
    // the E-column input (conj Z) and the score read-out (S = conj of the E-row output).
    for (; i < n; i += ncl, ++it) {
        tc::mbar_wait(mbar, phase);
        phase ^= 1;
        float2 v[64];
        float za = 0.f, zb = 0.f, mt = -INFINITY, mall = 0.f, zall = 1.f;
        double gq = 0.0;         // this pair's log2 maximum (pass 1 -> pass 3)
        float zq = 1.f, rpa = 0.f, rpb = 0.f;
        float row_s = 0.f, sref = 0.f;  // OVL: this row's score reference (pass 1 -> pass 2); the CTA's
        // the four passes as four code bodies (with the linear transpose layout: c4 28.1 -> 23.5 ms; with the XOR
        // swizzle the unrolled variant was slower); SRMRA_FFT128_PASS_ROLLED builds one shared body for A/B
#ifdef SRMRA_FFT128_PASS_ROLLED
#pragma unroll 1
#else
#pragma unroll
#endif
        for (int pass = 0; pass < 4; ++pass) {
            if (pass == 0) {
                // all of this column's Yhat reads first (64 loads in flight), the TMEM stash, then the products
                // in place
#pragma unroll
                for (int m = 0; m < 64; ++m) {
                    const int k1 = 2 * m + h;
                    v[m] = Ys[(flip ? ((LL - k1) & (LL - 1)) : k1) * YR + sk2];
                }
#pragma unroll
                for (int ch = 0; ch < 8; ++ch) {
                    float ys[16];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        ys[2 * e] = v[ch * 8 + e].x;
                        ys[2 * e + 1] = v[ch * 8 + e].y;
                    }
                    tc::tmem_st16(ty + 16 * ch, ys);
                }
#pragma unroll
                for (int m = 0; m < 64; ++m) {
                    const int k1 = 2 * m + h;
                    const float2 yv = v[m];
#ifndef SRMRA_FFT128_LO_F32
                    const float2 ch = __ldg(CH + k1 * LL);
                    const unsigned lw = __ldg(CLB + k1 * LL);
                    const float2 cl = make_float2(__uint_as_float(lw << 16), __uint_as_float(lw & 0xffff0000u));
#else
                    const float2 ch = __ldg(CH + k1 * LL), cl = __ldg(CL + k1 * LL);
#endif
                    const float ny = ysg * yv.y;  // -Y.y of the true spectrum value
                    // v = Y.x (A, B) + (-Y.y) (-B, A), lo part first; the pair is the first operand (its swapped,
                    // half-negated form is then an operand modifier)
                    const float2 lo = px::fma(cl, px::bc(yv.x), px::mul(make_float2(-cl.y, cl.x), px::bc(ny)));
                    v[m] = px::fma(ch, px::bc(yv.x), px::fma(make_float2(-ch.y, ch.x), px::bc(ny), lo));
                    if (m == 0 && (l | h) == 0) v[m] = make_float2(0.f, 0.f);
                }
            } else if (pass == 1) {
#pragma unroll
                for (int m = 0; m < 64; ++m) v[m] = W[wrow + 2 * m];
            } else if (pass == 3) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    v[j] = W[wcol + j * WSP];
                    v[32 + j] = W[wcol + (64 + j) * WSP + 8];
                }
            }
            // pass 2: v holds the posterior row of the pair (forward transform along n2)
            if (pass >= 2) dif_xall<-1>(v, h != 0, std::make_integer_sequence<int, 32>{});
            fft_sr2<64, -1, false>(v);  // split radix, packed FP32x2 (pair-constant twiddles: fewer spills here)
            if (pass < 2) dit_xall<-1>(v, h != 0, h ? -1.f : 1.f, std::make_integer_sequence<int, 32>{});

            if (pass == 0) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    W[wcol + j * WSP] = v[j];
                    W[wcol + (64 + j) * WSP + 8] = v[32 + j];
                }
                __syncthreads();
                // Yhat_i has been consumed: stream the next observation's spectrum in behind passes 1-3
                if (t == 0 && i + ncl < n) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(mbar, YBYTES);
                    bulk_g2s(tc::smem_u32(Ys), a.yhat + (int64_t)(i + ncl) * (LL * YR), YBYTES, mbar);
                }
                if (it > 0) vex_update();  // columns 0 / 64 of the previous observation (zc, yc of its pass 3)
            } else if (pass == 1) {
                // S_a + i S_b = conj(v) at n2 = 32h + j (v[j]) and 64 + 32h + j (v[32 + j]), without the DC
                // terms D_c = ysum_i mean(x_c) (float64): S_c = . + D_c; scores are kept relative to D_a
                const double ysi = a.ysum[i];
                const double Da = ysi * __ldg(a.par64 + KK + 1 + ra);  // mean of x_ra
                const float dba = has_b ? (float)(ysi * __ldg(a.par64 + KK + 1 + rb) - Da) : 0.f;
                float lmax = -INFINITY;
#pragma unroll
                for (int j = 0; j < 64; ++j) {
                    v[j].y = dba - v[j].y;
                    lmax = fmaxf(lmax, has_b ? fmaxf(v[j].x, v[j].y) : v[j].x);
                }
                // OVL: the line's two threads share one reference (the pass-2 transform mixes their halves, so
                // the deferred row factor must be common to both)
                if constexpr (OVL) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, 1));
                const float sref_t = lmax;  // this thread's score reference (relative to D_a)
                // posterior (eq:weights_EM) in log2 units: v2 = (S - sref_t) log2e / sigma^2 + bias
                const float2 biasAB = make_float2(biasA, biasB);
#pragma unroll
                for (int j = 0; j < 64; ++j) {
                    float2 vab = px::fma(px::sub(v[j], px::bc(sref_t)), px::bc(a.c2), px::add(biasAB, lrp[h * 65 + j]));
                    if (!has_b) vab.y = -INFINITY;
                    v[j] = vab;
                    mt = fmaxf(mt, fmaxf(vab.x, vab.y));
                }
                if constexpr (OVL) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 1));
                const float mref = mt == -INFINITY ? 0.f : mt;
                float2 zab = make_float2(0.f, 0.f), zab1 = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < 64; ++j) {
                    const float2 dm = px::sub(v[j], px::bc(mref));
                    v[j] = make_float2(ex2(dm.x), has_b ? ex2(dm.y) : 0.f);
                    if (j & 1) zab1 = px::add(zab1, v[j]);
                    else zab = px::add(zab, v[j]);
                }
                za = zab.x + zab1.x;
                zb = zab.y + zab1.y;
                sref = sref_t;
                mall = mt;
                zall = za + zb;
                if constexpr (OVL) {
                    row_s = sref_t;
                    smz_warp(sref, mall, zall, a.c2);
                    if (lane == 0) {
                        reinterpret_cast<float4*>(red)[warp] = make_float4(sref, mall, zall, 0.f);
                        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar2) : "memory");
                    }
                } else {
                cta_smz(sref, mall, zall, a.c2, reinterpret_cast<float4*>(red), lane, warp);
                const double sref_d = Da + (double)sref;  // the pair's score reference, float64
                // log-sum-exp over all classes: combine the pairs of the cluster (log2 units, float64)
                // g_q = log2 of this pair's largest unnormalised weight: Sref c2 + m_q
                gq = mall == -INFINITY ? -INFINITY : sref_d * a.c2d + (double)mall;
                zq = zall;
                if (NP > 1) {  // publish (g_q, z_q); the wait is deferred to pass 3 (pass 2 overlaps the exchange)
                    const int slot = (it & 1) * MAXNP;
                    const unsigned long long gb = (unsigned long long)__double_as_longlong(gq);
                    if (t < NP)
                        st_cluster_f4(tc::smem_u32(&xch[slot + q]), (uint32_t)t,
                                      make_float4(__uint_as_float((unsigned)gb), __uint_as_float((unsigned)(gb >> 32)),
                                                  zall, 0.f));
                    // only warp 0 (t < NP) wrote remote data: the other warps arrive without a release fence
                    if (warp == 0) cluster_arrive();
                    else cluster_arrive_relaxed();
                }
                // weights relative to this pair's reference; the cluster factor 2^(g_q - G) / Z scales them after
                // the (linear) forward transforms, in pass 3
                const float floc = mt == -INFINITY ? 0.f : ex2(fmaf(sref_t - sref, a.c2, mt - mall));
                rpa = za * floc;
                rpb = zb * floc;
#pragma unroll
                for (int j = 0; j < 64; ++j) v[j] = make_float2(v[j].x * floc, v[j].y * floc);
                }  // !OVL
            } else if (pass == 2) {
                if constexpr (OVL) {
                    // every warp's summary is in red: the CTA (pair) reduction in the fixed warp order of cta_smz
                    tc::mbar_wait(mbar2, phase2);
                    phase2 ^= 1;
                    const float4* red4 = reinterpret_cast<const float4*>(red);
                    float S = red4[0].x, Mx = red4[0].y, Z = red4[0].z;
#pragma unroll
                    for (int w = 1; w < NT / 32; ++w) smz_combine(S, Mx, Z, red4[w].x, red4[w].y, red4[w].z, a.c2);
                    // the class-ra DC term of pass 1 re-read (not kept live across the transform)
                    const double sref_d = a.ysum[i] * __ldg(a.par64 + KK + 1 + ra) + (double)S;
                    gq = Mx == -INFINITY ? -INFINITY : sref_d * a.c2d + (double)Mx;
                    zq = Z;
                    if (NP > 1) {  // publish (g_q, z_q); the wait is in pass 3
                        const int slot = (it & 1) * MAXNP;
                        const unsigned long long gb = (unsigned long long)__double_as_longlong(gq);
                        if (t < NP)
                            st_cluster_f4(tc::smem_u32(&xch[slot + q]), (uint32_t)t,
                                          make_float4(__uint_as_float((unsigned)gb), __uint_as_float((unsigned)(gb >> 32)), Z,
                                                      0.f));
                        if (warp == 0) cluster_arrive();
                        else cluster_arrive_relaxed();
                    }
                    // weights relative to the pair's reference: the row factor on the transformed row
                    const float floc = mt == -INFINITY ? 0.f : ex2(fmaf(row_s - S, a.c2, mt - Mx));
                    rpa = za * floc;
                    rpb = zb * floc;
#pragma unroll
                    for (int j = 0; j < 64; ++j) v[j] = px::mul(v[j], px::bc(floc));
                }
                // each thread rewrites the row elements it read in pass 1
#pragma unroll
                for (int k = 0; k < 64; ++k) W[wrow + 2 * k] = v[k];
                __syncthreads();
            } else {
                // cluster factor of this pair: 2^(g_q - G) / Z (log-sum-exp over all classes, float64)
                double G = gq, Z = (double)zq;
                if (NP > 1) {
                    cluster_wait();
                    const int slot = (it & 1) * MAXNP;
                    // two passes over the exchange slots (no local array: it would live in local memory)
                    G = -INFINITY;
                    for (int r = 0; r < NP; ++r) G = fmax(G, xch_g(xch[slot + r]));
                    Z = 0.0;
                    for (int r = 0; r < NP; ++r) {
                        const float4 e = xch[slot + r];
                        const double gr = xch_g(e);
                        if (gr != -INFINITY) Z += (double)e.z * (double)ex2((float)(gr - G));
                    }
                }
                const float fcl = gq == -INFINITY ? 0.f : ex2((float)(gq - G)) / (float)Z;
                rsumA = fmaf(rpa, fcl, rsumA);
                rsumB = fmaf(rpb, fcl, rsumB);
                if (q == 0 && t == 0) {
                    const double lse = 0.69314718055994530942 * (G + (double)log2f((float)Z)) -
                                       (emin_cta + a.ynorm[i]) * a.inv_2s2;
                    ll_acc += lse;
                    if (a.llobs) a.llobs[i] = lse;
                }
#pragma unroll
                for (int m = 0; m < 64; ++m) v[m] = px::mul(v[m], px::bc(fcl));
                // v[m] = Z_{i,q}[k1 = 2m + h][l]
                if (h == 0) {
                    cu.x += v[0].x;
                    cu.y += v[0].y;
                }
                // U_q[2m+h][l] += Yhat conj(Z) (l < 65);  V_q[-(2m+h)][128-l] += Yhat[-(2m+h)][128-l] Z[2m+h][l]
#pragma unroll
                for (int ch = 0; ch < 8; ++ch) {
                    float ys[16], ac[16];
                    tc::tmem_ld16x2(ty + 16 * ch, ys, tacc + 16 * ch, ac);
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int m = ch * 8 + e;
                        const float2 z = v[m];
                        const float zy = su * z.y;
                        {
                            const float2 yy = make_float2(ys[2 * e], ys[2 * e + 1]);
                            const float2 r = px::fma(make_float2(-yy.y, yy.x), px::bc(zy),
                                                     px::fma(yy, px::bc(z.x), make_float2(ac[2 * e], ac[2 * e + 1])));
                            ac[2 * e] = r.x;
                            ac[2 * e + 1] = r.y;
                        }
                        if (both) {
                            zc[(l >> 6) * LL + 2 * m + h] = z;
                            yc[(l >> 6) * LL + 2 * m + h] = make_float2(ys[2 * e], ys[2 * e + 1]);
                        }
                    }
                    tc::tmem_st16(tacc + 16 * ch, ac);
                }
                tc::tmem_wait_st();
            }
        }
    }
    __syncthreads();
    if (it > 0) vex_update();

    // ---- this cluster's partials: U / V of pair q, row sums of classes ra / rb, pair line CU
    float2* P = a.part + (size_t)cl * a.PB;
    float2* Uq = P + (size_t)(2 * q) * LL * LH;
    float2* Vq = Uq + (size_t)LL * LH;
#pragma unroll
    for (int ch = 0; ch < 8; ch += 2) {
        float ac0[16], ac1[16];
        tc::tmem_ld16x2(tacc + 16 * ch, ac0, tacc + 16 * ch + 16, ac1);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int m = ch * 8 + e;
            const float2 val = e < 8 ? make_float2(ac0[2 * e], ac0[2 * e + 1]) : make_float2(ac1[2 * e - 16], ac1[2 * e - 15]);
            if (role_u) Uq[(2 * m + h) * LH + l] = val;
            else Vq[((LL - 2 * m - h) & (LL - 1)) * LH + (LL - l)] = val;
        }
    }
    Vq[(t & (LL - 1)) * LH + (t >> 7) * (LL / 2)] = vex;
    float2* R = P + (size_t)2 * NP * LL * LH;  // [KK][LL]
    float2* CU = R + (size_t)KK * LL;          // [NP][LL]
    const float rA = rsumA + __shfl_xor_sync(0xffffffffu, rsumA, 1);
    const float rB = rsumB + __shfl_xor_sync(0xffffffffu, rsumB, 1);
    if (h == 0) {
        R[ra * LL + l] = make_float2(rA, 0.f);
        if (has_b) R[rb * LL + l] = make_float2(rB, 0.f);
        CU[q * LL + l] = cu;
    }
    if (q == 0 && t == 0) a.llpart[cl] = ll_acc;
    tc::fence_before();
    __syncthreads();
    if (NP > 1) cluster_sync_all();  // no peer still writes into this CTA's exchange slots
    if (warp == 0) tc::tmem_dealloc<512>(*tslot);
    // the last CTA to finish marks the launch's end
    __syncthreads();
    if (threadIdx.x == 0 && emt_slot >= 0 && emt_slot < a.emt_cap) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        atomicMax(a.emt + 2 * emt_slot + 1, t1);
    }
}


}  // namespace fft128

using namespace fft128;

static cudaLaunchConfig_t em128_config(const srmra_ctx* c, cudaLaunchAttribute* attr, int clusters) {
    const int NP = (c->KK + 1) / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(clusters * NP));
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = c->stream;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = NP;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

bool fft128_supported(int K) { return K >= 1 && 2 * MAXNP >= K * K; }

static bool coef_mode() {  // SRMRA_FFT128_COEF=0: the compensated complex products (A/B)
    static const bool on = [] {
        const char* e = getenv("SRMRA_FFT128_COEF");
        return !(e && atoi(e) == 0);
    }();
    return on;
}
static auto em128_kernel(int KK) {
    if (coef_mode()) return KK % 2 == 0 ? k_fft_em128<true, true> : k_fft_em128<false, true>;
    return KK % 2 == 0 ? k_fft_em128<true, false> : k_fft_em128<false, false>;
}
size_t fft128_coef_float4(int KK) { return (size_t)((KK + 1) / 2) * LL * LL; }  // [2][NP][LL][LL] float2

cudaError_t fft128_plan(srmra_ctx* c) {
    auto kern = em128_kernel(c->KK);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // = the tail's
    if (e != cudaSuccess) return e;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = em128_config(c, attr, 1);
    int max_clusters = 0;
    e = cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg);
    if (e != cudaSuccess) return e;
    if (max_clusters < 1) return cudaErrorInvalidConfiguration;
    int64_t clusters = max_clusters;
    if (clusters > c->n_local) clusters = c->n_local;
    if (c->opt.grid_cap > 0 && clusters > c->opt.grid_cap) clusters = c->opt.grid_cap;  // test hook: several obs per cluster
    if (clusters < 1) clusters = 1;
    c->fft_grid = (int)clusters;  // partial slots (one per cluster)
    c->fft_groups = (c->KK + 1) / 2;
    c->fft_threads = NT;
    c->fft_smem = SMEM;
    c->fft_xs = 0;
    return cudaSuccess;
}

cudaError_t launch_fft_em128(srmra_ctx* c) {
    Em128Args a;
    const int64_t off = c->em_n >= 0 ? c->em_off : 0;  // srmra_load_iterate: one observation range
    a.yhat = c->d_yhat + off * (LL * YR);
    a.ynorm = c->d_ynorm + off;
    a.ysum = c->d_ysum + off;
    a.xhat = reinterpret_cast<const float4*>(c->d_xhat);
    a.coef = reinterpret_cast<const float2*>(c->d_xcoef);
    a.par32 = c->par.f32;
    a.par64 = c->par.f64;
    a.n = c->em_n >= 0 ? c->em_n : c->n_local;
    a.L = c->L;
    a.K = c->K;
    a.KK = c->KK;
    a.NP = (c->KK + 1) / 2;
    if (coef_mode()) {
        k_fft128_coef<<<2 * c->num_sms, 256, 0, c->stream>>>(a.xhat, a.NP, reinterpret_cast<float2*>(c->d_xcoef));
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    a.PB = fft_partial_bins(c->KK, LL);
    a.c2 = (float)(1.4426950408889634074 * c->inv_s2);
    a.c2d = 1.4426950408889634074 * c->inv_s2;
    a.inv_2s2 = c->inv_2s2;
    a.part = c->em_n >= 0 ? c->em_part : c->d_part;
    a.llpart = c->em_n >= 0 ? c->em_llpart : c->d_llpart;
    a.llobs = c->d_llobs ? c->d_llobs + off : nullptr;
    a.run = c->d_run;
    a.emt = c->d_emt;
    a.iter = c->d_iter;
    a.emt_cap = c->opt.trace_cap;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = em128_config(c, attr, c->fft_grid);
    return cudaLaunchKernelEx(&cfg, em128_kernel(c->KK), a);
}

}  // namespace srmra
