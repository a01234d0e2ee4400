// regfft.cuh — register-resident FFTs with compile-time twiddles (radix 2, radix 4 and split radix; the
// E/M kernels use split radix, the fewest twiddle products), shared by the FFT-path
// E/M kernels (k_fft.cu: one thread per line, L_low <= 64; k_fft128.cu: a thread pair per line,
// L_low = 128).  fft<N, SIGN>: in place, natural order in and out, unnormalised,
// X[k] = sum_n x[n] exp(SIGN 2 pi i n k / N)  (SIGN = -1 forward, +1 inverse).
#pragma once
#include <cuda_runtime.h>

#include <utility>

namespace srmra {
namespace regfft {

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


// ------------------------------------------------------------------ register FFT (radix 4)
// Two radix-2 DIT stages (lengths 2H and 4H) merged into one radix-4 butterfly per quad (B + j, + H, + 2H,
// + 3H): with b~ = W_4H^{2j} b, c~ = W_4H^j c, d~ = W_4H^{3j} d the outputs are a +- b~ +- (c~ + d~) and
// a -+ b~ ... (-+ i)(c~ - d~) — 3 twiddle products per quad instead of 4, the same 8 complex additions.
template <int N, int SIGN, int TK>
__device__ __forceinline__ float2 twmul(float2 b) {
    constexpr int T = ((TK % N) + N) % N;
    if constexpr (T == 0) {
        return b;
    } else if constexpr (2 * T == N) {
        return make_float2(-b.x, -b.y);
    } else if constexpr (4 * T == N) {
        if constexpr (SIGN > 0) return make_float2(-b.y, b.x);  // * (+i)
        else return make_float2(b.y, -b.x);                     // * (-i)
    } else if constexpr (4 * T == 3 * N) {
        if constexpr (SIGN > 0) return make_float2(b.y, -b.x);  // * (-i)
        else return make_float2(-b.y, b.x);                     // * (+i)
    } else {
        constexpr float c = (float)cos2pi(T, N);
        constexpr float s = (float)(SIGN * sin2pi(T, N));
        return make_float2(fmaf(b.x, c, -b.y * s), fmaf(b.x, s, b.y * c));
    }
}
template <int N, int SIGN, int H, int B, int J>
__device__ __forceinline__ void bfly4(float2* t) {
    constexpr int S = N / (4 * H);  // W_4H^k = W_N^{k S}
    const float2 a = t[B + J];
    const float2 bt = twmul<N, SIGN, 2 * J * S>(t[B + J + H]);
    const float2 ct = twmul<N, SIGN, J * S>(t[B + J + 2 * H]);
    const float2 dt = twmul<N, SIGN, 3 * J * S>(t[B + J + 3 * H]);
    const float2 p = make_float2(a.x + bt.x, a.y + bt.y), m = make_float2(a.x - bt.x, a.y - bt.y);
    const float2 cp = make_float2(ct.x + dt.x, ct.y + dt.y), cm = make_float2(ct.x - dt.x, ct.y - dt.y);
    // the (b', d') pair's twiddle W_4H^{j+H} = W_4H^j W_4H^H, W_4H^H = W_N^{N/4} = -+i:
    // out[j + H] = m + W_N^{N/4} (c~ - d~), out[j + 3H] = m - W_N^{N/4} (c~ - d~)
    const float2 q = twmul<N, SIGN, N / 4>(cm);
    t[B + J] = make_float2(p.x + cp.x, p.y + cp.y);
    t[B + J + 2 * H] = make_float2(p.x - cp.x, p.y - cp.y);
    t[B + J + H] = make_float2(m.x + q.x, m.y + q.y);
    t[B + J + 3 * H] = make_float2(m.x - q.x, m.y - q.y);
}
template <int N, int SIGN, int H, int B, int... Js>
__device__ __forceinline__ void bfly4_block(float2* t, std::integer_sequence<int, Js...>) {
    (bfly4<N, SIGN, H, B, Js>(t), ...);
}
template <int N, int SIGN, int H, int... Bs>
__device__ __forceinline__ void fft_stage4(float2* t, std::integer_sequence<int, Bs...>) {
    (bfly4_block<N, SIGN, H, Bs * 4 * H>(t, std::make_integer_sequence<int, H>{}), ...);
}
// stages: radix-2 (length 2) when log2 N is odd, then radix-4 stages of quarter sizes H = 2^k
template <int N, int SIGN, int H>
__device__ __forceinline__ void fft4_stages(float2* t) {
    if constexpr (4 * H <= N) {
        fft_stage4<N, SIGN, H>(t, std::make_integer_sequence<int, N / (4 * H)>{});
        fft4_stages<N, SIGN, 4 * H>(t);
    }
}
template <int N, int SIGN>
__device__ __forceinline__ void fft_r4(float2 (&v)[N]) {
    float2 t[N];
    bitrev_copy<N>(t, v, std::make_integer_sequence<int, N>{});
    if constexpr (ilog2(N) % 2 == 1) {
        fft_stage<N, SIGN, 2>(t, std::make_integer_sequence<int, N / 2>{});
        fft4_stages<N, SIGN, 2>(t);
    } else {
        fft4_stages<N, SIGN, 1>(t);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = t[i];
}

// ------------------------------------------------------------------ register FFT (split radix)
// X = DFT_N of x[OFF + ST n]: U = DFT_{N/2} of the even samples, Z / Z' = DFT_{N/4} of the samples 4n + 1 /
// 4n + 3;  X[k] = U[k] + (W^k Z[k] + W^{3k} Z'[k]),  X[k + N/2] = U[k] - (...),
// X[k + N/4] = U[k + N/4] + W^{N/4} (W^k Z[k] - W^{3k} Z'[k]),  X[k + 3N/4] = U[k + N/4] - W^{N/4} (...).
template <int N, int SIGN, int OFF, int ST>
__device__ __forceinline__ void sr_rec(const float2* x, float2* X);
template <int N, int SIGN, int K>
__device__ __forceinline__ void sr_comb(const float2* U, const float2* Z, const float2* Zp, float2* X) {
    const float2 a = twmul<N, SIGN, K>(Z[K]), b = twmul<N, SIGN, 3 * K>(Zp[K]);
    const float2 sm = make_float2(a.x + b.x, a.y + b.y);
    const float2 id = twmul<N, SIGN, N / 4>(make_float2(a.x - b.x, a.y - b.y));
    const float2 u0 = U[K], u1 = U[K + N / 4];
    X[K] = make_float2(u0.x + sm.x, u0.y + sm.y);
    X[K + N / 2] = make_float2(u0.x - sm.x, u0.y - sm.y);
    X[K + N / 4] = make_float2(u1.x + id.x, u1.y + id.y);
    X[K + 3 * N / 4] = make_float2(u1.x - id.x, u1.y - id.y);
}
template <int N, int SIGN, int... Ks>
__device__ __forceinline__ void sr_combine(const float2* U, const float2* Z, const float2* Zp, float2* X,
                                           std::integer_sequence<int, Ks...>) {
    (sr_comb<N, SIGN, Ks>(U, Z, Zp, X), ...);
}
template <int N, int SIGN, int OFF, int ST>
__device__ __forceinline__ void sr_rec(const float2* x, float2* X) {
    if constexpr (N == 1) {
        X[0] = x[OFF];
    } else if constexpr (N == 2) {
        const float2 a = x[OFF], b = x[OFF + ST];
        X[0] = make_float2(a.x + b.x, a.y + b.y);
        X[1] = make_float2(a.x - b.x, a.y - b.y);
    } else {
        float2 U[N / 2], Z[N / 4], Zp[N / 4];
        sr_rec<N / 2, SIGN, OFF, 2 * ST>(x, U);
        sr_rec<N / 4, SIGN, OFF + ST, 4 * ST>(x, Z);
        sr_rec<N / 4, SIGN, OFF + 3 * ST, 4 * ST>(x, Zp);
        sr_combine<N, SIGN>(U, Z, Zp, X, std::make_integer_sequence<int, N / 4>{});
    }
}
template <int N, int SIGN>
__device__ __forceinline__ void fft_sr(float2 (&v)[N]) {
    float2 X[N];
    sr_rec<N, SIGN, 0, 1>(v, X);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = X[i];
}

// ------------------------------------------------------------------ packed FP32x2 arithmetic (sm_100)
// add / sub / mul / fma .rn.f32x2 on a float2 held in a register pair: one issue slot for both halves
// (FADD2 / FMUL2 / FFMA2; the pipe throughput per FP32 operation is unchanged, tools/fp32x2_peak.cu), so an
// issue-bound kernel sheds half of its complex-arithmetic instructions.  Scalars broadcast into a pair
// (bc) become ".F32" operands in SASS, and the halves of a pair can be swapped as an operand.
namespace px {
__device__ __forceinline__ unsigned long long u(float2 v) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
    return r;
}
__device__ __forceinline__ float2 f(unsigned long long r) {
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ float2 add(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(u(a)), "l"(u(b)));
    return f(d);
}
__device__ __forceinline__ float2 sub(float2 a, float2 b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(u(a)), "l"(u(b)));
    return f(d);
}
__device__ __forceinline__ float2 mul(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(u(a)), "l"(u(b)));
    return f(d);
}
__device__ __forceinline__ float2 fma(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(u(a)), "l"(u(b)), "l"(u(c)));
    return f(d);
}
__device__ __forceinline__ float2 bc(float x) { return make_float2(x, x); }
}  // namespace px

// b * W_N^TK (SIGN convention of twmul) in packed form; +-i and -1 as swaps / signs.  IMM: b w = c b + s (i b),
// both constants scalar immediates of FMUL2 / FFMA2 and i b = (-b.y, b.x) a free operand modifier (swapped
// halves, one negated: .F32x2.LO_HI.NP).  !IMM: bx (c, s) + by (-s, c), whose constant pairs are moved into
// registers (UMOV / MOV) for every product — 232 fewer instructions per k_fft_em body with IMM, but at L_low = 128
// (255 registers) ptxas spills more with IMM and k_fft_em128 measured slower (23.00 vs 22.62 ms), so it keeps !IMM
template <int N, int SIGN, int TK, bool IMM>
__device__ __forceinline__ float2 twmul2(float2 b) {
    constexpr int T = ((TK % N) + N) % N;
    if constexpr (T == 0 || 2 * T == N || 4 * T == N || 4 * T == 3 * N) {
        return twmul<N, SIGN, TK>(b);  // trivial: sign flips and swaps fold into the consumer
    } else {
        constexpr float c = (float)cos2pi(T, N);
        constexpr float s = (float)(SIGN * sin2pi(T, N));
        if constexpr (IMM) return px::fma(make_float2(-b.y, b.x), px::bc(s), px::mul(b, px::bc(c)));
        else return px::fma(px::bc(b.y), make_float2(-s, c), px::mul(px::bc(b.x), make_float2(c, s)));
    }
}
template <int N, int SIGN, bool IMM, int K>
__device__ __forceinline__ void sr2_comb(const float2* U, const float2* Z, const float2* Zp, float2* X) {
    const float2 a = twmul2<N, SIGN, K, IMM>(Z[K]), b = twmul2<N, SIGN, 3 * K, IMM>(Zp[K]);
    const float2 sm = px::add(a, b);
    const float2 id = twmul<N, SIGN, N / 4>(px::sub(a, b));
    const float2 u0 = U[K], u1 = U[K + N / 4];
    X[K] = px::add(u0, sm);
    X[K + N / 2] = px::sub(u0, sm);
    X[K + N / 4] = px::add(u1, id);
    X[K + 3 * N / 4] = px::sub(u1, id);
}
template <int N, int SIGN, bool IMM, int... Ks>
__device__ __forceinline__ void sr2_combine(const float2* U, const float2* Z, const float2* Zp, float2* X,
                                            std::integer_sequence<int, Ks...>) {
    (sr2_comb<N, SIGN, IMM, Ks>(U, Z, Zp, X), ...);
}
template <int N, int SIGN, bool IMM, int OFF, int ST>
__device__ __forceinline__ void sr2_rec(const float2* x, float2* X) {
    if constexpr (N == 1) {
        X[0] = x[OFF];
    } else if constexpr (N == 2) {
        const float2 a = x[OFF], b = x[OFF + ST];
        X[0] = px::add(a, b);
        X[1] = px::sub(a, b);
    } else {
        float2 U[N / 2], Z[N / 4], Zp[N / 4];
        sr2_rec<N / 2, SIGN, IMM, OFF, 2 * ST>(x, U);
        sr2_rec<N / 4, SIGN, IMM, OFF + ST, 4 * ST>(x, Z);
        sr2_rec<N / 4, SIGN, IMM, OFF + 3 * ST, 4 * ST>(x, Zp);
        sr2_combine<N, SIGN, IMM>(U, Z, Zp, X, std::make_integer_sequence<int, N / 4>{});
    }
}
// split radix in packed FP32x2 arithmetic
template <int N, int SIGN, bool IMM = true>
__device__ __forceinline__ void fft_sr2(float2 (&v)[N]) {
    float2 X[N];
    sr2_rec<N, SIGN, IMM, 0, 1>(v, X);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = X[i];
}

}  // namespace regfft
}  // namespace srmra
