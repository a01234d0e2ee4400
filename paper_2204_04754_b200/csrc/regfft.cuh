// regfft.cuh — register-resident radix-2 FFTs with compile-time twiddles, shared by the FFT-path
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

}  // namespace regfft
}  // namespace srmra
