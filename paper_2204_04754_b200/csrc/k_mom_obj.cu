// k_mom_obj.cu — NEXT-2: the least-squares moment objective eq:LS_SR and its gradient,
// evaluated in the Fourier domain without forming C_x, plus Algorithm 1's driver
// (PAPER.md:359-374): L-BFGS steps on the host, the projection every F steps, the sigma schedule.
//
// Notation: L = L_high, Ll = L_low, u in Z_L^2, k in Z_Ll^2, ubar = u mod Ll; hats are 2-D DFTs with
// exp(-2 pi i u.p / L).  With v_s = P R_s x (Eq. (2)), decimation aliases the spectrum:
//     vtilde_s[k] = K^-2 sum_{m in Z_K^2} xhat[k + Ll m] w_L^{-(k + Ll m).s}, so with Mtilde = F M F^H,
//     Mtilde2[k, k'] = K^-4 sum_{m, m'} xhat[u] conj(xhat[u']) rhohat[u - u'] + sigma^2 Ll^2 delta_kk',
//     Mtilde1[k]     = K^-2 sum_m xhat[u] rhohat[u]                 (u = k + Ll m, u' = k' + Ll m'),
// and Parseval gives f = Ll^-4 sum |Etilde|^2 + lambda Ll^-2 sum |etilde|^2, Etilde = Mtilde2 - F M2hat F^H,
// etilde = Mtilde1 - F M1hat.  The gradient (derivation in DESIGN.md §6.9; the oracle's spatial form is
// pinned by finite differences):
//     df/dx[w]   = Re sum_u Ax[u] w_L^{-u.w},   Ax[u] = 4 L^-4 sum_{u'} conj(Etilde[ubar, ubar']) rhohat[u - u']
//                                                       conj(xhat[u']) + 2 lambda Ll^-2 K^-2 conj(etilde[ubar]) rhohat[u]
//     df/drho[s] = Re sum_v Gr[v] w_L^{+v.s},   Gr[v]  = 2 L^-4 sum_u Etilde[ubar, (u - v)bar] conj(xhat[u]) xhat[u - v]
//                                                       + 2 lambda Ll^-2 K^-2 etilde[vbar] conj(xhat[v])
// Three O(L^4) float64 kernels (E, A, G), a few O(L^3) DFT passes; the O(Ll^5) transform of the data
// moments runs once per srmra_mom_set_moments.
#include <math.h>

#include <algorithm>
#include <vector>

#include "srmra_internal.cuh"

namespace srmra {

struct MomState {
    int L = 0, Ll = 0, K = 0;
    double lambda = 0.0;
    double2* tw = nullptr;  // [L] exp(-2 pi i j / L)
    double2* t2 = nullptr;  // [Ll2][Ll2] F M2hat F^H - sigma^2 Ll^2 I
    double2* t1 = nullptr;  // [Ll2] F M1hat
    double2* et = nullptr;  // [Ll2][Ll2] Etilde
    double2* e1 = nullptr;  // [Ll2] etilde
    double2* xh = nullptr;  // [L2]
    double2* rh = nullptr;  // [2L] 1-D spectra of rho1 | rho2 (allocated [L2])
    double2* ax = nullptr;  // [L2]
    double2* gr = nullptr;  // [L2]
    double2* tmp = nullptr; // [L2] DFT scratch
    double* theta = nullptr;  // [L2 + 2L] x | rho1 | rho2
    double* out = nullptr;    // [1 + L2 + 2L + L2] f | grad x | grad rho1 | grad rho2 | grad rho (joint)
    double* fpart = nullptr;  // [2 Ll2] per-block |Etilde|^2 | |etilde|^2
    bool ready = false;
};

namespace momo {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a conj(b)
    return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 conj2(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

__device__ __forceinline__ double2 block_csum(double2 v, double* red) {
    v.x = block_sum(v.x, red);
    __syncthreads();
    v.y = block_sum(v.y, red);
    __syncthreads();
    return v;
}

__global__ void k_twiddle(double2* tw, int L) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < L; j += gridDim.x * blockDim.x) {
        double s, c;
        sincospi(-2.0 * (double)j / (double)L, &s, &c);
        tw[j] = make_double2(c, s);
    }
}

__global__ void k_real_to_c(const double* __restrict__ in, double2* __restrict__ out, int64_t n) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = make_double2(in[e], 0.0);
}

// symmetric part of a real [n][n] matrix, as complex (the objective uses M2hat through <E, E>; E symmetric)
__global__ void k_sym_to_c(const double* __restrict__ in, double2* __restrict__ out, int n) {
    const int64_t total = (int64_t)n * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int a = (int)(e / n), b = (int)(e - (int64_t)a * n);
        out[e] = make_double2(0.5 * (in[(int64_t)a * n + b] + in[(int64_t)b * n + a]), 0.0);
    }
}

// one DFT axis: out[o][k][i] = sum_j in[o][j][i] w^{sgn k j}, w = exp(-2 pi i / n) = tw[step], n step = L
__global__ void k_dft_axis(const double2* __restrict__ in, double2* __restrict__ out, int64_t outer, int n,
                           int64_t inner, int sgn, const double2* __restrict__ tw, int step) {
    const int64_t total = outer * n * inner;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = e / ((int64_t)n * inner), rem = e - o * n * inner;
        const int k = (int)(rem / inner);
        const int64_t i = rem - (int64_t)k * inner;
        const double2* src = in + o * n * inner + i;
        double2 acc = make_double2(0.0, 0.0);
        int idx = 0;  // (k j) mod n
        for (int j = 0; j < n; ++j) {
            double2 w = tw[idx * step];
            if (sgn > 0) w.y = -w.y;
            acc = cadd(acc, cmul(src[(int64_t)j * inner], w));
            idx += k;
            if (idx >= n) idx -= n;
        }
        out[e] = acc;
    }
}

// 2-D transforms of the [L][L] spectra: one block per line (row: line_stride L, elem_stride 1; column: 1, L),
// the line and the twiddles staged in shared memory
__global__ void k_dft_line(const double2* __restrict__ in, double2* __restrict__ out, int n, int64_t line_stride,
                           int64_t elem_stride, int sgn, const double2* __restrict__ tw, int step) {
    extern __shared__ double2 sl[];  // line [n] | twiddles [n]
    double2* tws = sl + n;
    const double2* src = in + (int64_t)blockIdx.x * line_stride;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        sl[j] = src[(int64_t)j * elem_stride];
        double2 w = tw[j * step];
        if (sgn > 0) w.y = -w.y;
        tws[j] = w;
    }
    __syncthreads();
    double2* dst = out + (int64_t)blockIdx.x * line_stride;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        double2 acc = make_double2(0.0, 0.0);
        int idx = 0;
        for (int j = 0; j < n; ++j) {
            acc = cadd(acc, cmul(sl[j], tws[idx]));
            idx += k;
            if (idx >= n) idx -= n;
        }
        dst[(int64_t)k * elem_stride] = acc;
    }
}

__global__ void k_sub_diag(double2* t2, int n, double v) {
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x) t2[(int64_t)a * n + a].x -= v;
}

// rhohat = rhohat1 (x) rhohat2 (D_rho = diag vec(rho1 rho2^T)): the kernels below take the two
// 1-D spectra rh[0 .. L) | rh[L .. 2L) and form rhohat[d1][d2] = rh1[d1] rh2[d2] on the fly
__global__ void k_rhohat(const double* __restrict__ r, int L, const double2* __restrict__ tw, double2* __restrict__ rh) {
    extern __shared__ double2 st[];  // twiddles [L] | rho_j [L] (as .x)
    const int j = blockIdx.x;        // rho1 | rho2
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        st[i] = tw[i];
        st[L + i].x = r[j * L + i];
    }
    __syncthreads();
    for (int u = threadIdx.x; u < L; u += blockDim.x) {
        double2 a = make_double2(0.0, 0.0);
        int idx = 0;
        for (int s = 0; s < L; ++s) {
            const double2 w = st[idx];
            const double v = st[L + s].x;
            a.x += v * w.x;
            a.y += v * w.y;
            idx += u;
            if (idx >= L) idx -= L;
        }
        rh[j * L + u] = a;
    }
}

constexpr int MC = 16;  // frequencies u = ubar + Ll m handled per pass (accumulators per thread)

// block-wide sum of n complex accumulators (blockDim = 256); results in out[0 .. n) of shared memory
__device__ __forceinline__ void block_csum_n(double2* acc, int n, double2* sred /*[8][MC]*/, double2* out) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int m = 0; m < n; ++m) {
        double2 v = acc[m];
        v.x = warp_sum(v.x);
        v.y = warp_sum(v.y);
        if (lane == 0) sred[w * MC + m] = v;
    }
    __syncthreads();
    if (threadIdx.x < n) {
        double2 t = make_double2(0.0, 0.0);
        for (int j = 0; j < 8; ++j) t = cadd(t, sred[j * MC + threadIdx.x]);
        out[threadIdx.x] = t;
    }
    __syncthreads();
}

// Etilde[k][k'] (one block per k, threads over k') and etilde[k]; |.|^2 partials per block.
//   sum_{m, m'} xhat[u] conj(xhat[u']) rh1[u1 - u1'] rh2[u2 - u2'], inner sum over m2 first.
// KT = K <= 4: u1 - u1' = k1 - k1' + Ll (m1 - m1') takes 2K - 1 values, so the prior factors are gathered
// once per k' and the K^4 sum is done as two K^3 contractions.
template <int KT>
__global__ void __launch_bounds__(256) k_mom_E(const double2* __restrict__ xh, const double2* __restrict__ rh,
                                               const double2* __restrict__ t2, const double2* __restrict__ t1, int L,
                                               int Ll, int K, double2* __restrict__ et, double2* __restrict__ e1,
                                               double* __restrict__ fpart) {
    extern __shared__ double2 sm[];  // rh1 [L] | rh2 [L] | xs [K^2]
    __shared__ double red[32];
    double2* r1s = sm;
    double2* r2s = sm + L;
    double2* xs = sm + 2 * L;
    const int Ll2 = Ll * Ll, KK = K * K;
    const int k = blockIdx.x, k1 = k / Ll, k2 = k - k1 * Ll;
    for (int j = threadIdx.x; j < 2 * L; j += blockDim.x) sm[j] = rh[j];
    for (int m = threadIdx.x; m < KK; m += blockDim.x) xs[m] = xh[(k1 + Ll * (m / K)) * L + k2 + Ll * (m % K)];
    __syncthreads();
    const double invK4 = 1.0 / ((double)KK * KK);
    double part = 0.0;
    for (int kp = threadIdx.x; kp < Ll2; kp += blockDim.x) {
        const int kp1 = kp / Ll, kp2 = kp - kp1 * Ll;
        double2 acc = make_double2(0.0, 0.0);
        if constexpr (KT > 0) {
            double2 A1[2 * KT - 1], A2[2 * KT - 1], B[KT][KT];
#pragma unroll
            for (int dl = 0; dl < 2 * KT - 1; ++dl) {
                int d1 = k1 - kp1 + Ll * (dl - (KT - 1)), d2 = k2 - kp2 + Ll * (dl - (KT - 1));
                d1 += d1 < 0 ? L : 0;
                d1 -= d1 >= L ? L : 0;
                d2 += d2 < 0 ? L : 0;
                d2 -= d2 >= L ? L : 0;
                A1[dl] = r1s[d1];
                A2[dl] = r2s[d2];
            }
#pragma unroll
            for (int m1 = 0; m1 < KT; ++m1)
#pragma unroll
                for (int mp2 = 0; mp2 < KT; ++mp2) {
                    double2 t = make_double2(0.0, 0.0);
#pragma unroll
                    for (int m2 = 0; m2 < KT; ++m2) t = cadd(t, cmul(xs[m1 * KT + m2], A2[m2 - mp2 + KT - 1]));
                    B[m1][mp2] = t;
                }
#pragma unroll
            for (int mp1 = 0; mp1 < KT; ++mp1)
#pragma unroll
                for (int mp2 = 0; mp2 < KT; ++mp2) {
                    double2 in = make_double2(0.0, 0.0);
#pragma unroll
                    for (int m1 = 0; m1 < KT; ++m1) in = cadd(in, cmul(A1[m1 - mp1 + KT - 1], B[m1][mp2]));
                    acc = cadd(acc, cmulc(in, xh[(kp1 + Ll * mp1) * L + kp2 + Ll * mp2]));
                }
        } else {
            for (int mp1 = 0; mp1 < K; ++mp1) {
                const int up1 = kp1 + Ll * mp1;
                for (int mp2 = 0; mp2 < K; ++mp2) {
                    const int up2 = kp2 + Ll * mp2;
                    double2 in = make_double2(0.0, 0.0);
                    for (int m1 = 0; m1 < K; ++m1) {
                        int d1 = k1 + Ll * m1 - up1;
                        d1 += d1 < 0 ? L : 0;
                        double2 row = make_double2(0.0, 0.0);
                        for (int m2 = 0; m2 < K; ++m2) {
                            int d2 = k2 + Ll * m2 - up2;
                            d2 += d2 < 0 ? L : 0;
                            row = cadd(row, cmul(xs[m1 * K + m2], r2s[d2]));
                        }
                        in = cadd(in, cmul(row, r1s[d1]));
                    }
                    acc = cadd(acc, cmulc(in, xh[up1 * L + up2]));
                }
            }
        }
        const double2 t = t2[(int64_t)k * Ll2 + kp];
        const double2 E = make_double2(acc.x * invK4 - t.x, acc.y * invK4 - t.y);
        et[(int64_t)k * Ll2 + kp] = E;
        part += E.x * E.x + E.y * E.y;
    }
    part = block_sum(part, red);
    if (threadIdx.x == 0) {
        fpart[k] = part;
        double2 m1 = make_double2(0.0, 0.0);
        for (int m = 0; m < KK; ++m)
            m1 = cadd(m1, cmul(xs[m], cmul(r1s[k1 + Ll * (m / K)], r2s[k2 + Ll * (m % K)])));
        const double2 e = make_double2(m1.x / KK - t1[k].x, m1.y / KK - t1[k].y);
        e1[k] = e;
        fpart[Ll2 + k] = e.x * e.x + e.y * e.y;
    }
}

// Ax[u] for the K^2 frequencies u = ubar + Ll m of one block: conj(row ubar of Etilde) and the 1-D prior
// spectra staged in shared memory; each term h = conj(Etilde[ubar, ubar']) conj(xhat[u']) is formed once,
// multiplied by the K values rh1[u1 - u1'] (m1) and then by the K values rh2[u2 - u2'] (m2) into the K^2
// accumulators.  KT = K for K <= 4 (fully unrolled); KT = 0: any K, MC frequencies per pass.
template <int KT>
__global__ void __launch_bounds__(256) k_mom_A(const double2* __restrict__ xh, const double2* __restrict__ rh,
                                               const double2* __restrict__ et, const double2* __restrict__ e1, int L,
                                               int Ll, int K, double c2, double c1, double2* __restrict__ ax) {
    extern __shared__ double2 sm[];  // erow [Ll2] | rh1 [L] | rh2 [L]
    __shared__ double2 sred[8 * MC], sout[MC];
    const int Ll2 = Ll * Ll, KK = K * K;
    double2* erow = sm;
    double2* r1s = sm + Ll2;
    double2* r2s = r1s + L;
    const int ub = blockIdx.x, ub1 = ub / Ll, ub2 = ub - ub1 * Ll;
    for (int j = threadIdx.x; j < Ll2; j += blockDim.x) erow[j] = conj2(et[(int64_t)ub * Ll2 + j]);
    for (int j = threadIdx.x; j < 2 * L; j += blockDim.x) r1s[j] = rh[j];
    __syncthreads();
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int m0 = 0; m0 < KK; m0 += MC) {
        const int nm = KT ? KT * KT : min(MC, KK - m0);
        double2 acc[MC];
        int o1[MC], o2[MC];
#pragma unroll
        for (int m = 0; m < MC; ++m) {
            acc[m] = make_double2(0.0, 0.0);
            const int mm = m0 + m;
            o1[m] = ub1 + Ll * (mm / K);  // u1 of accumulator m (KT: o1 indexed by m1 only)
            o2[m] = ub2 + Ll * (mm % K);
        }
        for (int up1 = ty; up1 < L; up1 += 8) {
            const double2* erow1 = erow + (up1 % Ll) * Ll;
            int ub2p = tx % Ll;
            for (int up2 = tx; up2 < L; up2 += 32) {
                const double2 h = cmulc(erow1[ub2p], xh[up1 * L + up2]);
                ub2p += 32;
                while (ub2p >= Ll) ub2p -= Ll;
                if constexpr (KT > 0) {
                    double2 r2[KT];
#pragma unroll
                    for (int m2 = 0; m2 < KT; ++m2) {
                        int d2 = ub2 + Ll * m2 - up2;
                        d2 += d2 < 0 ? L : 0;
                        r2[m2] = r2s[d2];
                    }
#pragma unroll
                    for (int m1 = 0; m1 < KT; ++m1) {
                        int d1 = ub1 + Ll * m1 - up1;
                        d1 += d1 < 0 ? L : 0;
                        const double2 hr = cmul(h, r1s[d1]);
#pragma unroll
                        for (int m2 = 0; m2 < KT; ++m2) acc[m1 * KT + m2] = cadd(acc[m1 * KT + m2], cmul(hr, r2[m2]));
                    }
                } else {
#pragma unroll
                    for (int m = 0; m < MC; ++m) {
                        if (m < nm) {
                            int d1 = o1[m] - up1, d2 = o2[m] - up2;
                            d1 += d1 < 0 ? L : 0;
                            d2 += d2 < 0 ? L : 0;
                            acc[m] = cadd(acc[m], cmul(cmul(h, r1s[d1]), r2s[d2]));
                        }
                    }
                }
            }
        }
        block_csum_n(acc, nm, sred, sout);
        if (threadIdx.x < nm) {
            const int mm = m0 + threadIdx.x, m1 = mm / K, m2 = mm - m1 * K;
            const int u1 = ub1 + Ll * m1, u2 = ub2 + Ll * m2;
            const double2 t = cmul(conj2(e1[ub]), cmul(r1s[u1], r2s[u2]));
            const double2 a = sout[threadIdx.x];
            ax[u1 * L + u2] = make_double2(c2 * a.x + c1 * t.x, c2 * a.y + c1 * t.y);
        }
    }
}

// Gr[v] for the K^2 frequencies v = vbar + Ll m of one block (the diagonal Etilde[j, j - vbar] staged);
// each term h = Etilde[ubar, ubar - vbar] conj(xhat[u]) is formed once for all K^2 shifts v
template <int KT>
__global__ void __launch_bounds__(256) k_mom_G(const double2* __restrict__ xh, const double2* __restrict__ et,
                                               const double2* __restrict__ e1, int L, int Ll, int K, double c2,
                                               double c1, double2* __restrict__ gr) {
    extern __shared__ double2 ediag[];  // [Ll2]
    __shared__ double2 sred[8 * MC], sout[MC];
    const int Ll2 = Ll * Ll, KK = K * K;
    const int vb = blockIdx.x, vb1 = vb / Ll, vb2 = vb - vb1 * Ll;
    for (int j = threadIdx.x; j < Ll2; j += blockDim.x) {
        const int j1 = j / Ll, j2 = j - j1 * Ll;
        ediag[j] = et[(int64_t)j * Ll2 + imod(j1 - vb1, Ll) * Ll + imod(j2 - vb2, Ll)];
    }
    __syncthreads();
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int m0 = 0; m0 < KK; m0 += MC) {
        const int nm = KT ? KT * KT : min(MC, KK - m0);
        double2 acc[MC];
        int o1[MC], o2[MC];
#pragma unroll
        for (int m = 0; m < MC; ++m) {
            acc[m] = make_double2(0.0, 0.0);
            const int mm = m0 + m;
            o1[m] = vb1 + Ll * (mm / K);
            o2[m] = vb2 + Ll * (mm % K);
        }
        for (int u1 = ty; u1 < L; u1 += 8) {
            const double2* ed1 = ediag + (u1 % Ll) * Ll;
            int ub2 = tx % Ll;
            for (int u2 = tx; u2 < L; u2 += 32) {
                const double2 h = cmulc(ed1[ub2], xh[u1 * L + u2]);
                ub2 += 32;
                while (ub2 >= Ll) ub2 -= Ll;
                if constexpr (KT > 0) {
#pragma unroll
                    for (int m1 = 0; m1 < KT; ++m1) {
                        int w1 = u1 - vb1 - Ll * m1;
                        w1 += w1 < 0 ? L : 0;
                        const double2* xrow = xh + w1 * L;
#pragma unroll
                        for (int m2 = 0; m2 < KT; ++m2) {
                            int w2 = u2 - vb2 - Ll * m2;
                            w2 += w2 < 0 ? L : 0;
                            acc[m1 * KT + m2] = cadd(acc[m1 * KT + m2], cmul(h, xrow[w2]));
                        }
                    }
                } else {
#pragma unroll
                    for (int m = 0; m < MC; ++m) {
                        if (m < nm) {
                            int w1 = u1 - o1[m], w2 = u2 - o2[m];
                            w1 += w1 < 0 ? L : 0;
                            w2 += w2 < 0 ? L : 0;
                            acc[m] = cadd(acc[m], cmul(h, xh[w1 * L + w2]));
                        }
                    }
                }
            }
        }
        block_csum_n(acc, nm, sred, sout);
        if (threadIdx.x < nm) {
            const int mm = m0 + threadIdx.x, m1 = mm / K, m2 = mm - m1 * K;
            const int v1 = vb1 + Ll * m1, v2 = vb2 + Ll * m2;
            const double2 t = cmulc(e1[vb], xh[v1 * L + v2]);
            const double2 a = sout[threadIdx.x];
            gr[v1 * L + v2] = make_double2(c2 * a.x + c1 * t.x, c2 * a.y + c1 * t.y);
        }
    }
}

// f (one block)
__global__ void k_mom_fsum(const double* __restrict__ fpart, int Ll2, double lam, double* __restrict__ out) {
    __shared__ double red[32];
    double a = 0.0, b = 0.0;
    for (int k = threadIdx.x; k < Ll2; k += blockDim.x) {
        a += fpart[k];
        b += fpart[Ll2 + k];
    }
    a = block_sum(a, red);
    __syncthreads();
    b = block_sum(b, red);
    if (threadIdx.x == 0) out[0] = a / ((double)Ll2 * Ll2) + lam * b / (double)Ll2;
}

// grad x = Re(DFT(Ax)), grad rho (joint) = Re(IDFT(Gr)) row s; grad rho1[s], grad rho2[s] (block s)
__global__ void k_mom_grad(const double2* __restrict__ gxc, const double2* __restrict__ grc,
                           const double* __restrict__ theta, int L, double* __restrict__ out) {
    __shared__ double red[32];
    const int L2 = L * L, s = blockIdx.x;
    double* gx = out + 1;
    double* g1 = gx + L2;
    double* g2 = g1 + L;
    double* gj = g2 + L;
    const double* r1 = theta + L2;
    const double* r2 = r1 + L;
    double a = 0.0, b = 0.0;
    for (int t = threadIdx.x; t < L; t += blockDim.x) {
        gx[s * L + t] = gxc[s * L + t].x;
        const double v = grc[s * L + t].x;
        gj[s * L + t] = v;
        a += v * r2[t];
        b += grc[t * L + s].x * r1[t];
    }
    a = block_sum(a, red);
    __syncthreads();
    b = block_sum(b, red);
    if (threadIdx.x == 0) {
        g1[s] = a;
        g2[s] = b;
    }
}

// Algorithm 1's projection with the built-in stand-in D (3x3 circular box filter, clamp to [-1, 1]; one block)
__global__ void k_mom_project(double* __restrict__ x, double* __restrict__ tmp, int L) {
    const int L2 = L * L;
    for (int p = threadIdx.x; p < L2; p += blockDim.x) tmp[p] = x[p];
    __syncthreads();
    for (int p = threadIdx.x; p < L2; p += blockDim.x) {
        const int p1 = p / L, p2 = p - p1 * L;
        double acc = 0.0;
        for (int d1 = -1; d1 <= 1; ++d1)
            for (int d2 = -1; d2 <= 1; ++d2) acc += tmp[imod(p1 + d1, L) * L + imod(p2 + d2, L)];
        const double v = acc / 9.0;
        x[p] = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
    }
}

unsigned grid_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8192)); }

}  // namespace momo

using namespace momo;

bool mom_supported(const srmra_ctx* c) { return c->Ll <= 64; }
bool mom_ready(const srmra_ctx* c) { return c->mom && c->mom->ready; }

void mom_free(srmra_ctx* c) {
    MomState* m = c->mom;
    if (!m) return;
    for (void* p : {(void*)m->tw, (void*)m->t2, (void*)m->t1, (void*)m->et, (void*)m->e1, (void*)m->xh, (void*)m->rh,
                    (void*)m->ax, (void*)m->gr, (void*)m->tmp, (void*)m->theta, (void*)m->out, (void*)m->fpart})
        if (p) cudaFree(p);
    delete m;
    c->mom = nullptr;
}

#define MCK(x)                                    \
    do {                                          \
        cudaError_t e_ = (x);                     \
        if (e_ != cudaSuccess) return e_;         \
    } while (0)

static cudaError_t mom_alloc(srmra_ctx* c) {
    if (c->mom) return cudaSuccess;
    MomState* m = new MomState();
    c->mom = m;
    m->L = c->L;
    m->Ll = c->Ll;
    m->K = c->K;
    m->lambda = 1.0 / ((double)c->L2 * (1.0 + c->sigma * c->sigma));
    const size_t Ll4 = (size_t)c->Ll2 * c->Ll2;
    MCK(cudaMalloc(&m->tw, sizeof(double2) * c->L));
    MCK(cudaMalloc(&m->t2, sizeof(double2) * Ll4));
    MCK(cudaMalloc(&m->t1, sizeof(double2) * c->Ll2));
    MCK(cudaMalloc(&m->et, sizeof(double2) * Ll4));
    MCK(cudaMalloc(&m->e1, sizeof(double2) * c->Ll2));
    for (double2** p : {&m->xh, &m->rh, &m->ax, &m->gr, &m->tmp}) MCK(cudaMalloc(p, sizeof(double2) * c->L2));
    MCK(cudaMalloc(&m->theta, sizeof(double) * (c->L2 + 2 * c->L)));
    MCK(cudaMalloc(&m->out, sizeof(double) * (1 + 2 * c->L2 + 2 * c->L)));
    MCK(cudaMalloc(&m->fpart, sizeof(double) * 2 * c->Ll2));
    k_twiddle<<<grid_for(c->L), 256, 0, c->stream>>>(m->tw, c->L);
    return cudaGetLastError();
}

// 2-D DFT of a complex [n][n] array in place through scratch (sgn -1 forward, +1 inverse-sign, unnormalised)
static cudaError_t dft2(srmra_ctx* c, double2* a, double2* scratch, int n, int sgn) {
    MomState* m = c->mom;
    const int step = m->L / n;
    const int th = std::min(n, 256);
    const size_t sh = sizeof(double2) * 2 * n;
    k_dft_line<<<n, th, sh, c->stream>>>(a, scratch, n, n, 1, sgn, m->tw, step);         // rows
    k_dft_line<<<n, th, sh, c->stream>>>(scratch, a, n, 1, n, sgn, m->tw, step);         // columns
    return cudaGetLastError();
}

// Fourier-domain data moments from device M1 | M2 (float64, [Ll2] | [Ll2][Ll2])
static cudaError_t mom_transform(srmra_ctx* c, const double* mdev) {
    MomState* m = c->mom;
    const int Ll = c->Ll, Ll2 = c->Ll2, step = c->K;
    const int64_t Ll4 = (int64_t)Ll2 * Ll2;
    double2* s4 = nullptr;
    MCK(cudaMallocAsync(&s4, sizeof(double2) * Ll4, c->stream));
    k_sym_to_c<<<grid_for(Ll4), 256, 0, c->stream>>>(mdev + Ll2, m->t2, Ll2);
    // axes a1, a2 (sign -), b1, b2 (sign +) of M2[a1][a2][b1][b2]
    const int64_t L3 = (int64_t)Ll * Ll2;
    k_dft_axis<<<grid_for(Ll4), 256, 0, c->stream>>>(m->t2, s4, 1, Ll, L3, -1, m->tw, step);
    k_dft_axis<<<grid_for(Ll4), 256, 0, c->stream>>>(s4, m->t2, Ll, Ll, Ll2, -1, m->tw, step);
    k_dft_axis<<<grid_for(Ll4), 256, 0, c->stream>>>(m->t2, s4, Ll2, Ll, Ll, +1, m->tw, step);
    k_dft_axis<<<grid_for(Ll4), 256, 0, c->stream>>>(s4, m->t2, L3, Ll, 1, +1, m->tw, step);
    k_sub_diag<<<grid_for(Ll2), 256, 0, c->stream>>>(m->t2, Ll2, c->sigma * c->sigma * (double)Ll2);
    k_real_to_c<<<grid_for(Ll2), 256, 0, c->stream>>>(mdev, m->t1, Ll2);
    k_dft_axis<<<grid_for(Ll2), 256, 0, c->stream>>>(m->t1, s4, 1, Ll, Ll, -1, m->tw, step);
    k_dft_axis<<<grid_for(Ll2), 256, 0, c->stream>>>(s4, m->t1, Ll, Ll, 1, -1, m->tw, step);
    cudaFreeAsync(s4, c->stream);
    return cudaGetLastError();
}

// srmra_mom_set_moments: host moments (m1, m2 non-NULL) or the empirical ones of the loaded data
int mom_set(srmra_ctx* c, const double* m1, const double* m2, std::string& err) {
    cudaError_t e = mom_alloc(c);
    const size_t nout = (size_t)c->Ll2 + (size_t)c->Ll2 * c->Ll2;
    double* mdev = nullptr;
    if (e == cudaSuccess) e = cudaMallocAsync(&mdev, sizeof(double) * nout, c->stream);
    int rc = SRMRA_OK;
    if (e == cudaSuccess) {
        if (m1 && m2) {
            e = cudaMemcpyAsync(mdev, m1, sizeof(double) * c->Ll2, cudaMemcpyHostToDevice, c->stream);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(mdev + c->Ll2, m2, sizeof(double) * c->Ll2 * c->Ll2, cudaMemcpyHostToDevice, c->stream);
        } else {
            rc = moments_dev(c, mdev, err);
        }
    }
    if (e == cudaSuccess && rc == SRMRA_OK) e = mom_transform(c, mdev);
    if (mdev) cudaFreeAsync(mdev, c->stream);
    const cudaError_t es = cudaStreamSynchronize(c->stream);  // host sources may be pageable / go out of scope
    if (e == cudaSuccess) e = es;
    if (rc != SRMRA_OK) return rc;
    if (e != cudaSuccess) {
        err = std::string("srmra_mom_set_moments: ") + cudaGetErrorString(e);
        return SRMRA_ERR_CUDA;
    }
    c->mom->ready = true;
    return SRMRA_OK;
}

// objective + gradient at the device theta (m->theta); result in m->out
static cudaError_t mom_eval_dev(srmra_ctx* c) {
    MomState* m = c->mom;
    const int L = c->L, Ll = c->Ll, K = c->K, L2 = c->L2, Ll2 = c->Ll2;
    const double L4 = (double)L2 * L2;
    const double c1 = 2.0 * m->lambda / ((double)Ll2 * K * K);
    k_real_to_c<<<grid_for(L2), 256, 0, c->stream>>>(m->theta, m->xh, L2);
    MCK(dft2(c, m->xh, m->tmp, L, -1));
    k_rhohat<<<2, std::min(L, 256), sizeof(double2) * 2 * L, c->stream>>>(m->theta + L2, L, m->tw, m->rh);
    const size_t sa = sizeof(double2) * (Ll2 + 2 * L), sg = sizeof(double2) * Ll2;
#define MOM_AG(KT)                                                                                                 \
    k_mom_E<KT><<<Ll2, 256, sizeof(double2) * (2 * L + K * K), c->stream>>>(m->xh, m->rh, m->t2, m->t1, L, Ll, K,   \
                                                                          m->et, m->e1, m->fpart);              \
    k_mom_A<KT><<<Ll2, 256, sa, c->stream>>>(m->xh, m->rh, m->et, m->e1, L, Ll, K, 4.0 / L4, c1, m->ax);        \
    k_mom_G<KT><<<Ll2, 256, sg, c->stream>>>(m->xh, m->et, m->e1, L, Ll, K, 2.0 / L4, c1, m->gr)
    switch (K) {
        case 1: MOM_AG(1); break;
        case 2: MOM_AG(2); break;
        case 3: MOM_AG(3); break;
        case 4: MOM_AG(4); break;
        default: MOM_AG(0); break;
    }
#undef MOM_AG
    MCK(dft2(c, m->ax, m->tmp, L, -1));
    MCK(dft2(c, m->gr, m->tmp, L, +1));
    k_mom_fsum<<<1, 256, 0, c->stream>>>(m->fpart, Ll2, m->lambda, m->out);
    k_mom_grad<<<L, std::min(L, 128), 0, c->stream>>>(m->ax, m->gr, m->theta, L, m->out);
    return cudaGetLastError();
}

static PerDeviceOnce mom_attr_once;
static cudaError_t mom_attrs_set() {
    const int bytes = (int)sizeof(double2) * (64 * 64 + 2 * 4096);  // Ll <= 64; L <= 4096
#define MOM_ATTR(KT)                                                                             \
    MCK(cudaFuncSetAttribute(k_mom_A<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)); \
    MCK(cudaFuncSetAttribute(k_mom_G<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes))
    MOM_ATTR(0);
    MOM_ATTR(1);
    MOM_ATTR(2);
    MOM_ATTR(3);
    MOM_ATTR(4);
#undef MOM_ATTR
    return cudaSuccess;
}
static cudaError_t mom_attrs(int) { return mom_attr_once.run(mom_attrs_set); }

// srmra_mom_objective: theta from host (x | rho1 | rho2), outputs to host (any NULL)
int mom_objective(srmra_ctx* c, const double* x, const double* r1, const double* r2, double* f, double* gx,
                  double* g1, double* g2, std::string& err) {
    MomState* m = c->mom;
    const int L = c->L, L2 = c->L2;
    std::vector<double> th(L2 + 2 * L), out(1 + 2 * L2 + 2 * L);
    std::copy(x, x + L2, th.begin());
    std::copy(r1, r1 + L, th.begin() + L2);
    std::copy(r2, r2 + L, th.begin() + L2 + L);
    cudaError_t e = mom_attrs(c->Ll2);
    if (e == cudaSuccess) e = cudaMemcpyAsync(m->theta, th.data(), sizeof(double) * th.size(), cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = mom_eval_dev(c);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out.data(), m->out, sizeof(double) * out.size(), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        err = std::string("srmra_mom_objective: ") + cudaGetErrorString(e);
        return SRMRA_ERR_CUDA;
    }
    if (f) *f = out[0];
    if (gx) std::copy(out.begin() + 1, out.begin() + 1 + L2, gx);
    if (g1) std::copy(out.begin() + 1 + L2, out.begin() + 1 + L2 + L, g1);
    if (g2) std::copy(out.begin() + 1 + L2 + L, out.begin() + 1 + L2 + 2 * L, g2);
    return SRMRA_OK;
}

// ---------------------------------------------------------------- Algorithm 1 driver (host L-BFGS)
// Variables z = (x [L2], a1 [L], a2 [L]) with rho_j = softmax(a_j) (keeps the shift pmfs on the simplex;
// DESIGN.md reading R14).  Each step: two-loop L-BFGS direction (memory 10), Armijo backtracking from
// step 1; every F steps the projection x <- D(x, sigma_j) (sigma_j = 2^(-(j-1)/10), eq:decaying_function)
// and a memory reset.  Stops after max_steps steps, when ||grad||_inf <= gtol, or when the line search
// finds no decrease.
struct Lbfgs {
    int n = 0, mem = 10;
    std::vector<std::vector<double>> S, Y;
    std::vector<double> rhoinv;
    void reset() { S.clear(); Y.clear(); rhoinv.clear(); }
    void push(const std::vector<double>& s, const std::vector<double>& y) {
        double sy = 0.0, ss = 0.0, yy = 0.0;
        for (int i = 0; i < n; ++i) { sy += s[i] * y[i]; ss += s[i] * s[i]; yy += y[i] * y[i]; }
        if (!(sy > 1e-12 * sqrt(ss * yy))) return;  // curvature condition: keep H positive definite
        if ((int)S.size() == mem) { S.erase(S.begin()); Y.erase(Y.begin()); rhoinv.erase(rhoinv.begin()); }
        S.push_back(s);
        Y.push_back(y);
        rhoinv.push_back(sy);
    }
    void direction(const std::vector<double>& g, std::vector<double>& d) const {
        d = g;
        const int k = (int)S.size();
        std::vector<double> al(k);
        for (int j = k - 1; j >= 0; --j) {
            double a = 0.0;
            for (int i = 0; i < n; ++i) a += S[j][i] * d[i];
            al[j] = a / rhoinv[j];
            for (int i = 0; i < n; ++i) d[i] -= al[j] * Y[j][i];
        }
        if (k > 0) {
            double yy = 0.0;
            for (int i = 0; i < n; ++i) yy += Y[k - 1][i] * Y[k - 1][i];
            const double gam = rhoinv[k - 1] / yy;
            for (int i = 0; i < n; ++i) d[i] *= gam;
        }
        for (int j = 0; j < k; ++j) {
            double b = 0.0;
            for (int i = 0; i < n; ++i) b += Y[j][i] * d[i];
            b /= rhoinv[j];
            for (int i = 0; i < n; ++i) d[i] += S[j][i] * (al[j] - b);
        }
        for (int i = 0; i < n; ++i) d[i] = -d[i];
    }
};

static void softmax(const double* a, int L, double* r) {
    double mx = a[0];
    for (int i = 1; i < L; ++i) mx = std::max(mx, a[i]);
    double s = 0.0;
    for (int i = 0; i < L; ++i) s += (r[i] = exp(a[i] - mx));
    for (int i = 0; i < L; ++i) r[i] /= s;
}

int mom_run(srmra_ctx* c, int max_steps, int F, double gtol, double* f_out, int* steps_out, std::string& err) {
    MomState* m = c->mom;
    const int L = c->L, L2 = c->L2, n = L2 + 2 * L;
    std::vector<double> th(L2 + 2 * L), out(1 + 2 * L2 + 2 * L);
    cudaError_t e = mom_attrs(c->Ll2);
    if (e == cudaSuccess) e = cudaMemcpyAsync(th.data(), c->d_x64, sizeof(double) * L2, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(th.data() + L2, c->d_rho, sizeof(double) * 2 * L, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        err = std::string("srmra_mom_run: ") + cudaGetErrorString(e);
        return SRMRA_ERR_CUDA;
    }
    std::vector<double> z(n), g(n), d, zn(n), gn(n), s(n), yv(n);
    for (int i = 0; i < L2; ++i) z[i] = th[i];
    for (int i = 0; i < 2 * L; ++i) z[L2 + i] = log(std::max(th[L2 + i], 1e-300));
    // f and df/dz at z (theta = (x, softmax(a1), softmax(a2)))
    auto eval = [&](const std::vector<double>& zz, std::vector<double>& gg, double& fv) -> cudaError_t {
        std::copy(zz.begin(), zz.begin() + L2, th.begin());
        softmax(zz.data() + L2, L, th.data() + L2);
        softmax(zz.data() + L2 + L, L, th.data() + L2 + L);
        MCK(cudaMemcpyAsync(m->theta, th.data(), sizeof(double) * th.size(), cudaMemcpyHostToDevice, c->stream));
        MCK(mom_eval_dev(c));
        MCK(cudaMemcpyAsync(out.data(), m->out, sizeof(double) * (1 + L2 + 2 * L), cudaMemcpyDeviceToHost, c->stream));
        MCK(cudaStreamSynchronize(c->stream));
        fv = out[0];
        std::copy(out.begin() + 1, out.begin() + 1 + L2, gg.begin());
        for (int j = 0; j < 2; ++j) {  // d/da_j of softmax: r (g - <r, g>)
            const double* r = th.data() + L2 + j * L;
            const double* gr = out.data() + 1 + L2 + j * L;
            double dot = 0.0;
            for (int i = 0; i < L; ++i) dot += r[i] * gr[i];
            for (int i = 0; i < L; ++i) gg[L2 + j * L + i] = r[i] * (gr[i] - dot);
        }
        return cudaSuccess;
    };
    auto ginf = [&](const std::vector<double>& gg) {
        double mx = 0.0;
        for (double v : gg) mx = std::max(mx, fabs(v));
        return mx;
    };
    Lbfgs H;
    H.n = n;
    double f = 0.0, fn = 0.0;
    int steps = 0, nproj = 0;
    e = eval(z, g, f);
    for (; e == cudaSuccess && steps < max_steps && isfinite(f) && ginf(g) > gtol; ++steps) {
        H.direction(g, d);
        double gd = 0.0;
        for (int i = 0; i < n; ++i) gd += g[i] * d[i];
        if (!(gd < 0.0)) {  // not a descent direction: steepest descent, fresh memory
            H.reset();
            for (int i = 0; i < n; ++i) d[i] = -g[i];
            gd = 0.0;
            for (int i = 0; i < n; ++i) gd += g[i] * d[i];
        }
        double a = 1.0;
        if (H.S.empty()) {  // first step of a memory: unit step along d / ||d||_inf
            double dn = 0.0;
            for (double v : d) dn = std::max(dn, fabs(v));
            a = dn > 0 ? std::min(1.0, 1.0 / dn) : 1.0;
        }
        bool ok = false;
        for (int bt = 0; bt < 60 && e == cudaSuccess; ++bt, a *= 0.5) {  // Armijo backtracking
            for (int i = 0; i < n; ++i) zn[i] = z[i] + a * d[i];
            e = eval(zn, gn, fn);
            if (e == cudaSuccess && isfinite(fn) && fn <= f + 1e-4 * a * gd) {
                ok = true;
                break;
            }
        }
        if (e != cudaSuccess || !ok) break;
        for (int i = 0; i < n; ++i) { s[i] = zn[i] - z[i]; yv[i] = gn[i] - g[i]; }
        H.push(s, yv);
        z.swap(zn);
        g.swap(gn);
        f = fn;
        if (F > 0 && (steps + 1) % F == 0) {  // Algorithm 1 step 2(b)-(c): x <- D(x, sigma_j)
            const double sig = pow(2.0, -(double)(nproj++) / 10.0);
            e = cudaMemcpyAsync(m->theta, z.data(), sizeof(double) * L2, cudaMemcpyHostToDevice, c->stream);
            if (e != cudaSuccess) break;
            if (c->denoiser) {
                if (c->denoiser(m->theta, L, sig, (void*)c->stream, c->denoiser_user) != 0) {
                    err = "denoiser hook failed";
                    return SRMRA_ERR_NUMERIC;
                }
            } else {
                double* tmpx = reinterpret_cast<double*>(m->tmp);
                k_mom_project<<<1, 1024, 0, c->stream>>>(m->theta, tmpx, L);
                e = cudaGetLastError();
            }
            if (e == cudaSuccess) e = cudaMemcpyAsync(z.data(), m->theta, sizeof(double) * L2, cudaMemcpyDeviceToHost, c->stream);
            if (e == cudaSuccess) e = eval(z, g, f);
            H.reset();
        }
    }
    if (e != cudaSuccess) {
        err = std::string("srmra_mom_run: ") + cudaGetErrorString(e);
        return SRMRA_ERR_CUDA;
    }
    // the result becomes the context's estimate (x64 | x32 | rho1 | rho2)
    std::copy(z.begin(), z.begin() + L2, th.begin());
    softmax(z.data() + L2, L, th.data() + L2);
    softmax(z.data() + L2 + L, L, th.data() + L2 + L);
    std::vector<float> x32(L2);
    for (int i = 0; i < L2; ++i) x32[i] = (float)th[i];
    e = cudaMemcpyAsync(c->d_x64, th.data(), sizeof(double) * L2, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->d_x32, x32.data(), sizeof(float) * L2, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->d_rho, th.data() + L2, sizeof(double) * 2 * L, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        err = std::string("srmra_mom_run: ") + cudaGetErrorString(e);
        return SRMRA_ERR_CUDA;
    }
    if (f_out) *f_out = f;
    if (steps_out) *steps_out = steps;
    return isfinite(f) ? SRMRA_OK : SRMRA_ERR_NUMERIC;
}

}  // namespace srmra
