// k_fft_aux.cu — the small per-iteration kernels around the FFT-path E/M kernel (k_fft.cu), all in
// float64 with a power-of-two L_low (masked twiddle indices, twiddle table from the host):
//   k_fft_init   (once per load)  Yhat_i = rfft2(y_i)
//   k_fft_prep   (a1)  blocks 0..K^2-1: Xhat_r = rfft2(x_r) / L_low^2;  block K^2: E_r = ||x_r||^2,
//                      E_min, log rho1, log rho2, beta_r = (E_min - E_r)/(2 sigma^2)   (k_common.cu)
//   k_fft_reduce (a5)  fixed-order float64 sum of the per-CTA float32 partials (deterministic)
//   k_fft_fold   (a5)  b_r = irfft2(Bhat_r)/L_low^2 scattered to b[(K m - r) mod L] (eq:x_EM numerator);
//                      block (0,0) also forms class mass and the marginals of eq:rho_EM from the mass
//                      lines (column k2 = 0 and row k1 = 0 of sum_i What_{i,r}).
#include <math.h>

#include "srmra_internal.cuh"

namespace srmra {

int ystride_of(int Ll);
int fft_partial_bins(int KK, int Ll);

namespace fftaux {

// forward real 2-D DFT of the Ll x Ll image `src` (smem, float64) -> half spectrum `out` (float32),
// scaled; `tmp` holds Ll x Lh complex; cs/sn: cos/sin(2 pi j / Ll), j < Ll.
__device__ void dft2_real_fwd(const double* src, double2* tmp, const double* cs, const double* sn, int Ll,
                              double scale, float2* out) {
    const int Lh = Ll / 2 + 1, M = Ll - 1;
    for (int e = threadIdx.x; e < Ll * Lh; e += blockDim.x) {  // along n2: tmp[n1][k2]
        const int n1 = e / Lh, k2 = e - n1 * Lh;
        const double* row = src + n1 * Ll;
        double re = 0, im = 0;
        for (int n2 = 0; n2 < Ll; ++n2) {
            const int j = (k2 * n2) & M;
            re = fma(row[n2], cs[j], re);
            im = fma(-row[n2], sn[j], im);
        }
        tmp[e] = make_double2(re, im);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < Ll * Lh; e += blockDim.x) {  // along n1: out[k1][k2]
        const int k1 = e / Lh, k2 = e - k1 * Lh;
        double re = 0, im = 0;
        for (int n1 = 0; n1 < Ll; ++n1) {
            const int j = (k1 * n1) & M;
            const double2 t = tmp[n1 * Lh + k2];
            re += t.x * cs[j] + t.y * sn[j];  // t * exp(-i theta)
            im += t.y * cs[j] - t.x * sn[j];
        }
        out[e] = make_float2((float)(re * scale), (float)(im * scale));
    }
}

__device__ void load_tw(const double* tw, double* cs, double* sn, int Ll) {
    for (int j = threadIdx.x; j < Ll; j += blockDim.x) {
        cs[j] = tw[j];
        sn[j] = tw[Ll + j];
    }
}

__global__ void k_fft_init(const float* __restrict__ y, int64_t n, int Ll, int ystride, const double* __restrict__ tw,
                           float2* __restrict__ yhat) {
    extern __shared__ double sm[];
    const int Lh = Ll / 2 + 1;
    double* cs = sm;
    double* sn = cs + Ll;
    double* src = sn + Ll;
    double2* tmp = reinterpret_cast<double2*>(src + Ll * Ll);
    load_tw(tw, cs, sn, Ll);
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        for (int k = threadIdx.x; k < Ll * Ll; k += blockDim.x) src[k] = (double)y[i * Ll * Ll + k];
        __syncthreads();
        dft2_real_fwd(src, tmp, cs, sn, Ll, 1.0, yhat + i * ystride);
        if (threadIdx.x == 0 && ystride > Ll * Lh) yhat[i * ystride + Ll * Lh] = make_float2(0.f, 0.f);
        __syncthreads();
    }
}

__global__ void k_fft_prep(const double* __restrict__ x, const double* __restrict__ rho, int L, int K, double inv_2s2,
                           const double* __restrict__ tw, float2* __restrict__ xhat, float* __restrict__ f32,
                           double* __restrict__ f64) {
    extern __shared__ double sm[];
    const int Ll = L / K, Lh = Ll / 2 + 1, KK = K * K;
    if ((int)blockIdx.x < KK) {
        const int r = blockIdx.x, r1 = r / K, r2 = r % K;
        double* cs = sm;
        double* sn = cs + Ll;
        double* src = sn + Ll;
        double2* tmp = reinterpret_cast<double2*>(src + Ll * Ll);
        load_tw(tw, cs, sn, Ll);
        for (int m = threadIdx.x; m < Ll * Ll; m += blockDim.x) {
            const int m1 = m / Ll, m2 = m - m1 * Ll;
            src[m] = x[(size_t)imod(K * m1 - r1, L) * L + imod(K * m2 - r2, L)];   // x_r[m]
        }
        __syncthreads();
        dft2_real_fwd(src, tmp, cs, sn, Ll, 1.0 / ((double)Ll * Ll), xhat + (size_t)r * Ll * Lh);
        return;
    }
    // logit bias block (same arithmetic as k_common.cu k_prep)
    __shared__ double red[32];
    double* Es = sm;  // [KK]
    for (int r = 0; r < KK; ++r) {
        const int r1 = r / K, r2 = r % K;
        double acc = 0.0;
        for (int m = threadIdx.x; m < Ll * Ll; m += blockDim.x) {
            const int m1 = m / Ll, m2 = m - m1 * Ll;
            const double v = x[(size_t)imod(K * m1 - r1, L) * L + imod(K * m2 - r2, L)];
            acc += v * v;
        }
        acc = block_sum(acc, red);
        if (threadIdx.x == 0) Es[r] = acc;
    }
    __syncthreads();
    double emin = Es[0];
    for (int r = 1; r < KK; ++r) emin = fmin(emin, Es[r]);
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
        const double a = rho[k], b = rho[L + k];
        f32[k] = a > 0.0 ? (float)log(a) : -INFINITY;
        f32[L + k] = b > 0.0 ? (float)log(b) : -INFINITY;
    }
    for (int r = threadIdx.x; r < KK; r += blockDim.x) {
        f32[2 * L + r] = (float)((emin - Es[r]) * inv_2s2);
        f64[r] = Es[r];
    }
    if (threadIdx.x == 0) f64[KK] = emin;
}

// blockDim = (32 bins) x (8 slices); slice s sums partials s, s+8, ...; slices combined in order.
__global__ void k_fft_reduce(const float2* __restrict__ part, const double* __restrict__ llpart, int nparts, int PB,
                             double* __restrict__ bhat, double* __restrict__ ll) {
    __shared__ double2 acc[8][33];
    const int b = threadIdx.x & 31, sl = threadIdx.x >> 5;
    const int k = blockIdx.x * 32 + b;
    double sx = 0.0, sy = 0.0;
    if (k < PB) {
        for (int c = sl; c < nparts; c += 8) {
            const float2 v = part[(size_t)c * PB + k];
            sx += v.x;
            sy += v.y;
        }
    }
    acc[sl][b] = make_double2(sx, sy);
    __syncthreads();
    if (sl == 0 && k < PB) {
        double tx = 0.0, ty = 0.0;
        for (int j = 0; j < 8; ++j) {
            tx += acc[j][b].x;
            ty += acc[j][b].y;
        }
        bhat[2 * k] = tx;
        bhat[2 * k + 1] = ty;
    }
    if (blockIdx.x == 0 && sl == 1) {  // log-likelihood partials: strided lanes, fixed-order shuffle tree
        double s = 0.0;
        for (int c = b; c < nparts; c += 32) s += llpart[c];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (b == 0) *ll = s;
    }
}

// grid (KK, nchunk): block (r, ch) produces rows m1 in [ch*R, ch*R + R) of b_r.
__global__ void k_fft_fold(const double* __restrict__ bhat, const double* __restrict__ cline, int L, int K,
                           const double* __restrict__ tw, double* __restrict__ pack, int64_t off_cm, int64_t off_m1,
                           int64_t off_m2) {
    extern __shared__ double sm[];
    const int Ll = L / K, Lh = Ll / 2 + 1, KK = K * K, M = Ll - 1;
    const int r = blockIdx.x, r1 = r / K, r2 = r % K;
    const int R = Ll / gridDim.y, m1a = blockIdx.y * R;
    double* cs = sm;
    double* sn = cs + Ll;
    double2* B = reinterpret_cast<double2*>(sn + Ll);  // [Ll][Lh]
    double2* T = B + Ll * Lh;                          // [R][Lh]
    load_tw(tw, cs, sn, Ll);
    const double2* Bg = reinterpret_cast<const double2*>(bhat) + (size_t)r * Ll * Lh;
    for (int e = threadIdx.x; e < Ll * Lh; e += blockDim.x) B[e] = Bg[e];
    __syncthreads();
    for (int e = threadIdx.x; e < R * Lh; e += blockDim.x) {  // inverse along k1
        const int mm = e / Lh, k2 = e - mm * Lh, m1 = m1a + mm;
        double re = 0, im = 0;
        for (int k1 = 0; k1 < Ll; ++k1) {
            const int j = (k1 * m1) & M;
            const double2 t = B[k1 * Lh + k2];
            re += t.x * cs[j] - t.y * sn[j];  // t * exp(+i theta)
            im += t.y * cs[j] + t.x * sn[j];
        }
        T[e] = make_double2(re, im);
    }
    __syncthreads();
    const double inv = 1.0 / ((double)Ll * Ll);
    for (int e = threadIdx.x; e < R * Ll; e += blockDim.x) {  // c2r along k2
        const int mm = e / Ll, m2 = e - mm * Ll, m1 = m1a + mm;
        const double2* Tr = T + mm * Lh;
        double acc = Tr[0].x + ((m2 & 1) ? -Tr[Ll / 2].x : Tr[Ll / 2].x);
        for (int k2 = 1; k2 < Ll / 2; ++k2) {
            const int j = (k2 * m2) & M;
            acc += 2.0 * (Tr[k2].x * cs[j] - Tr[k2].y * sn[j]);
        }
        pack[(size_t)imod(K * m1 - r1, L) * L + imod(K * m2 - r2, L)] = acc * inv;
    }
    if (blockIdx.x != 0 || blockIdx.y != 0) return;
    // class mass and marginals from the mass lines of every class (fixed order, no atomics)
    const double2* C = reinterpret_cast<const double2*>(cline);
    for (int rr = threadIdx.x; rr < KK; rr += blockDim.x) pack[off_cm + rr] = C[(size_t)rr * (Ll + Lh)].x;
    const double invL = 1.0 / Ll;
    for (int s = threadIdx.x; s < L; s += blockDim.x) {
        const int rs = s % K, t = s / K;
        double a1 = 0.0, a2 = 0.0;
        for (int ro = 0; ro < K; ++ro) {
            // marg1[s] = sum_{r2} R_{(rs, r2)}[t];  R_r[t] = (1/Ll) Re sum_k1 Ccol_r[k1] e^{+2 pi i k1 t / Ll}
            const double2* Cc = C + (size_t)(rs * K + ro) * (Ll + Lh);
            for (int k1 = 0; k1 < Ll; ++k1) {
                const int j = (k1 * t) & M;
                a1 += Cc[k1].x * cs[j] - Cc[k1].y * sn[j];
            }
            // marg2[s] = sum_{r1} C_{(r1, rs)}[t]; C_r[t] from the half row k1 = 0 (real signal)
            const double2* Cr = C + (size_t)(ro * K + rs) * (Ll + Lh) + Ll;
            a2 += Cr[0].x + ((t & 1) ? -Cr[Ll / 2].x : Cr[Ll / 2].x);
            for (int k2 = 1; k2 < Ll / 2; ++k2) {
                const int j = (k2 * t) & M;
                a2 += 2.0 * (Cr[k2].x * cs[j] - Cr[k2].y * sn[j]);
            }
        }
        pack[off_m1 + s] = a1 * invL;
        pack[off_m2 + s] = a2 * invL;
    }
}

}  // namespace fftaux

using namespace fftaux;

static size_t dft_smem(int Ll) { return sizeof(double) * (2 * Ll + Ll * Ll) + sizeof(double2) * Ll * (Ll / 2 + 1); }

cudaError_t launch_fft_init(srmra_ctx* c) {
    if (c->n_local == 0) return cudaSuccess;
    const size_t sm = dft_smem(c->Ll);
    cudaError_t e = cudaFuncSetAttribute(k_fft_init, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    const int64_t grid = c->n_local < 65536 ? c->n_local : 65536;
    k_fft_init<<<(unsigned)grid, 256, sm, c->stream>>>(c->d_y, c->n_local, c->Ll, ystride_of(c->Ll), c->d_tw,
                                                         c->d_yhat);
    return cudaGetLastError();
}

cudaError_t launch_fft_prep(srmra_ctx* c) {
    cudaError_t e = cudaMemsetAsync(c->d_pack, 0, sizeof(double) * c->pk.total, c->stream);
    if (e != cudaSuccess) return e;
    size_t sm = dft_smem(c->Ll);
    if (sm < sizeof(double) * 256) sm = sizeof(double) * 256;
    e = cudaFuncSetAttribute(k_fft_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_fft_prep<<<c->KK + 1, 256, sm, c->stream>>>(c->d_x64, c->d_rho, c->L, c->K, c->inv_2s2, c->d_tw, c->d_xhat,
                                                  c->par.f32, c->par.f64);
    return cudaGetLastError();
}

cudaError_t launch_fft_fold(srmra_ctx* c) {
    const int Ll = c->Ll, Lh = Ll / 2 + 1;
    const int PB = fft_partial_bins(c->KK, Ll);
    cudaError_t e;
    if (c->n_local > 0) {
        k_fft_reduce<<<(PB + 31) / 32, 256, 0, c->stream>>>(c->d_part, c->d_llpart, c->fft_grid, PB, c->d_bhat,
                                                           c->d_pack + c->pk.ll);
    } else {
        e = cudaMemsetAsync(c->d_bhat, 0, sizeof(double) * 2 * (size_t)PB, c->stream);
        if (e != cudaSuccess) return e;
    }
    const int nchunk = Ll >= 8 ? Ll / 8 : 1;
    const int R = Ll / nchunk;
    const size_t sm = sizeof(double) * 2 * Ll + sizeof(double2) * ((size_t)Ll * Lh + (size_t)R * Lh);
    e = cudaFuncSetAttribute(k_fft_fold, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_fft_fold<<<dim3(c->KK, nchunk), 256, sm, c->stream>>>(c->d_bhat, c->d_bhat + (size_t)2 * c->KK * Ll * Lh, c->L,
                                                            c->K, c->d_tw, c->d_pack, c->pk.cmass, c->pk.m1,
                                                            c->pk.m2);
    return cudaGetLastError();
}

}  // namespace srmra
