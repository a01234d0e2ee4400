// finalize.cuh — a7 (x' = b / A, rho' from the marginals, LL_t) and a8 (projection D) as a block-level
// device function, included by k_common.cu (direct path k_finalize) and k_fft_aux.cu (last block of
// the FFT fold).  Cited: PAPER.md:255-263 (eq:x_EM), 266-268 (eq:rho_EM), 384-388 (Algorithm 2 step 2).
#pragma once
#include "srmra_internal.cuh"

namespace srmra {

// Block-level body (any block size); called by k_finalize (direct path) and by the last block of
// the FFT path's fold kernel.  xs_dyn: dynamic shared memory of >= 8 L^2 bytes when L^2 <= 16384.
__device__ inline void finalize_body(const double* __restrict__ pack, int64_t off_cm, int64_t off_m1,
                              int64_t off_m2, int64_t off_ll, int L, int K, double tau, int project,
                              double* __restrict__ x64, float* __restrict__ x32, double* __restrict__ rho,
                              double* __restrict__ xtmp, double* __restrict__ trace, int t, int trace_cap,
                              int* __restrict__ flag, double* xs_dyn, const double* __restrict__ colsum = nullptr,
                              double* __restrict__ rhoj = nullptr) {
    __shared__ double red[32];
    __shared__ double cm[256];
    const int KK = K * K, L2 = L * L;
    for (int r = threadIdx.x; r < KK; r += blockDim.x) cm[r] = pack[off_cm + r];
    __syncthreads();
    double tot = 0.0;
    for (int r = 0; r < KK; ++r) tot += cm[r];   // sum_i sum_s' w^{i,s'} (eq:rho_EM denominator)
    // rho' (eq:rho_EM, separable marginals).  A shift with rho_t = 0 has w = 0 for every observation,
    // so its marginal is exactly 0 (kept exact here; the frequency-domain path would otherwise leave
    // rounding noise there); other marginals are clamped at 0 and each axis is normalised by its own
    // total sum_i sum_s w (the eq:rho_EM denominator) so that sum rho = 1 to rounding.
    if (rhoj) {
        // joint prior (NEXT-3): eq:rho_EM as written, rho'[s] = sum_i w^{i,s} / sum_i sum_s' w^{i,s'}
        // (zero prior mass gives w = 0 exactly); rho1 | rho2 become its marginals
        if (tot > 0.0) {
            for (int s = threadIdx.x; s < L2; s += blockDim.x) rhoj[s] = fmax(colsum[s], 0.0) / tot;
            for (int k = threadIdx.x; k < L; k += blockDim.x) {
                rho[k] = fmax(pack[off_m1 + k], 0.0) / tot;
                rho[L + k] = fmax(pack[off_m2 + k], 0.0) / tot;
            }
        }
        __syncthreads();
    }
    double m1s = 0.0, m2s = 0.0;
    for (int k = threadIdx.x; k < L && !rhoj; k += blockDim.x) {
        m1s += rho[k] == 0.0 ? 0.0 : fmax(pack[off_m1 + k], 0.0);
        m2s += rho[L + k] == 0.0 ? 0.0 : fmax(pack[off_m2 + k], 0.0);
    }
    m1s = block_sum(m1s, red);
    m2s = block_sum(m2s, red);
    __syncthreads();  // every thread has read rho_t above
    if (!rhoj && tot > 0.0 && m1s > 0.0 && m2s > 0.0) {
        for (int k = threadIdx.x; k < L; k += blockDim.x) {
            rho[k] = rho[k] == 0.0 ? 0.0 : fmax(pack[off_m1 + k], 0.0) / m1s;
            rho[L + k] = rho[L + k] == 0.0 ? 0.0 : fmax(pack[off_m2 + k], 0.0) / m2s;
        }
    }
    // x' = b / A (eq:x_EM, A diagonal; A[p] = class mass of class (-p mod K)); keep x_t if A <= tau.
    // With projection, x' is staged in shared memory when it fits (L^2 <= 16384), else in xtmp.
    double* stage = (L2 <= 16384 && xs_dyn) ? xs_dyn : xtmp;
    double* dst = project ? stage : x64;
    int bad = 0;
    for (int p = threadIdx.x; p < L2; p += blockDim.x) {
        const int p1 = p / L, p2 = p - p1 * L;
        const double A = cm[imod(-p1, K) * K + imod(-p2, K)];
        const double v = A > tau ? pack[p] / A : x64[p];
        dst[p] = v;
        if (!project) x32[p] = (float)v;
        bad |= !isfinite(v);
    }
    if (project) {
        __syncthreads();  // stage complete (global writes of this block are visible after the barrier too)
        for (int p = threadIdx.x; p < L2; p += blockDim.x) {
            const int p1 = p / L, p2 = p - p1 * L;
            const int rm = (p1 == 0 ? L - 1 : p1 - 1) * L, r0 = p1 * L, rp = (p1 == L - 1 ? 0 : p1 + 1) * L;
            const int cm1 = p2 == 0 ? L - 1 : p2 - 1, cp1 = p2 == L - 1 ? 0 : p2 + 1;
            double acc = stage[rm + cm1] + stage[rm + p2] + stage[rm + cp1];
            acc += stage[r0 + cm1] + stage[r0 + p2] + stage[r0 + cp1];
            acc += stage[rp + cm1] + stage[rp + p2] + stage[rp + cp1];
            double v = acc / 9.0;
            v = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
            x64[p] = v;
            x32[p] = (float)v;
        }
    }
    double b2 = block_sum((double)bad, red);
    if (threadIdx.x == 0) {
        const double ll = pack[off_ll];
        if (t < trace_cap) trace[t] = ll;
        if (b2 != 0.0 || !isfinite(ll)) atomicOr(flag, 1);
    }
}

}  // namespace srmra
