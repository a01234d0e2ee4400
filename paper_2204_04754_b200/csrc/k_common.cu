// k_common.cu — path-independent kernels of one EM iteration:
//   a0 init     ||y_i||^2 in float64
//   a1 prep     theta_t -> logit bias (log rho1, log rho2, class terms), E_r = ||x_r||^2
//   a5/a6 pack  colsum -> class mass, marginals (packed with b and LL for the all-reduce)
//   a7/a8 finalize   x' = b / A, rho' = marginals / mass, LL_t, projection D (3x3 box + clamp)
// Cited passages: PAPER.md:228-233 (eq:likelihood_EM), 247-250 (eq:weights_EM), 255-263
// (eq:x_EM, P^{-1} := P^T so A[p] is the class mass of class (-p mod K)), 266-268 (eq:rho_EM),
// 384-388 (Algorithm 2 projection step).
#include <math.h>

#include "finalize.cuh"
#include "srmra_internal.cuh"

namespace srmra {

// ---------------------------------------------------------------- a0: ||y_i||^2 (float64)
// One warp per observation; float4 loads (Ll^2 is a multiple of 4 for every supported shape).
// ||y_i||^2 in float64; it is non-finite exactly when some y_i[n] is, which sets bit 1 of *flag (the
// init-time validation of y runs here instead of a serial host scan)
__global__ void k_ynorm(const float* __restrict__ y, int64_t n, int Ll2, double* __restrict__ out, int* flag) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= n) return;
    const float* yi = y + i * Ll2;
    double acc = 0.0;
    if ((Ll2 & 3) == 0) {
        const float4* v = reinterpret_cast<const float4*>(yi);
        for (int k = lane; k < (Ll2 >> 2); k += 32) {
            float4 a = v[k];
            acc += (double)a.x * a.x + (double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w;
        }
    } else {
        for (int k = lane; k < Ll2; k += 32) acc += (double)yi[k] * yi[k];
    }
    acc = warp_sum(acc);
    if (lane == 0) {
        out[i] = acc;
        if (!isfinite(acc)) atomicOr(flag, 2);
    }
}

cudaError_t launch_init_obs(srmra_ctx* c, int64_t first, int64_t count) {
    if (count > 0) {
        const int wpb = 8;
        int64_t blocks = (count + wpb - 1) / wpb;
        k_ynorm<<<(unsigned)blocks, wpb * 32, 0, c->stream>>>(c->d_y + first * c->Ll2, count, c->Ll2,
                                                              c->d_ynorm + first, c->d_flag);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a1: prep
// Logit of shift s for observation i (derivation in DESIGN.md, "E-step numerics"):
//   ell[s] = log rho1[s1] + log rho2[s2] - ||y_i - P R_s x||^2 / (2 sigma^2)
//          = v[s] + Sref_i / sigma^2 - (E_min + ||y_i||^2) / (2 sigma^2)
//   v[s]   = (S[i,s] - Sref_i) / sigma^2 + lr1[s1] + lr2[s2] + beta[r(s)]
//   beta_r = (E_min - E_r) / (2 sigma^2),  E_r = ||x_r||^2 = ||P R_s x||^2 for every s in class r.
// E_r, E_min and beta are formed in float64; lr and beta are stored as float32 for the hot loop.
__global__ void k_prep(const double* __restrict__ x, const double* __restrict__ rho, int L, int K,
                       double inv_2s2, float* __restrict__ f32, double* __restrict__ f64,
                       const double* __restrict__ rhoj, float* __restrict__ lrj) {
    __shared__ double red[32];
    __shared__ double Es[256];
    const int KK = K * K, Ll = L / K;
    for (int r = 0; r < KK; ++r) {
        const int r1 = r / K, r2 = r % K;
        double acc = 0.0;
        for (int m = threadIdx.x; m < Ll * Ll; m += blockDim.x) {
            const int m1 = m / Ll, m2 = m % Ll;
            const double v = x[(size_t)imod(K * m1 - r1, L) * L + imod(K * m2 - r2, L)];
            acc += v * v;
        }
        acc = block_sum(acc, red);
        if (threadIdx.x == 0) Es[r] = acc;
    }
    __syncthreads();
    double emin = Es[0];
    for (int r = 1; r < KK; ++r) emin = fmin(emin, Es[r]);
    float* lr1 = f32;
    float* lr2 = f32 + L;
    float* beta = f32 + 2 * L;
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
        const double a = rho[k], b = rho[L + k];
        // joint prior (NEXT-3): the whole log prior sits in the per-shift table lrj
        lr1[k] = rhoj ? 0.f : (a > 0.0 ? (float)log(a) : -INFINITY);
        lr2[k] = rhoj ? 0.f : (b > 0.0 ? (float)log(b) : -INFINITY);
    }
    if (rhoj)
        for (int s = threadIdx.x; s < L * L; s += blockDim.x) lrj[s] = rhoj[s] > 0.0 ? (float)log(rhoj[s]) : -INFINITY;
    for (int r = threadIdx.x; r < KK; r += blockDim.x) {
        beta[r] = (float)((emin - Es[r]) * inv_2s2);
        f64[r] = Es[r];
    }
    if (threadIdx.x == 0) f64[KK] = emin;
}

cudaError_t launch_prep(srmra_ctx* c) {
    cudaError_t e;
    if (c->path == SRMRA_PATH_DIRECT &&
        (e = cudaMemsetAsync(c->d_colsum, 0, sizeof(double) * c->L2, c->stream)) != cudaSuccess)
        return e;
    if ((e = cudaMemsetAsync(c->d_pack, 0, sizeof(double) * c->pk.total, c->stream)) != cudaSuccess) return e;
    k_prep<<<1, 1024, 0, c->stream>>>(c->d_x64, c->d_rho, c->L, c->K, c->inv_2s2, c->par.f32, c->par.f64,
                                      c->joint ? c->d_rhoj : nullptr, c->d_lrj);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a5: pack statistics
// class mass c[r] = sum_{s in class r} colsum[s]; marg1[s1] = sum_{s2} colsum; marg2[s2] = sum_{s1}.
__global__ void k_pack(const double* __restrict__ colsum, int L, int K, double* __restrict__ pack,
                       int64_t off_cm, int64_t off_m1, int64_t off_m2) {
    __shared__ double cm[256];
    const int KK = K * K;
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
        double a = 0.0, b = 0.0;
        for (int j = 0; j < L; ++j) {
            a += colsum[(size_t)k * L + j];   // row k: s1 = k
            b += colsum[(size_t)j * L + k];   // column k: s2 = k
        }
        pack[off_m1 + k] = a;
        pack[off_m2 + k] = b;
    }
    // class masses: one block-wide float64 sum per class over its Ll^2 members s = r + K t
    const int Ll = L / K;
    __shared__ double red[32];
    for (int r = 0; r < KK; ++r) {
        const int r1 = r / K, r2 = r % K;
        double a = 0.0;
        for (int t = threadIdx.x; t < Ll * Ll; t += blockDim.x)
            a += colsum[(size_t)(r1 + K * (t / Ll)) * L + r2 + K * (t % Ll)];
        a = block_sum(a, red);
        if (threadIdx.x == 0) cm[r] = a;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < KK; r += blockDim.x) pack[off_cm + r] = cm[r];
}

cudaError_t launch_pack(srmra_ctx* c) {
    k_pack<<<1, 1024, 0, c->stream>>>(c->d_colsum, c->L, c->K, c->d_pack, c->pk.cmass, c->pk.m1, c->pk.m2);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a7 + a8: finalize, projection
__global__ void k_finalize(const double* __restrict__ pack, int64_t off_cm, int64_t off_m1,
                           int64_t off_m2, int64_t off_ll, int L, int K, double tau, int project,
                           double* __restrict__ x64, float* __restrict__ x32, double* __restrict__ rho,
                           double* __restrict__ xtmp, double* __restrict__ trace, int t, int trace_cap,
                           int* __restrict__ flag, const double* __restrict__ colsum, double* __restrict__ rhoj) {
    extern __shared__ double xs_dyn[];
    finalize_body(pack, off_cm, off_m1, off_m2, off_ll, L, K, tau, project, x64, x32, rho, xtmp, trace, t,
                  trace_cap, flag, xs_dyn, colsum, rhoj);
}

cudaError_t launch_finalize(srmra_ctx* c, int t, int project) {
    const size_t sm = c->L2 <= 16384 ? sizeof(double) * c->L2 : 0;
    static PerDeviceOnce attr;
    cudaError_t e = attr.run([] { return cudaFuncSetAttribute(k_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 8); });
    if (e != cudaSuccess) return e;
    k_finalize<<<1, 1024, sm, c->stream>>>(c->d_pack, c->pk.cmass, c->pk.m1, c->pk.m2, c->pk.ll, c->L, c->K,
                                          c->tau, project, c->d_x64, c->d_x32, c->d_rho, c->d_xtmp,
                                          c->d_trace, t, c->opt.trace_cap, c->d_flag, c->d_colsum,
                                          c->joint ? c->d_rhoj : nullptr);
    return cudaGetLastError();
}

// x32 = (float) x64 after a denoiser hook modified x64 (srmra_set_denoiser)
__global__ void k_x32_from_x64(const double* __restrict__ x64, int n, float* __restrict__ x32) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) x32[p] = (float)x64[p];
}
cudaError_t launch_x32_from_x64(srmra_ctx* c) {
    k_x32_from_x64<<<(c->L2 + 255) / 256, 256, 0, c->stream>>>(c->d_x64, c->L2, c->d_x32);
    return cudaGetLastError();
}

// NEXT-4, evaluation: corr[s] = sum_p xhat[(p - s) mod L] xref[p] for every shift s, so
// that ||R_s xhat - xref||^2 = ||xhat||^2 + ||xref||^2 - 2 corr[s]; one block per shift, float64.
__global__ void k_shift_corr(const double* __restrict__ xhat, const double* __restrict__ xref, int L,
                             double* __restrict__ corr) {
    __shared__ double red[32];
    const int s = blockIdx.x, s1 = s / L, s2 = s - s1 * L;
    double acc = 0.0;
    for (int p = threadIdx.x; p < L * L; p += blockDim.x) {
        const int p1 = p / L, p2 = p - p1 * L;
        const int q1 = p1 - s1 < 0 ? p1 - s1 + L : p1 - s1, q2 = p2 - s2 < 0 ? p2 - s2 + L : p2 - s2;
        acc = fma(xhat[q1 * L + q2], xref[p], acc);
    }
    acc = block_sum(acc, red);
    if (threadIdx.x == 0) corr[s] = acc;
}
cudaError_t launch_shift_corr(srmra_ctx* c, const double* xref_dev, double* corr_dev) {
    k_shift_corr<<<c->L2, 256, 0, c->stream>>>(c->d_x64, xref_dev, c->L, corr_dev);
    return cudaGetLastError();
}

}  // namespace srmra
