// k_direct.cu — direct SIMT E-step + M-step (path SRMRA_PATH_DIRECT), for small shapes
// (L_high^2 <= 4096).  One CTA per group of observations, everything staged in shared memory.
//
//   E-step scores  S[i,s] = <y_i, P R_s x> = sum_n y_i[n] x[(n1 K - s1) mod L, (n2 K - s2) mod L]
//                  (PAPER.md:37-38 index form; the residual ||y||^2 + E_r - 2 S of eq:likelihood_EM)
//   posterior      w^{i,s} = exp(ell[s] - lse_i)  (eq:weights_EM), see k_common.cu for v[s]
//   M-step         b[p] += sum_n y_i[n] w^{i,(nK - p) mod L}   (eq:x_EM with P^{-1} := P^T:
//                  pixel p is sampled at low-res index n under exactly one shift s = nK - p)
//                  colsum[s] += w^{i,s}                     (eq:rho_EM numerator)
// The per-CTA partial b / colsum are kept in shared memory in float32 across the CTA's
// observations and added to the global float64 accumulators once at the end.
#include <math.h>

#include "srmra_internal.cuh"

namespace srmra {

constexpr int kDirectThreads = 256;

bool direct_supported(int L, int Ll, int K) { return L * L <= 4096 && L >= 2 && Ll >= 1; }

__global__ void __launch_bounds__(kDirectThreads)
k_direct_em(const float* __restrict__ y, const double* __restrict__ ynorm, int64_t n,
            const float* __restrict__ x32, const float* __restrict__ par32,
            const double* __restrict__ par64, int L, int K, float inv_s2f, double inv_s2,
            double inv_2s2, double* __restrict__ b_out, double* __restrict__ colsum_out,
            double* __restrict__ ll_out, double* __restrict__ llobs, const float* __restrict__ lrj) {
    extern __shared__ float smem[];
    const int Ll = L / K, L2 = L * L, Ll2 = Ll * Ll, KK = K * K;
    float* xs = smem;           // [L2]
    float* ys = xs + L2;        // [Ll2]
    float* sc = ys + Ll2;       // [L2]  scores -> v -> w
    float* bacc = sc + L2;      // [L2]
    float* cacc = bacc + L2;    // [L2]
    float* lr1 = cacc + L2;     // [L]
    float* lr2 = lr1 + L;       // [L]
    float* beta = lr2 + L;      // [KK]
    __shared__ float redf[32];
    __shared__ double redd[32];

    const int tid = threadIdx.x;
    for (int k = tid; k < L2; k += blockDim.x) {
        xs[k] = x32[k];
        bacc[k] = 0.f;
        cacc[k] = 0.f;
    }
    for (int k = tid; k < 2 * L + KK; k += blockDim.x) lr1[k] = par32[k];
    const double emin = par64[KK];
    double ll_acc = 0.0;
    __syncthreads();

    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        for (int k = tid; k < Ll2; k += blockDim.x) ys[k] = y[i * Ll2 + k];
        __syncthreads();
        // ---- E-step scores and row reference Sref = max_s S
        float lmax = -INFINITY;
        for (int s = tid; s < L2; s += blockDim.x) {
            const int s1 = s / L, s2 = s - s1 * L;
            const int c0 = s2 == 0 ? 0 : L - s2;
            int row = s1 == 0 ? 0 : L - s1;
            float acc = 0.f;
            for (int n1 = 0; n1 < Ll; ++n1) {
                const float* xr = xs + row * L;
                const float* yr = ys + n1 * Ll;
                int col = c0;
                for (int n2 = 0; n2 < Ll; ++n2) {
                    acc = fmaf(yr[n2], xr[col], acc);
                    col += K;
                    if (col >= L) col -= L;
                }
                row += K;
                if (row >= L) row -= L;
            }
            sc[s] = acc;
            lmax = fmaxf(lmax, acc);
        }
        const float sref = block_max(lmax, redf, -INFINITY);
        // ---- v[s] and its max
        float vmax = -INFINITY;
        for (int s = tid; s < L2; s += blockDim.x) {
            const int s1 = s / L, s2 = s - s1 * L;
            const float v = (sc[s] - sref) * inv_s2f + lr1[s1] + lr2[s2] + beta[(s1 % K) * K + (s2 % K)] +
                            (lrj ? __ldg(lrj + s) : 0.f);  // joint log prior (NEXT-3)
            sc[s] = v;
            vmax = fmaxf(vmax, v);
        }
        const float m = block_max(vmax, redf, -INFINITY);
        // ---- e = exp(v - m), Z = sum e
        float zs = 0.f;
        for (int s = tid; s < L2; s += blockDim.x) {
            const float e = expf(sc[s] - m);
            sc[s] = e;
            zs += e;
        }
        const double Z = block_sum((double)zs, redd);
        const float invZ = (float)(1.0 / Z);
        for (int s = tid; s < L2; s += blockDim.x) {
            const float w = sc[s] * invZ;
            sc[s] = w;
            cacc[s] += w;
        }
        if (tid == 0) {
            const double lse = (double)sref * inv_s2 + (double)m + log(Z) - (emin + ynorm[i]) * inv_2s2;
            ll_acc += lse;
            if (llobs) llobs[i] = lse;
        }
        __syncthreads();
        // ---- M-step: b[p] += sum_n y[n] w[(nK - p) mod L]
        for (int p = tid; p < L2; p += blockDim.x) {
            const int p1 = p / L, p2 = p - p1 * L;
            const int c0 = p2 == 0 ? 0 : L - p2;
            int row = p1 == 0 ? 0 : L - p1;
            float acc = 0.f;
            for (int n1 = 0; n1 < Ll; ++n1) {
                const float* wr = sc + row * L;
                const float* yr = ys + n1 * Ll;
                int col = c0;
                for (int n2 = 0; n2 < Ll; ++n2) {
                    acc = fmaf(yr[n2], wr[col], acc);
                    col += K;
                    if (col >= L) col -= L;
                }
                row += K;
                if (row >= L) row -= L;
            }
            bacc[p] += acc;
        }
        __syncthreads();
    }
    for (int k = tid; k < L2; k += blockDim.x) {
        atomicAdd(&b_out[k], (double)bacc[k]);
        atomicAdd(&colsum_out[k], (double)cacc[k]);
    }
    if (tid == 0) atomicAdd(ll_out, ll_acc);
}

cudaError_t launch_direct_em(srmra_ctx* c) {
    if (c->n_local == 0) return cudaSuccess;
    const size_t smem = sizeof(float) * (4 * (size_t)c->L2 + c->Ll2 + 2 * c->L + c->KK);
    static PerDeviceOnce attr;
    cudaError_t ea = attr.run([] { return cudaFuncSetAttribute(k_direct_em, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024); });
    if (ea != cudaSuccess) return ea;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_direct_em, kDirectThreads, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)c->num_sms * per_sm;
    if (grid > c->n_local) grid = c->n_local;
    k_direct_em<<<(unsigned)grid, kDirectThreads, smem, c->stream>>>(
        c->d_y, c->d_ynorm, c->n_local, c->d_x32, c->par.f32, c->par.f64, c->L, c->K, (float)c->inv_s2,
        c->inv_s2, c->inv_2s2, c->d_pack + c->pk.b, c->d_colsum, c->d_pack + c->pk.ll, c->d_llobs,
        c->joint ? c->d_lrj : nullptr);
    return cudaGetLastError();
}

}  // namespace srmra
