// k_synth.cu — NEXT-4's device data generator (srmra_generate): the observations of eq:model_1 in its
// explicit form, y_j[n] = x[(n1 K - s^1) mod L, (n2 K - s^2) mod L] + sigma z, drawn on the
// GPU from a counter-based generator so that large-N workloads need no host generation or transfer.
// Philox4x32-10 (Salmon et al., SC'11), keyed by the seed, counter = (global index j, block b); the
// scheme (shift inverse CDF on float64 partial sums, Box-Muller on 23-bit uniforms) is documented in
// include/srmra.h and mirrored by synth/philox.py, which the tests compare against draw by draw.
#include <math.h>

#include <algorithm>

#include "srmra_internal.cuh"

namespace srmra {
namespace synthk {

__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

// min k with U < C[k], clamped to the last k with positive mass (`last`)
__device__ __forceinline__ int inv_cdf(uint32_t u, const double* __restrict__ C, int L, int last) {
    const double U = ((double)u + 0.5) * 0x1p-32;
    int lo = 0, hi = L;  // first index with C[k] > U
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (C[mid] > U) hi = mid;
        else lo = mid + 1;
    }
    return lo < last ? lo : last;
}

// one block per observation (grid-stride); C = cumsum(rho1) | cumsum(rho2), last = last positive index per axis
__global__ void k_generate(float* __restrict__ y, int64_t n, int64_t first, const float* __restrict__ x, int L, int Ll,
                           int K, float sigma, const double* __restrict__ C, int last1, int last2, uint32_t k0,
                           uint32_t k1, int* __restrict__ shifts) {
    const int P = Ll * Ll, nb = (P + 3) / 4;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const uint64_t j = (uint64_t)(first + i);
        const uint32_t jl = (uint32_t)j, jh = (uint32_t)(j >> 32);
        const uint4 u = philox(make_uint4(jl, jh, 0u, 0u), k0, k1);
        const int s1 = inv_cdf(u.x, C, L, last1), s2 = inv_cdf(u.y, C + L, L, last2);
        if (threadIdx.x == 0 && shifts) {
            shifts[2 * i] = s1;
            shifts[2 * i + 1] = s2;
        }
        float* yi = y + i * P;
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            const uint4 r = philox(make_uint4(jl, jh, 1u + (uint32_t)b, 0u), k0, k1);
            // 23-bit uniforms: (m + 0.5) 2^-23 is exact in float32 for m < 2^23
            const float v0 = ((float)(r.x >> 9) + 0.5f) * 0x1p-23f, v1 = ((float)(r.y >> 9) + 0.5f) * 0x1p-23f;
            const float v2 = ((float)(r.z >> 9) + 0.5f) * 0x1p-23f, v3 = ((float)(r.w >> 9) + 0.5f) * 0x1p-23f;
            const float ra = sqrtf(-2.f * logf(v0)), rb = sqrtf(-2.f * logf(v2));
            float sa, ca, sb, cb;
            sincospif(2.f * v1, &sa, &ca);
            sincospif(2.f * v3, &sb, &cb);
            const float z[4] = {ra * ca, ra * sa, rb * cb, rb * sb};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int p = 4 * b + e;
                if (p < P) {
                    const int n1 = p / Ll, n2 = p - n1 * Ll;
                    const int a1 = imod(n1 * K - s1, L), a2 = imod(n2 * K - s2, L);
                    yi[p] = fmaf(sigma, z[e], x[a1 * L + a2]);
                }
            }
        }
    }
}

}  // namespace synthk

cudaError_t launch_generate(srmra_ctx* c, const float* x_dev, const double* cdf_dev, int last1, int last2,
                            uint64_t seed, int64_t first, int* shifts_dev) {
    if (c->n_local == 0) return cudaSuccess;
    const int64_t grid = std::min<int64_t>(c->n_local, (int64_t)c->num_sms * 16);
    synthk::k_generate<<<(unsigned)grid, 256, 0, c->stream>>>(c->d_y, c->n_local, first, x_dev, c->L, c->Ll, c->K,
                                                               (float)c->sigma, cdf_dev, last1, last2, (uint32_t)seed,
                                                               (uint32_t)(seed >> 32), shifts_dev);
    return cudaGetLastError();
}

}  // namespace srmra
