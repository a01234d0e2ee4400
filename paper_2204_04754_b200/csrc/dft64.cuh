// dft64.cuh — small float64 DFT helpers (power-of-two L_low, masked twiddle index, host twiddle table)
// shared by the init-time rfft2 of the observations and the per-iteration tail kernel.
#pragma once
#include "srmra_internal.cuh"

namespace srmra {
namespace dft64 {

// forward real 2-D DFT of the Ll x Ll image `src` (smem, float64) -> half spectrum `out` (float32),
// scaled; `tmp` holds Ll x Lh complex; cs/sn: cos/sin(2 pi j / Ll), j < Ll.
// out row stride `orow` (>= Lh) float2; src may be float (exact for float32 data) or double.
template <typename T>
__device__ inline void dft2_real_fwd(const T* src, double2* tmp, const double* cs, const double* sn, int Ll,
                                     double scale, float2* out, int orow) {
    const int Lh = Ll / 2 + 1, M = Ll - 1;
    for (int e = threadIdx.x; e < Ll * Lh; e += blockDim.x) {  // along n2: tmp[n1][k2]
        const int n1 = e / Lh, k2 = e - n1 * Lh;
        const T* row = src + n1 * Ll;
        double re = 0, im = 0;
        for (int n2 = 0; n2 < Ll; ++n2) {
            const int j = (k2 * n2) & M;
            const double xv = (double)row[n2];
            re = fma(xv, cs[j], re);
            im = fma(-xv, sn[j], im);
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
        out[(size_t)k1 * orow + k2] = make_float2((float)(re * scale), (float)(im * scale));
    }
}

__device__ inline void load_tw(const double* tw, double* cs, double* sn, int Ll) {
    for (int j = threadIdx.x; j < Ll; j += blockDim.x) {
        cs[j] = tw[j];
        sn[j] = tw[Ll + j];
    }
}

}  // namespace dft64
}  // namespace srmra
