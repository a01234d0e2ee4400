// k_fft_aux.cu — init-time kernel of the FFT path: Yhat_i = rfft2(y_i) for every observation of the
// shard, in float64, stored as float32.  The per-iteration small kernels live in
// k_fft_tail.cu.
#include <math.h>

#include "dft64.cuh"
#include "srmra_internal.cuh"

namespace srmra {

int ystride_of(int Ll);
int yrow_of(int Ll);

namespace fftaux {
using namespace dft64;

__global__ void k_fft_init(const float* __restrict__ y, int64_t n, int Ll, int yrow, int ystride,
                           const double* __restrict__ tw, float2* __restrict__ yhat, double* __restrict__ ysum) {
    __shared__ double scratch[32];
    extern __shared__ double sm[];
    const int Lh = Ll / 2 + 1;
    double* cs = sm;
    double* sn = cs + Ll;
    double2* tmp = reinterpret_cast<double2*>(sn + Ll);                 // [Ll][Lh]
    float* src = reinterpret_cast<float*>(tmp + (size_t)Ll * Lh);      // [Ll][Ll] (float32 input: exact)
    load_tw(tw, cs, sn, Ll);
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        double s = 0.0;
        for (int k = threadIdx.x; k < Ll * Ll; k += blockDim.x) {
            const float v = y[i * Ll * Ll + k];
            src[k] = v;
            s += (double)v;
        }
        s = block_sum(s, scratch);  // (synchronises)
        if (threadIdx.x == 0) ysum[i] = s;
        float2* out = yhat + i * ystride;
        dft2_real_fwd(src, tmp, cs, sn, Ll, 1.0, out, yrow);
        // zero the row padding and the tail pad (never read by the kernels; kept deterministic)
        for (int k = threadIdx.x; k < ystride; k += blockDim.x) {
            const int k1 = k / yrow, k2 = k - k1 * yrow;
            if (k1 >= Ll || k2 >= Lh) out[k] = make_float2(0.f, 0.f);
        }
        __syncthreads();
    }
}

}  // namespace fftaux

using namespace fftaux;

static size_t dft_smem(int Ll) {
    return sizeof(double) * 2 * Ll + sizeof(double2) * Ll * (Ll / 2 + 1) + sizeof(float) * Ll * Ll;
}

cudaError_t launch_fft_init(srmra_ctx* c, int64_t first, int64_t count) {
    if (count <= 0) return cudaSuccess;
    const size_t sm = dft_smem(c->Ll);
    cudaError_t e = cudaFuncSetAttribute(k_fft_init, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    const int64_t grid = count < 65536 ? count : 65536;
    const int ys = ystride_of(c->Ll);
    k_fft_init<<<(unsigned)grid, 256, sm, c->stream>>>(c->d_y + first * c->Ll2, count, c->Ll, yrow_of(c->Ll), ys,
                                                         c->d_tw, c->d_yhat + first * ys, c->d_ysum + first);
    return cudaGetLastError();
}

}  // namespace srmra
