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

// L_low >= 32: the same rfft2 as a float64 radix-2 FFT in shared memory (the O(L_low^3) DFT above took 630 ms for
// configs[4]'s 10^5 observations of 128 x 128).  Two real rows form one complex row z = y_2r + i y_2r+1 (loaded
// in bit-reversed order), L_low/2 in-place DIT row FFTs, the row pair separated (X_2r = (Z[k] + conj Z[-k]) / 2,
// X_2r+1 = (Z[k] - conj Z[-k]) / 2i) into T[bitrev(n1)][k2] (k2 <= L_low/2) over the same buffer, L_low/2+1 in-place
// DIT column FFTs, float32 out.  Shared memory: L_low (L_low/2 + 1) complex doubles (133 KB at 128).
__device__ __forceinline__ int brev(int i, int lg) { return (int)(__brev((unsigned)i) >> (32 - lg)); }

__global__ void __launch_bounds__(256) k_fft_init_fft(const float* __restrict__ y, int64_t n, int Ll, int lg, int yrow,
                                                      int ystride, const double* __restrict__ tw,
                                                      float2* __restrict__ yhat, double* __restrict__ ysum) {
    __shared__ double scratch[32];
    extern __shared__ double sm[];
    const int Lh = Ll / 2 + 1, H = Ll / 2, M = Ll - 1;
    double* cs = sm;
    double* sn = cs + Ll;
    double2* Z = reinterpret_cast<double2*>(sn + Ll);  // [H][Ll] then T [Ll][Lh]
    load_tw(tw, cs, sn, Ll);
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const float* yi = y + i * (int64_t)Ll * Ll;
        double s = 0.0;
        for (int k = threadIdx.x; k < H * Ll; k += blockDim.x) {  // z[r][bitrev(c)] = y[2r][c] + i y[2r+1][c]
            const int r = k / Ll, c = k - r * Ll;
            const float a = yi[(2 * r) * Ll + c], b = yi[(2 * r + 1) * Ll + c];
            s += (double)a + (double)b;
            Z[r * Ll + brev(c, lg)] = make_double2(a, b);
        }
        s = block_sum(s, scratch);  // (synchronises)
        if (threadIdx.x == 0) ysum[i] = s;
        for (int m = 1; m < Ll; m <<= 1) {  // row stages
            const int tstep = Ll / (2 * m);
            for (int b = threadIdx.x; b < H * H; b += blockDim.x) {
                const int r = b / H, j = b - r * H, pos = j & (m - 1), i0 = r * Ll + ((j - pos) << 1) + pos;
                const double c = cs[pos * tstep], sv = -sn[pos * tstep];
                const double2 u = Z[i0], v = Z[i0 + m];
                const double2 t = make_double2(v.x * c - v.y * sv, v.x * sv + v.y * c);
                Z[i0] = make_double2(u.x + t.x, u.y + t.y);
                Z[i0 + m] = make_double2(u.x - t.x, u.y - t.y);
            }
            __syncthreads();
        }
        // separate the row pairs (all reads before any write: the outputs overlay the inputs)
        constexpr int PER = (64 * 65 + 255) / 256;  // items per thread at Ll = 128 (fewer at smaller Ll)
        double2 za[PER], zb[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int k = threadIdx.x + u * 256;
            if (k < H * Lh) {
                const int r = k / Lh, k2 = k - r * Lh;
                za[u] = Z[r * Ll + k2];
                zb[u] = Z[r * Ll + ((Ll - k2) & M)];
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int k = threadIdx.x + u * 256;
            if (k >= H * Lh) continue;
            const int r = k / Lh, k2 = k - r * Lh;
            const double2 a = za[u], b = zb[u];  // Z[k], Z[-k]
            // X_2r = (Z[k] + conj Z[-k]) / 2,  X_2r+1 = (Z[k] - conj Z[-k]) / (2i)
            Z[brev(2 * r, lg) * Lh + k2] = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
            Z[brev(2 * r + 1, lg) * Lh + k2] = make_double2(0.5 * (a.y + b.y), -0.5 * (a.x - b.x));
        }
        __syncthreads();
        for (int m = 1; m < Ll; m <<= 1) {  // column stages over T [Ll][Lh] (rows in bit-reversed order)
            const int tstep = Ll / (2 * m);
            for (int b = threadIdx.x; b < H * Lh; b += blockDim.x) {
                const int c = b % Lh, j = b / Lh, pos = j & (m - 1), r0 = ((j - pos) << 1) + pos;
                const double cc = cs[pos * tstep], sv = -sn[pos * tstep];
                const double2 u = Z[r0 * Lh + c], v = Z[(r0 + m) * Lh + c];
                const double2 t = make_double2(v.x * cc - v.y * sv, v.x * sv + v.y * cc);
                Z[r0 * Lh + c] = make_double2(u.x + t.x, u.y + t.y);
                Z[(r0 + m) * Lh + c] = make_double2(u.x - t.x, u.y - t.y);
            }
            __syncthreads();
        }
        float2* out = yhat + i * ystride;
        for (int k = threadIdx.x; k < ystride; k += blockDim.x) {
            const int k1 = k / yrow, k2 = k - k1 * yrow;
            const double2 v = (k1 < Ll && k2 < Lh) ? Z[k1 * Lh + k2] : make_double2(0.0, 0.0);
            out[k] = make_float2((float)v.x, (float)v.y);
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
    if (c->Ll >= 32) {
        const int Ll = c->Ll, lg = __builtin_ctz(Ll);
        const size_t sm = sizeof(double) * 2 * Ll + sizeof(double2) * (size_t)Ll * (Ll / 2 + 1);
        static PerDeviceOnce attr;
        cudaError_t e = attr.run([] {
            return cudaFuncSetAttribute(k_fft_init_fft, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(sizeof(double) * 2 * 128 + sizeof(double2) * 128 * 65));
        });
        if (e != cudaSuccess) return e;
        const int64_t grid = count < 65536 ? count : 65536;
        const int ys = ystride_of(Ll);
        k_fft_init_fft<<<(unsigned)grid, 256, sm, c->stream>>>(c->d_y + first * c->Ll2, count, Ll, lg, yrow_of(Ll), ys,
                                                               c->d_tw, c->d_yhat + first * ys, c->d_ysum + first);
        return cudaGetLastError();
    }
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
