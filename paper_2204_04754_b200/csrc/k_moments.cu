// k_moments.cu — NEXT-2: the empirical moments of the projected method of moments (Algorithm 1,
// PAPER.md:359-374), eq:empiric_MOM with D = 2:
//     M1 = (1/N) sum_i vec(y_i),   M2 = (1/N) sum_i vec(y_i) vec(y_i)^T = Y^T Y / N.
// M2 is a dense contraction over the observations, so it runs on the tensor cores: Y^T (L_low^2 rows,
// observations along K) split into tf32 hi / lo, with an all-ones row appended, is multiplied by itself
// in the TMA-fed 3xTF32 tcgen05 GEMM of k_gemm_tma.cu; the all-ones row gives N M1 in the same pass.
// With world > 1 the float64 sums are all-reduced over NCCL before the division by the global N.
#include <math.h>

#include <algorithm>

#include "srmra_internal.cuh"
#include "tcgen05.cuh"

namespace srmra {


namespace momk {


// yt[h][k][i] (h = tf32 hi / lo): y_i[k] for k < Ll2, 1 for k = Ll2 (i < n), 0 otherwise; ldw >= n
__global__ void k_mom_yt(const float* __restrict__ y, int64_t n, int Ll2, int R, int64_t ldw, float* __restrict__ yt) {
    __shared__ float tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32;
    const int k0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int r = ty; r < 32; r += 8) {  // coalesced along k
        const int64_t i = i0 + r;
        const int k = k0 + tx;
        tile[r][tx] = (i < n && k < Ll2) ? y[i * Ll2 + k] : (i < n && k == Ll2 ? 1.f : 0.f);
    }
    __syncthreads();
    const size_t plane = (size_t)R * ldw;
    for (int r = ty; r < 32; r += 8) {  // coalesced along i
        const int k = k0 + r;
        const int64_t i = i0 + tx;
        if (k < R && i < ldw) {
            float hi, lo;
            tc::split_tf32(tile[tx][r], hi, lo);
            yt[(size_t)k * ldw + i] = hi;
            yt[plane + (size_t)k * ldw + i] = lo;
        }
    }
}

// raw float64 sums: out[0 .. Ll2) = sum_i y_i (the all-ones column), out[Ll2 + a Ll2 + b] = sum_i y_i[a] y_i[b].
// C holds the 128 x 128 tiles with column tile >= row tile (the symmetric GEMM skips the others); inside a
// diagonal tile the two triangles (same products, different accumulation order) are averaged.
__global__ void k_mom_out(const double* __restrict__ C, int ldc, int Ll2, double* __restrict__ out) {
    const int64_t total = (int64_t)Ll2 + (int64_t)Ll2 * Ll2;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        if (e < Ll2) {
            out[e] = C[(size_t)e * ldc + Ll2];
        } else {
            const int64_t f = e - Ll2;
            const int a = (int)(f / Ll2), b = (int)(f - (int64_t)a * Ll2);
            const int i = min(a, b), j = max(a, b);
            out[e] = (i >> 7) == (j >> 7) ? 0.5 * (C[(size_t)i * ldc + j] + C[(size_t)j * ldc + i]) : C[(size_t)i * ldc + j];
        }
    }
}

}  // namespace momk

using namespace momk;

__global__ void k_mom_scale(double* __restrict__ out, int64_t total, double inv) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
        out[e] *= inv;
}

// The moments over all ranks on the device: out[0 .. Ll2) = M1, out[Ll2 ..) = M2 (row-major), float64.
// Enqueued on the context stream (temporaries stream-ordered); returns a CUDA or NCCL error code.
int moments_dev(srmra_ctx* c, double* out, std::string& err) {
    const int Ll2 = c->Ll2, R = (Ll2 + 1 + 15) / 16 * 16;  // + the all-ones row; 16-aligned rows
    const int64_t n = c->n_local, ldw = std::max<int64_t>(8, (n + 7) / 8 * 8);
    const size_t nout = (size_t)Ll2 + (size_t)Ll2 * Ll2;
    float* yt = nullptr;
    double* C = nullptr;
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double) * nout, c->stream);
    if (e == cudaSuccess && n > 0) {
        e = cudaMallocAsync(&yt, sizeof(float) * 2 * (size_t)R * ldw, c->stream);
        if (e == cudaSuccess) e = cudaMallocAsync(&C, sizeof(double) * (size_t)R * R, c->stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(C, 0, sizeof(double) * (size_t)R * R, c->stream);
        if (e == cudaSuccess) {
            dim3 grid((unsigned)((ldw + 31) / 32), (unsigned)((R + 31) / 32));
            k_mom_yt<<<grid, 256, 0, c->stream>>>(c->d_y, n, Ll2, R, ldw, yt);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess)
            // float64-accumulating tensor-core SYRK: float32 TMEM chains of 48 MMA accumulations drained into
            // float64 registers; the K range sliced over ~2 waves of CTAs (float64 atomics); upper tiles only
            e = launch_gemm_tma_acc64(yt, yt + (size_t)R * ldw, R, ldw, yt, yt + (size_t)R * ldw, R, ldw, R, ldw, C, R, 1,
                                      c->num_sms, c->stream);
        if (e == cudaSuccess) {
            k_mom_out<<<(unsigned)std::min<int64_t>(((int64_t)nout + 255) / 256, 4096), 256, 0, c->stream>>>(C, R, Ll2, out);
            e = cudaGetLastError();
        }
    }
    if (yt) cudaFreeAsync(yt, c->stream);
    if (C) cudaFreeAsync(C, c->stream);
    if (e != cudaSuccess) {
        err = std::string("moments: ") + cudaGetErrorString(e);
        return SRMRA_ERR_CUDA;
    }
    const int rc = allreduce_doubles(c, out, nout);
    if (rc != SRMRA_OK) return rc;
    const double inv = c->n_global > 0 ? 1.0 / (double)c->n_global : 0.0;
    k_mom_scale<<<(unsigned)std::min<int64_t>(((int64_t)nout + 255) / 256, 4096), 256, 0, c->stream>>>(out, (int64_t)nout, inv);
    e = cudaGetLastError();
    if (e != cudaSuccess) {
        err = std::string("moments: ") + cudaGetErrorString(e);
        return SRMRA_ERR_CUDA;
    }
    return SRMRA_OK;
}

// srmra_moments: the moments copied to caller-owned host buffers (see srmra.h).
int moments(srmra_ctx* c, double* m1, double* m2, std::string& err) {
    const int Ll2 = c->Ll2;
    const size_t nout = (size_t)Ll2 + (size_t)Ll2 * Ll2;
    double* out = nullptr;
    cudaError_t e = cudaMallocAsync(&out, sizeof(double) * nout, c->stream);
    if (e != cudaSuccess) {
        err = std::string("srmra_moments: ") + cudaGetErrorString(e);
        return SRMRA_ERR_CUDA;
    }
    int rc = moments_dev(c, out, err);
    if (rc == SRMRA_OK) {
        if (m1) e = cudaMemcpyAsync(m1, out, sizeof(double) * Ll2, cudaMemcpyDeviceToHost, c->stream);
        if (e == cudaSuccess && m2)
            e = cudaMemcpyAsync(m2, out + Ll2, sizeof(double) * Ll2 * Ll2, cudaMemcpyDeviceToHost, c->stream);
    }
    cudaFreeAsync(out, c->stream);
    const cudaError_t es = cudaStreamSynchronize(c->stream);
    if (e == cudaSuccess) e = es;
    if (rc == SRMRA_OK && e != cudaSuccess) {
        err = std::string("srmra_moments: ") + cudaGetErrorString(e);
        rc = SRMRA_ERR_CUDA;
    }
    return rc;
}

}  // namespace srmra
