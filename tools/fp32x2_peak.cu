// FP32 FMA vs packed FFMA2 (fma.rn.f32x2) throughput on sm_100a: 8 independent chains per thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp32x2_peak tools/fp32x2_peak.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__global__ void k_ffma(float* out, int iters, float a, float b) {
    float x[8];
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, b);
    float s = 0;
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.f) out[0] = s;
}
__global__ void k_ffma2(float* out, int iters, float a, float b) {
    uint64_t x[8];
    uint64_t A, B;
    asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
    asm("mov.b64 %0, {%1, %1};" : "=l"(B) : "f"(b));
    for (int j = 0; j < 8; ++j) {
        float v = threadIdx.x * 1e-3f + j;
        asm("mov.b64 %0, {%1, %1};" : "=l"(x[j]) : "f"(v));
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma2(x[j], A, B);
    float s = 0;
    for (int j = 0; j < 8; ++j) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[j]));
        s += lo + hi;
    }
    if (s == 12345.f) out[0] = s;
}
int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    float* d;
    cudaMalloc(&d, 8);
    const int blocks = p.multiProcessorCount * 4, threads = 256, iters = 1 << 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int kind = 0; kind < 2; ++kind) {
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            if (kind == 0) k_ffma<<<blocks, threads>>>(d, iters, 0.999999f, 1e-9f);
            else k_ffma2<<<blocks, threads>>>(d, iters, 0.999999f, 1e-9f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 0 && ms < best) best = ms;
        }
        const double fmas = (double)blocks * threads * iters * 8 * (kind ? 2 : 1);
        printf("{\"kind\": \"%s\", \"fp32_tflops\": %.2f, \"ms\": %.3f}\n", kind ? "ffma2" : "ffma",
               2 * fmas / (best * 1e-3) / 1e12, best);
    }
    return 0;
}
