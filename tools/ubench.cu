// Per-SM instruction throughputs on B200 (sm_100a) that bound the FFT-path E/M kernels:
// FFMA, FADD, FFMA2 / FADD2 (packed FP32x2), SHFL, LDS.64 / LDS.128 / STS.64, MUFU.EX2, and the FP32
// peak they imply.  Each kernel runs 8 independent chains per thread at full occupancy; the result is
// warp-instructions per clock per SM (clock from the measured SM clock, nvidia-smi style, via clock64
// over the same loop) and, for the FP32 kinds, TFLOP/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench tools/ubench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t pk(float v) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(v));
    return r;
}
__device__ __forceinline__ float upk(uint64_t v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return lo + hi;
}

enum { FFMA, FADD, FFMA2, FADD2, SHFL, LDS64, LDS128, STS64, EX2, NKIND };
static const char* NAMES[NKIND] = {"ffma", "fadd", "ffma2", "fadd2", "shfl", "lds64", "lds128", "sts64", "mufu_ex2"};

template <int KIND>
__global__ void k_bench(float* out, int iters, float a, float b, unsigned long long* clk) {
    __shared__ float4 sm[1024];
    const int t = threadIdx.x;
    for (int k = t; k < 1024; k += blockDim.x) sm[k] = make_float4(k, k + 1, k + 2, k + 3);
    __syncthreads();
    unsigned long long c0 = clock64();
    float s = 0.f;
    if (KIND == FFMA || KIND == FADD || KIND == EX2) {
        float x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = t * 1e-3f + j;
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (KIND == FFMA) x[j] = fmaf(x[j], a, b);
                else if (KIND == FADD) x[j] = x[j] + b;
                else asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[j]));
            }
#pragma unroll
        for (int j = 0; j < 8; ++j) s += x[j];
    } else if (KIND == FFMA2 || KIND == FADD2) {
        uint64_t x[8], A = pk(a), B = pk(b);
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = pk(t * 1e-3f + j);
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = KIND == FFMA2 ? fma2(x[j], A, B) : add2(x[j], B);
#pragma unroll
        for (int j = 0; j < 8; ++j) s += upk(x[j]);
    } else if (KIND == SHFL) {
        float x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = t * 1e-3f + j;
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = __shfl_xor_sync(0xffffffffu, x[j], 1 + (j & 3));
#pragma unroll
        for (int j = 0; j < 8; ++j) s += x[j];
    } else if (KIND == LDS64 || KIND == LDS128) {
        // conflict-free: lane l reads consecutive 8 / 16-byte words
        const float2* s2 = reinterpret_cast<const float2*>(sm);
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int base = t & 31;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (KIND == LDS64) {
                    const float2 v = s2[(base + 64 * j + (i & 1) * 32) & 2047];
                    acc[j] += v.x;
                } else {
                    const float4 v = sm[(base + 32 * j + (i & 1) * 32) & 1023];
                    acc[j] += v.x;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) s += acc[j];
    } else if (KIND == STS64) {
        float2* s2 = reinterpret_cast<float2*>(sm);
        const int base = t & 31;
        const int w = (t >> 5) & 7;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 8; ++j) s2[(base + 32 * j + 256 * w) & 2047] = make_float2(i, j);
        }
        __syncthreads();
        s = s2[t & 2047].x;
    }
    unsigned long long c1 = clock64();
    if (t == 0 && blockIdx.x == 0) clk[0] = c1 - c0;
    if (s == 12345.f) out[0] = s;
}

template <int KIND>
double run(int blocks, int threads, int iters, float* d, unsigned long long* clk, double* per_clk) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    unsigned long long cyc = 0;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_bench<KIND><<<blocks, threads>>>(d, iters, 0.999999f, 1e-9f, clk);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) {
            best = ms;
            cudaMemcpy(&cyc, clk, 8, cudaMemcpyDeviceToHost);
        }
    }
    // warp-instructions per SM per clock: blocks/SM * warps/block * iters * 8 over the kernel's cycles
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const double warp_instr = (double)blocks * threads / 32 * iters * 8;
    *per_clk = warp_instr / p.multiProcessorCount / (double)cyc;
    return best;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    float* d;
    unsigned long long* clk;
    cudaMalloc(&d, 8);
    cudaMalloc(&clk, 8);
    const int blocks = p.multiProcessorCount * 4, threads = 256, iters = 1 << 14;
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"results\": [\n", p.name, p.multiProcessorCount);
    for (int k = 0; k < NKIND; ++k) {
        double pc = 0, ms = 0;
        switch (k) {
            case FFMA: ms = run<FFMA>(blocks, threads, iters, d, clk, &pc); break;
            case FADD: ms = run<FADD>(blocks, threads, iters, d, clk, &pc); break;
            case FFMA2: ms = run<FFMA2>(blocks, threads, iters, d, clk, &pc); break;
            case FADD2: ms = run<FADD2>(blocks, threads, iters, d, clk, &pc); break;
            case SHFL: ms = run<SHFL>(blocks, threads, iters, d, clk, &pc); break;
            case LDS64: ms = run<LDS64>(blocks, threads, iters, d, clk, &pc); break;
            case LDS128: ms = run<LDS128>(blocks, threads, iters, d, clk, &pc); break;
            case STS64: ms = run<STS64>(blocks, threads, iters, d, clk, &pc); break;
            case EX2: ms = run<EX2>(blocks, threads, iters, d, clk, &pc); break;
        }
        const double ops = (double)blocks * threads * iters * 8;
        const double lanes_flop = (k == FFMA) ? 2 : (k == FADD) ? 1 : (k == FFMA2) ? 4 : (k == FADD2) ? 2 : 0;
        printf("  {\"kind\": \"%s\", \"warp_instr_per_clk_per_sm\": %.3f, \"ms\": %.3f, \"fp32_tflops\": %.2f}%s\n",
               NAMES[k], pc, ms, lanes_flop * ops / (ms * 1e-3) / 1e12, k + 1 < NKIND ? "," : "");
    }
    printf("]}\n");
    return 0;
}
