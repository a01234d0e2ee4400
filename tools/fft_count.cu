// FP32 instruction counts of the register FFT variants (regfft.cuh) — compile only, no GPU:
//   for D in "" -DR4 -DSR; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//     --expt-relaxed-constexpr $D -cubin -o /tmp/fc.cubin tools/fft_count.cu && cuobjdump -sass /tmp/fc.cubin \
//     | grep -cE "FADD|FFMA|FMUL"; done
#include "../paper_2204_04754_b200/csrc/regfft.cuh"
using namespace srmra::regfft;
template <int N> __global__ void kk(float2* p) {
    float2 v[N];
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = p[threadIdx.x * N + i];
#if defined(R4)
    fft_r4<N, -1>(v);
#elif defined(SR)
    fft_sr<N, -1>(v);
#elif defined(SR2)
    fft_sr2<N, -1>(v);
#else
    fft<N, -1>(v);
#endif
#pragma unroll
    for (int i = 0; i < N; ++i) p[threadIdx.x * N + i] = v[i];
}
template __global__ void kk<32>(float2*);
template __global__ void kk<64>(float2*);
