#include "../../paper_2204_04754_b200/csrc/regfft.cuh"
using namespace srmra::regfft;
template <int N> __global__ void kk(float2* p) {
    float2 v[N];
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = p[threadIdx.x * N + i];
#if defined(R4)
    fft_r4<N, -1>(v);
#elif defined(SR)
    fft_sr<N, -1>(v);
#else
    fft<N, -1>(v);
#endif
#pragma unroll
    for (int i = 0; i < N; ++i) p[threadIdx.x * N + i] = v[i];
}
template __global__ void kk<32>(float2*);
template __global__ void kk<64>(float2*);
