#include "../../paper_2204_04754_b200/csrc/regfft.cuh"
using namespace srmra::regfft;
__global__ void k32(float2* p) {
    float2 v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = p[threadIdx.x * 32 + i];
    fft<32, -1>(v);
#pragma unroll
    for (int i = 0; i < 32; ++i) p[threadIdx.x * 32 + i] = v[i];
}
