#include <cstdint>
__device__ __forceinline__ uint64_t pk(float x, float y) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r; }
__device__ __forceinline__ float2 upk(uint64_t r) { float2 v; asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r)); return v; }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) { uint64_t d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) { uint64_t d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) { uint64_t d; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__global__ void k(float2* p, float c, float s) {
    float2 a = p[threadIdx.x], b = p[threadIdx.x + 32];
    // bw = b * (c + i s): (bx c - by s, bx s + by c) = bx*(c, s) + by*(-s, c)
    uint64_t bw = fma2(pk(b.y, b.y), pk(-s, c), mul2(pk(b.x, b.x), pk(c, s)));
    uint64_t A = pk(a.x, a.y);
    p[threadIdx.x + 64] = upk(add2(A, bw));
    p[threadIdx.x + 96] = upk(sub2(A, bw));
}
