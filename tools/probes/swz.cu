#include <stdint.h>
__device__ __forceinline__ uint64_t pk(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void upk(uint64_t v, float& a, float& b) { asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) { uint64_t d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
// complex multiply z*w with z, w as (re, im) pairs
__global__ void cm(const float2* __restrict__ z, const float2* __restrict__ w, float2* o, int n)
{
    int i = threadIdx.x + blockIdx.x * blockDim.x;
    float2 a = z[i], b = w[i];
    uint64_t t = mul2(pk(a.x, a.x), pk(b.x, b.y));
    uint64_t d = fma2(pk(a.y, a.y), pk(-b.y, b.x), t);
    float r0, r1; upk(d, r0, r1);
    o[i] = make_float2(r0, r1);
}
