// Throughput probe: FFMA vs FFMA2 (fma.rn.f32x2) vs FADD vs FADD2, 3-register forms,
// 8 independent chains per thread, full occupancy.  Prints Gop/s (lane-ops).
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ uint64_t pk(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(uint64_t v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a + b; }
template<int MODE>
__global__ void k(float* out, int iters, float s)
{
    float a[8]; uint64_t p[8];
    float m = s * threadIdx.x, n = 1.0001f + s;
    uint64_t m2 = pk(m, m + 1.f), n2 = pk(n, n * 1.1f);
#pragma unroll
    for (int i = 0; i < 8; i++) { a[i] = i * s; p[i] = pk(i * s, i * s + 1.f); }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (MODE == 0) a[i] = fmaf(a[i], n, m);
            if (MODE == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(n2), "l"(m2));
            if (MODE == 2) a[i] = a[i] + m;
            if (MODE == 3) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(m2));
            if (MODE == 4) a[i] = a[i] * n;
            if (MODE == 5) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(n2));
            if (MODE == 6) { uint64_t b = pk(a[i & 3], a[i & 3]); asm volatile("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(p[i]) : "l"(b), "l"(m2)); }
        }
    }
    float t = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) t += a[i] + lo(p[i]);
    if (t == 12345.f) out[0] = t;
}
int main()
{
    float* o; cudaMalloc(&o, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 20000, blocks = sms * 8, threads = 256;
    const char* names[] = {"FFMA", "FFMA2", "FADD", "FADD2", "FMUL", "FMUL2", "FFMA2b"};
    for (int mode = 0; mode < 7; mode++) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            switch (mode) {
            case 0: k<0><<<blocks, threads>>>(o, iters, 1e-7f); break;
            case 1: k<1><<<blocks, threads>>>(o, iters, 1e-7f); break;
            case 2: k<2><<<blocks, threads>>>(o, iters, 1e-7f); break;
            case 3: k<3><<<blocks, threads>>>(o, iters, 1e-7f); break;
            case 4: k<4><<<blocks, threads>>>(o, iters, 1e-7f); break;
            case 5: k<5><<<blocks, threads>>>(o, iters, 1e-7f); break;
            case 6: k<6><<<blocks, threads>>>(o, iters, 1e-7f); break;
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double lanes = (mode & 1) || mode == 6 ? 2.0 : 1.0;
        const double instr = double(blocks) * threads / 32 * iters * 8;
        printf("%-6s %8.3f ms  warp-instr/clk/SM-equiv: %.3f  lane-ops %.1f Gop/s\n", names[mode], ms,
               instr / (ms * 1e-3) / sms / 1.9e9, instr * 32 * lanes / (ms * 1e-3) / 1e9);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
