// Latency / throughput of paired fp32 (FFMA2) vs scalar FFMA on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_probe ffma2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template<int CHAINS, int PAIRED>
__global__ void k(float* out, int iters, long long* cyc)
{
    float2 a[CHAINS];
    float s[2 * CHAINS];
    for (int c = 0; c < CHAINS; c++) {
        a[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
        s[2 * c] = a[c].x;
        s[2 * c + 1] = a[c].y;
    }
    const float2 m = make_float2(0.9999f, 1.0001f), d = make_float2(1e-7f, 2e-7f);
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) {
            if constexpr (PAIRED == 1) {
                a[c] = __ffma2_rn(a[c], m, d);
            } else if constexpr (PAIRED == 2) {
                a[c] = __fadd2_rn(a[c], d);
            } else if constexpr (PAIRED == 3) {
                a[c] = __ffma2_rn(a[c], make_float2(m.x, m.x), d); // scalar-broadcast operand
            } else if constexpr (PAIRED == 4) {
                a[c] = __fmul2_rn(a[c], make_float2(0.99991f, 0.99991f)); // immediate
            } else if constexpr (PAIRED == 5) {
                s[2 * c] = s[2 * c] + d.x;
                s[2 * c + 1] = s[2 * c + 1] + d.y;
            } else {
                s[2 * c] = fmaf(s[2 * c], m.x, d.x);
                s[2 * c + 1] = fmaf(s[2 * c + 1], m.y, d.y);
            }
        }
    }
    long long t1 = clock64();
    float acc = 0.f;
    for (int c = 0; c < CHAINS; c++)
        acc += (PAIRED >= 1 && PAIRED <= 4) ? a[c].x + a[c].y : s[2 * c] + s[2 * c + 1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0)
        *cyc = t1 - t0;
}

template<int CHAINS, int PAIRED>
void run(int warps)
{
    float* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 8);
    const int iters = 4096;
    k<CHAINS, PAIRED><<<1, 32 * warps>>>(out, iters, cyc);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    // per warp instruction count: iters * CHAINS (paired) or 2 * iters * CHAINS (scalar)
    const bool pr = PAIRED >= 1 && PAIRED <= 4;
    const double ninst = double(iters) * CHAINS * (pr ? 1 : 2);
    const char* nm[] = {"FFMA ", "FFMA2", "FADD2", "FFMA2b", "FMUL2i", "FADD "};
    printf("%s chains %2d warps %2d: %.2f cycles per instr per warp, fp32 lane-ops/clk/SM %.1f\n",
           nm[PAIRED], CHAINS, warps, double(h) / ninst,
           double(iters) * CHAINS * 2 * 32 * warps / double(h));
    cudaFree(out);
    cudaFree(cyc);
}

int main()
{
    run<8, 0>(1); run<8, 1>(1); run<8, 2>(1); run<8, 3>(1); run<8, 4>(1); run<8, 5>(1);
    run<8, 0>(8); run<8, 1>(8); run<8, 2>(8); run<8, 3>(8); run<8, 4>(8); run<8, 5>(8);
    run<16, 1>(1); run<16, 2>(1); run<16, 0>(1);
    return 0;
}
