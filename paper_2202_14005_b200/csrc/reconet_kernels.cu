// Device kernels of the reconet driver (reconet.cpp).
#include "kernels.h"

#include <algorithm>

namespace mdnn {

namespace {

// one CTA per line y: any nonzero over (x, everything outside x/y)
__global__ void k_estimate_pattern(float2* p, const float2* __restrict__ k, long X, long Y, long rest)
{
    MDNN_PDL_ENTRY();
    const long y = blockIdx.x;
    int any = 0;
    for (long r = 0; r < rest && !any; r++)
        for (long x = threadIdx.x; x < X; x += blockDim.x) {
            const float2 v = k[x + X * (y + Y * r)];
            any |= (v.x != 0.f || v.y != 0.f);
        }
    any = __syncthreads_or(any);
    if (threadIdx.x == 0)
        p[y] = float2{any ? 1.f : 0.f, 0.f};
}

// md_zmax_abs per item (recon.hpp:472): one CTA per item, exact max of |v|
// computed in double (order-independent: max is exact)
__global__ void k_item_maxabs(double* out, const float2* __restrict__ x, long per)
{
    MDNN_PDL_ENTRY();
    const long b = blockIdx.x;
    double m = 0;
    for (long i = threadIdx.x; i < per; i += blockDim.x) {
        const float2 v = x[b * per + i];
        m = fmax(m, sqrt(double(v.x) * v.x + double(v.y) * v.y));
    }
    __shared__ double s[256];
    s[threadIdx.x] = m;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            s[threadIdx.x] = fmax(s[threadIdx.x], s[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0)
        out[b] = s[0];
}

// out = in * scale[item] (or / scale): md_mul2 with the per-item broadcast
__global__ void k_scale_items(float2* out, const float2* __restrict__ in, const float2* __restrict__ s, long per,
                              long n, bool invert)
{
    MDNN_PDL_ENTRY();
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < per * n; i += long(gridDim.x) * blockDim.x) {
        float2 sv = s[i / per];
        if (invert) { // complex reciprocal of a real scale
            const float d = sv.x * sv.x + sv.y * sv.y;
            sv = float2{sv.x / d, -sv.y / d};
        }
        const float2 v = in[i];
        out[i] = float2{v.x * sv.x - v.y * sv.y, v.x * sv.y + v.y * sv.x};
    }
}

} // namespace

void launch_estimate_pattern(cfloat* pattern, const cfloat* kspace, long X, long Y, long rest)
{
    pdl_launch(k_estimate_pattern, unsigned(Y), 256, 0, ctx().stream, pattern, kspace, X, Y, rest);
    KERNEL_CHECK();
}

void launch_item_maxabs(double* out, const cfloat* x, long per_item, long items)
{
    pdl_launch(k_item_maxabs, unsigned(items), 256, 0, ctx().stream, out, x, per_item);
    KERNEL_CHECK();
}

void launch_scale_items(cfloat* out, const cfloat* in, const cfloat* scale, long per_item, long items, bool invert)
{
    const long n = per_item * items;
    pdl_launch(k_scale_items, int(std::min<long>((n + 255) / 256, 4096)), 256, 0, ctx().stream, out, in, scale, per_item, items,
                                                                                       invert);
    KERNEL_CHECK();
}

} // namespace mdnn
