// Loss and optimiser kernels: MSE (MseNode, ops.hpp:874-906) and complex Adam
// (adam_step, optim.hpp:81-108; moments m complex, v = |g|^2 real).
#include "kernels.h"

#include <algorithm>

namespace mdnn {

namespace {

constexpr int kT = 256;

int grid_for(long n)
{
    long blocks = (n + kT - 1) / kT;
    return int(std::max(1L, std::min(blocks, long(ctx().sm_count) * 8)));
}

__global__ void k_diff(cfloat* __restrict__ d, const cfloat* __restrict__ p, const cfloat* __restrict__ r, long n)
{
    MDNN_PDL_ENTRY();
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        d[i] = float2{p[i].x - r[i].x, p[i].y - r[i].y};
}

__global__ void k_adam(cfloat* __restrict__ th, cfloat* __restrict__ m, float* __restrict__ v,
                       const cfloat* __restrict__ g, long n, float lr, float b1, float b2, float eps, float c1,
                       float c2, float gscale, bool real_w, bool nonneg)
{
    MDNN_PDL_ENTRY();
    for (long k = blockIdx.x * long(blockDim.x) + threadIdx.x; k < n; k += long(gridDim.x) * blockDim.x) {
        float2 gv = g[k];
        gv.x *= gscale;
        gv.y *= gscale;
        if (real_w)
            gv.y = 0.f; // realify (optim.hpp:384-385)
        float2 mv = m[k];
        // mv = b1 * mv + (1 - b1) * gv  (complex<R> arithmetic)
        mv = float2{b1 * mv.x + (1.f - b1) * gv.x, b1 * mv.y + (1.f - b1) * gv.y};
        m[k] = mv;
        float vv = b2 * v[k] + (1.f - b2) * (gv.x * gv.x + gv.y * gv.y);
        v[k] = vv;
        float denom = sqrtf(vv * c2) + eps;
        float2 t = th[k];
        t.x -= lr * (mv.x * c1) / denom;
        t.y -= lr * (mv.y * c1) / denom;
        if (real_w)
            t.y = 0.f;
        if (nonneg) // NonNegProx (nn.hpp:56-62)
            t = float2{t.x > 0.f ? t.x : 0.f, 0.f};
        th[k] = t;
    }
}

// sgd_step (optim.hpp:66-71) with run_step's clip scale, realify and prox (optim.hpp:383-396)
__global__ void k_sgd(float2* __restrict__ th, const float2* __restrict__ g, long n, float lr, float gscale,
                      bool real_w, bool nonneg)
{
    MDNN_PDL_ENTRY();
    for (long k = blockIdx.x * long(blockDim.x) + threadIdx.x; k < n; k += long(gridDim.x) * blockDim.x) {
        float2 gv = g[k];
        gv.x *= gscale;
        gv.y = real_w ? 0.f : gv.y * gscale;
        float2 t = th[k];
        t.x -= lr * gv.x;
        t.y -= lr * gv.y;
        if (real_w)
            t.y = 0.f;
        if (nonneg)
            t = float2{t.x > 0.f ? t.x : 0.f, 0.f};
        th[k] = t;
    }
}

__global__ void k_prox_nonneg(float2* w, long n)
{
    MDNN_PDL_ENTRY();
    for (long k = blockIdx.x * long(blockDim.x) + threadIdx.x; k < n; k += long(gridDim.x) * blockDim.x) {
        const float2 t = w[k];
        w[k] = float2{t.x > 0.f ? t.x : 0.f, 0.f};
    }
}

} // namespace

void sgd_update(cfloat* theta, const cfloat* g, long n, float lr, float gscale, bool real_weights, bool nonneg_prox)
{
    pdl_launch(k_sgd, grid_for(n), kT, 0, ctx().stream, theta, g, n, lr, gscale, real_weights, nonneg_prox);
    KERNEL_CHECK();
}

void launch_prox_nonneg(cfloat* w, long n)
{
    pdl_launch(k_prox_nonneg, grid_for(n), kT, 0, ctx().stream, w, n);
    KERNEL_CHECK();
}

void mse_forward(cfloat* loss, cfloat* diff, const cfloat* p, const cfloat* r, long n)
{
    pdl_launch(k_diff, grid_for(n), kT, 0, ctx().stream, diff, p, r, n);
    KERNEL_CHECK();
    launch_iso_reduce(loss, diff, diff, n, 1, 1, 2, float(1.0 / double(n)));
}

void adam_update(cfloat* theta, cfloat* m, float* v, const cfloat* g, long n, float lr, float b1, float b2,
                 float eps, float c1, float c2, float gscale, bool real_weights, bool nonneg_prox)
{
    pdl_launch(k_adam, grid_for(n), kT, 0, ctx().stream, theta, m, v, g, n, lr, b1, b2, eps, c1, c2, gscale, real_weights,
                                                 nonneg_prox);
    KERNEL_CHECK();
}

} // namespace mdnn
