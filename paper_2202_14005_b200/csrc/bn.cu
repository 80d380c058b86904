// Batch normalisation over an [inner][stat][outer] view (BatchNormNode,
// ops.hpp:1070-1298; MoDL normalises over x, y and batch per channel,
// recon.hpp:732).  Statistics use the deterministic double-accumulated ISO
// reductions of ew.cu; elementwise passes are vectorised grid-stride loops.
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

__global__ void k_sub_stat(cfloat* __restrict__ u, const cfloat* __restrict__ x, const cfloat* __restrict__ mu,
                           long inner, long nstat, long n)
{
    MDNN_PDL_ENTRY();
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        long s = (i / inner) % nstat;
        float2 v = x[i], m = mu[s];
        u[i] = float2{v.x - m.x, v.y - m.y};
    }
}

__global__ void k_stats_finish(cfloat* istd, cfloat* mean_out, cfloat* var_out, const cfloat* mean,
                               const cfloat* var, const cfloat* mean_in, const cfloat* var_in, long nstat, float eps,
                               float mom, int train)
{
    MDNN_PDL_ENTRY();
    for (long s = blockIdx.x * long(blockDim.x) + threadIdx.x; s < nstat; s += long(gridDim.x) * blockDim.x) {
        float v = var[s].x;
        istd[s] = float2{1.f / sqrtf(v + eps), 0.f};
        if (train) {
            // stat' = mom * batch + (1 - mom) * stat   (ops.hpp:1129-1132)
            float2 bm = mean[s], im = mean_in[s];
            float2 y{mom * bm.x, mom * bm.y};
            y.x += (1.f - mom) * im.x - 0.f * im.y;
            y.y += (1.f - mom) * im.y + 0.f * im.x;
            mean_out[s] = y;
            float2 bv = var[s], iv = var_in[s];
            float2 z{mom * bv.x, mom * bv.y};
            z.x += (1.f - mom) * iv.x;
            z.y += (1.f - mom) * iv.y;
            var_out[s] = z;
        }
    }
}

__global__ void k_stat_mul(cfloat* __restrict__ out, const cfloat* __restrict__ in, const cfloat* __restrict__ s,
                           long inner, long nstat, long n, bool cj)
{
    MDNN_PDL_ENTRY();
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        float2 v = in[i], w = s[(i / inner) % nstat];
        if (cj)
            w.y = -w.y;
        out[i] = float2{v.x * w.x - v.y * w.y, v.x * w.y + v.y * w.x};
    }
}

__global__ void k_stat_add(cfloat* __restrict__ out, const cfloat* __restrict__ in, const cfloat* __restrict__ b,
                           long inner, long nstat, long n)
{
    MDNN_PDL_ENTRY();
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        float2 v = in[i], w = b[(i / inner) % nstat];
        out[i] = float2{v.x + w.x, v.y + w.y};
    }
}

// dx = (g - gm[s]) * istd[s] + u * f[s]
__global__ void k_bn_combine(cfloat* __restrict__ dx, const cfloat* __restrict__ g, const cfloat* __restrict__ u,
                             const cfloat* __restrict__ gm, const cfloat* __restrict__ istd,
                             const cfloat* __restrict__ f, long inner, long nstat, long n)
{
    MDNN_PDL_ENTRY();
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        long s = (i / inner) % nstat;
        float2 gv = g[i], m = gm[s], uv = u[i], fs = f[s];
        float is = istd[s].x;
        float2 t{(gv.x - m.x) * is, (gv.y - m.y) * is};
        t.x += uv.x * fs.x - uv.y * fs.y;
        t.y += uv.x * fs.y + uv.y * fs.x;
        dx[i] = t;
    }
}

// f[s] = coef * Re(p[s]) * istd^3   (complex (f, 0))
__global__ void k_bn_f(cfloat* f, const cfloat* p, const cfloat* istd, long nstat, float coef)
{
    MDNN_PDL_ENTRY();
    for (long s = blockIdx.x * long(blockDim.x) + threadIdx.x; s < nstat; s += long(gridDim.x) * blockDim.x) {
        float is = istd[s].x;
        f[s] = float2{coef * p[s].x * is * is * is, 0.f};
    }
}

} // namespace

void launch_stat_mul(cfloat* out, const cfloat* in, const cfloat* s, const IsoGeom& g, bool conj_s)
{
    long n = g.inner * g.nstat * g.outer;
    pdl_launch(k_stat_mul, grid_for(n), kT, 0, ctx().stream, out, in, s, g.inner, g.nstat, n, conj_s);
    KERNEL_CHECK();
}

void launch_stat_add(cfloat* out, const cfloat* in, const cfloat* b, const IsoGeom& g)
{
    long n = g.inner * g.nstat * g.outer;
    pdl_launch(k_stat_add, grid_for(n), kT, 0, ctx().stream, out, in, b, g.inner, g.nstat, n);
    KERNEL_CHECK();
}

void launch_stat_mul_u_f(cfloat* out, const cfloat* u, const cfloat* f, const IsoGeom& g)
{
    launch_stat_mul(out, u, f, g, false);
}

namespace {
__global__ void k_real_to_complex(cfloat* out, const float* in, long n)
{
    MDNN_PDL_ENTRY();
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        out[i] = cfloat{in[i], 0.f};
}
} // namespace

void launch_real_to_complex(cfloat* out, const float* in, long n)
{
    pdl_launch(k_real_to_complex, grid_for(n), kT, 0, ctx().stream, out, in, n);
    KERNEL_CHECK();
}

void bn_train_forward(cfloat* y, cfloat* u, cfloat* istd, cfloat* mean_out, cfloat* var_out, const cfloat* x,
                      const cfloat* mean_in, const cfloat* var_in, const IsoGeom& g, float eps, float mom)
{
    auto& c = ctx();
    const long n = g.inner * g.nstat * g.outer;
    const float inv_m = float(1.0 / double(g.inner * g.outer));
    DArray mean(Dims{g.nstat}, false), var(Dims{g.nstat}, false);
    launch_iso_reduce(mean.data(), x, nullptr, g.inner, g.nstat, g.outer, 0, inv_m);
    pdl_launch(k_sub_stat, grid_for(n), kT, 0, c.stream, u, x, mean.data(), g.inner, g.nstat, n);
    KERNEL_CHECK();
    launch_iso_reduce(var.data(), u, u, g.inner, g.nstat, g.outer, 2, inv_m);
    pdl_launch(k_stats_finish, 1, 128, 0, c.stream, istd, mean_out, var_out, mean.data(), var.data(), mean_in, var_in,
                                            g.nstat, eps, mom, 1);
    KERNEL_CHECK();
    launch_stat_mul(y, u, istd, g, false);
}

void bn_infer_forward(cfloat* y, cfloat* u, cfloat* istd, const cfloat* x, const cfloat* mean_in,
                      const cfloat* var_in, const IsoGeom& g, float eps)
{
    auto& c = ctx();
    const long n = g.inner * g.nstat * g.outer;
    pdl_launch(k_stats_finish, 1, 128, 0, c.stream, istd, nullptr, nullptr, nullptr, var_in, nullptr, nullptr, g.nstat, eps,
                                            0.f, 0);
    KERNEL_CHECK();
    pdl_launch(k_sub_stat, grid_for(n), kT, 0, c.stream, u, x, mean_in, g.inner, g.nstat, n);
    KERNEL_CHECK();
    launch_stat_mul(y, u, istd, g, false);
}

void bn_train_adjoint_x(cfloat* dx, const cfloat* gin, const cfloat* u, const cfloat* istd, const IsoGeom& g)
{
    // dx = (g - mean(g)) istd - u Re(sum g conj u) istd^3 / m   (ops.hpp:1245-1263)
    auto& c = ctx();
    const long n = g.inner * g.nstat * g.outer;
    const double m = double(g.inner * g.outer);
    DArray gm(Dims{g.nstat}, false), p(Dims{g.nstat}, false), f(Dims{g.nstat}, false);
    launch_iso_reduce(gm.data(), gin, nullptr, g.inner, g.nstat, g.outer, 0, float(1.0 / m));
    launch_iso_reduce(p.data(), gin, u, g.inner, g.nstat, g.outer, 1, 1.f);
    pdl_launch(k_bn_f, 1, 128, 0, c.stream, f.data(), p.data(), istd, g.nstat, float(-1.0 / m));
    KERNEL_CHECK();
    pdl_launch(k_bn_combine, grid_for(n), kT, 0, c.stream, dx, gin, u, gm.data(), istd, f.data(), g.inner, g.nstat, n);
    KERNEL_CHECK();
}

void bn_train_deriv_x(cfloat* dy, const cfloat* dx, const cfloat* u, const cfloat* istd, const IsoGeom& g)
{
    // dmu = mean(dx); dv = (2/m) Re sum dx conj(u); dy = (dx - dmu) istd - u Re(dv)/2 istd^3 (ops.hpp:1172-1190)
    auto& c = ctx();
    const long n = g.inner * g.nstat * g.outer;
    const double m = double(g.inner * g.outer);
    DArray gm(Dims{g.nstat}, false), p(Dims{g.nstat}, false), f(Dims{g.nstat}, false);
    launch_iso_reduce(gm.data(), dx, nullptr, g.inner, g.nstat, g.outer, 0, float(1.0 / m));
    launch_iso_reduce(p.data(), dx, u, g.inner, g.nstat, g.outer, 1, 1.f);
    pdl_launch(k_bn_f, 1, 128, 0, c.stream, f.data(), p.data(), istd, g.nstat, float(-1.0 / m));
    KERNEL_CHECK();
    pdl_launch(k_bn_combine, grid_for(n), kT, 0, c.stream, dy, dx, u, gm.data(), istd, f.data(), g.inner, g.nstat, n);
    KERNEL_CHECK();
}

} // namespace mdnn
