// Fused MoDL denoiser block on channels-last activations:
//   out = CReLU(gamma * BN_train(x) + beta)
// replacing the reference chain BatchNormNode -> TenMul(bn_scale) ->
// BroadcastAddNode -> CReluNode (recon.hpp:748-776, ops.hpp:1070-1298,
// 153-209, 451-475) with 2 HBM passes forward (statistics, apply) and 2
// backward (reductions, apply) instead of ~12 + ~14.
//
// CHLAST element (pixel p, channel c): Re at f[p*2C + c], Im at f[p*2C + C + c].
// Per-channel statistics are accumulated in double in a fixed-order two-stage
// tree (bitwise run-to-run stable).  The forward output and the backward
// input-cotangent feed TF32 convolutions and are rounded RN to TF32 by this
// producer when `round_tf32` is set (the consumer's operand conversion, fused).
#include "kernels.h"
#include "profile.h"
#include "sm100.cuh"

#include <algorithm>

namespace mdnn {

namespace {

constexpr int kT = 256;

__device__ __forceinline__ float maybe_round(float v, bool r) { return r ? sm100::to_tf32(v) : v; }

// pass 1 forward: per block partial [Sum Re, Sum Im, Sum |x|^2] per channel
__global__ void __launch_bounds__(kT) k_stats(double* __restrict__ part, const float* __restrict__ x, long npix,
                                              int C, long pix_per_block)
{
    extern __shared__ double sh[];
    const int ppb = kT / C; // pixels per sweep (C divides 256)
    const int c = threadIdx.x % C, pl = threadIdx.x / C;
    const long p0 = long(blockIdx.x) * pix_per_block, p1 = min(npix, p0 + pix_per_block);
    double sr = 0, si = 0, sq = 0;
    for (long p = p0 + pl; p < p1; p += ppb) {
        const float re = x[p * 2 * C + c], im = x[p * 2 * C + C + c];
        sr += re;
        si += im;
        sq += double(re) * re + double(im) * im;
    }
    // reduce over the ppb pixel lanes of each channel (fixed order)
    double* s = sh;
    s[threadIdx.x * 3 + 0] = sr;
    s[threadIdx.x * 3 + 1] = si;
    s[threadIdx.x * 3 + 2] = sq;
    __syncthreads();
    if (threadIdx.x < C) {
        double a = 0, b = 0, q = 0;
        for (int k = 0; k < ppb; k++) {
            a += s[(k * C + c) * 3 + 0];
            b += s[(k * C + c) * 3 + 1];
            q += s[(k * C + c) * 3 + 2];
        }
        double* dst = part + (size_t(blockIdx.x) * C + c) * 3;
        dst[0] = a;
        dst[1] = b;
        dst[2] = q;
    }
}

// final: mean, var (biased), istd, moving statistics
__global__ void k_stats_final(float2* __restrict__ mu, float* __restrict__ istd, float2* __restrict__ mean_out,
                              float2* __restrict__ var_out, const double* __restrict__ part, int nblocks, int C,
                              long m, const float2* __restrict__ mean_in, const float2* __restrict__ var_in,
                              float eps, float mom)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C)
        return;
    double a = 0, b = 0, q = 0;
    for (int k = 0; k < nblocks; k++) {
        a += part[(size_t(k) * C + c) * 3 + 0];
        b += part[(size_t(k) * C + c) * 3 + 1];
        q += part[(size_t(k) * C + c) * 3 + 2];
    }
    const double mr = a / double(m), mi = b / double(m);
    const double var = q / double(m) - (mr * mr + mi * mi);
    const float meanr = float(mr), meani = float(mi), v = float(var > 0 ? var : 0);
    mu[c] = float2{meanr, meani};
    istd[c] = 1.f / sqrtf(v + eps);
    if (mean_out) {
        // stat' = mom * batch + (1 - mom) * stat  (ops.hpp:1129-1132)
        float2 im = mean_in[c], iv = var_in[c];
        mean_out[c] = float2{mom * meanr + (1.f - mom) * im.x, mom * meani + (1.f - mom) * im.y};
        var_out[c] = float2{mom * v + (1.f - mom) * iv.x, (1.f - mom) * iv.y};
    }
}

// pass 2 forward: out = crelu(g * (x - mu) * istd + beta)
__global__ void __launch_bounds__(kT) k_apply(float* __restrict__ out, const float* __restrict__ x,
                                              const float2* __restrict__ mu, const float* __restrict__ istd,
                                              const float2* __restrict__ gamma, const float2* __restrict__ beta,
                                              long npix, int C, bool rnd)
{
    const long n = npix * C;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        const int c = int(i % C);
        const long p = i / C;
        const float xr = x[p * 2 * C + c], xi = x[p * 2 * C + C + c];
        const float2 m = mu[c], g = gamma[c], bb = beta[c];
        const float s = istd[c];
        const float hr = (xr - m.x) * s, hi = (xi - m.y) * s;
        float zr = g.x * hr - g.y * hi + bb.x, zi = g.x * hi + g.y * hr + bb.y;
        out[p * 2 * C + c] = maybe_round(zr > 0.f ? zr : 0.f, rnd);
        out[p * 2 * C + C + c] = maybe_round(zi > 0.f ? zi : 0.f, rnd);
    }
}

// pass 1 backward: per block partial S1 = sum gz, S2 = sum gz * conj(yhat)
__global__ void __launch_bounds__(kT) k_bwd_reduce(double* __restrict__ part, const float* __restrict__ gout,
                                                   const float* __restrict__ x, const float2* __restrict__ mu,
                                                   const float* __restrict__ istd, const float2* __restrict__ gamma,
                                                   const float2* __restrict__ beta, long npix, int C,
                                                   long pix_per_block)
{
    extern __shared__ double sh[];
    const int ppb = kT / C;
    const int c = threadIdx.x % C, pl = threadIdx.x / C;
    const long p0 = long(blockIdx.x) * pix_per_block, p1 = min(npix, p0 + pix_per_block);
    const float2 m = mu[c], g = gamma[c], bb = beta[c];
    const float s = istd[c];
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (long p = p0 + pl; p < p1; p += ppb) {
        const float xr = x[p * 2 * C + c], xi = x[p * 2 * C + C + c];
        const float hr = (xr - m.x) * s, hi = (xi - m.y) * s;
        const float zr = g.x * hr - g.y * hi + bb.x, zi = g.x * hi + g.y * hr + bb.y;
        const float gr = zr > 0.f ? gout[p * 2 * C + c] : 0.f;
        const float gi = zi > 0.f ? gout[p * 2 * C + C + c] : 0.f;
        a0 += gr;
        a1 += gi;
        // gz * conj(yhat)
        a2 += double(gr) * hr + double(gi) * hi;
        a3 += double(gi) * hr - double(gr) * hi;
    }
    double* s4 = sh;
    s4[threadIdx.x * 4 + 0] = a0;
    s4[threadIdx.x * 4 + 1] = a1;
    s4[threadIdx.x * 4 + 2] = a2;
    s4[threadIdx.x * 4 + 3] = a3;
    __syncthreads();
    if (threadIdx.x < C) {
        double r[4] = {0, 0, 0, 0};
        for (int k = 0; k < ppb; k++)
            for (int j = 0; j < 4; j++)
                r[j] += s4[(k * C + c) * 4 + j];
        double* dst = part + (size_t(blockIdx.x) * C + c) * 4;
        for (int j = 0; j < 4; j++)
            dst[j] = r[j];
    }
}

// final backward: dbeta = S1, dgamma = S2, and the per-channel coefficients
//   gm = conj(g) S1 / m ;  fh = -Re(conj(g) S2) * istd / m   (dx = (gyh - gm) istd + yhat * fh)
__global__ void k_bwd_final(float2* __restrict__ dbeta, float2* __restrict__ dgamma, float2* __restrict__ gm,
                            float* __restrict__ fh, const double* __restrict__ part, int nblocks, int C, long m,
                            const float2* __restrict__ gamma, const float* __restrict__ istd)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C)
        return;
    double r[4] = {0, 0, 0, 0};
    for (int k = 0; k < nblocks; k++)
        for (int j = 0; j < 4; j++)
            r[j] += part[(size_t(k) * C + c) * 4 + j];
    if (dbeta)
        dbeta[c] = float2{float(r[0]), float(r[1])};
    if (dgamma)
        dgamma[c] = float2{float(r[2]), float(r[3])};
    const double gr = gamma[c].x, gi = gamma[c].y;
    // conj(g) * S1
    const double c1r = gr * r[0] + gi * r[1], c1i = gr * r[1] - gi * r[0];
    gm[c] = float2{float(c1r / double(m)), float(c1i / double(m))};
    // Re(conj(g) * S2)
    const double re2 = gr * r[2] + gi * r[3];
    fh[c] = float(-re2 * double(istd[c]) / double(m));
}

// pass 2 backward: dx = (gz conj(g) - gm) istd + yhat * fh
__global__ void __launch_bounds__(kT) k_bwd_apply(float* __restrict__ dx, const float* __restrict__ gout,
                                                  const float* __restrict__ x, const float2* __restrict__ mu,
                                                  const float* __restrict__ istd, const float2* __restrict__ gamma,
                                                  const float2* __restrict__ beta, const float2* __restrict__ gm,
                                                  const float* __restrict__ fh, long npix, int C, bool rnd)
{
    const long n = npix * C;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        const int c = int(i % C);
        const long p = i / C;
        const float xr = x[p * 2 * C + c], xi = x[p * 2 * C + C + c];
        const float2 m = mu[c], g = gamma[c], bb = beta[c], gmc = gm[c];
        const float s = istd[c], f = fh[c];
        const float hr = (xr - m.x) * s, hi = (xi - m.y) * s;
        const float zr = g.x * hr - g.y * hi + bb.x, zi = g.x * hi + g.y * hr + bb.y;
        const float gr = zr > 0.f ? gout[p * 2 * C + c] : 0.f;
        const float gi = zi > 0.f ? gout[p * 2 * C + C + c] : 0.f;
        // gyh = gz * conj(g)
        const float yr = gr * g.x + gi * g.y, yi = gi * g.x - gr * g.y;
        dx[p * 2 * C + c] = maybe_round((yr - gmc.x) * s + hr * f, rnd);
        dx[p * 2 * C + C + c] = maybe_round((yi - gmc.y) * s + hi * f, rnd);
    }
}

int reduce_blocks(long npix)
{
    long b = long(ctx().sm_count) * 4;
    return int(std::max(1L, std::min(b, (npix + 255) / 256)));
}

int grid_ew(long n)
{
    long b = (n + kT - 1) / kT;
    return int(std::max(1L, std::min(b, long(ctx().sm_count) * 16)));
}

} // namespace

void bnblock_forward(float* out, float2* mu, float* istd, float2* mean_out, float2* var_out, const float* x,
                     const float2* mean_in, const float2* var_in, const float2* gamma, const float2* beta, long npix,
                     int C, float eps, float mom, bool round_tf32)
{
    auto& c = ctx();
    if (256 % C != 0)
        throw ConfigError("bnblock: channel count must divide 256");
    const int nb = reduce_blocks(npix);
    const long ppb = (npix + nb - 1) / nb;
    double* part;
    CUDA_CHECK(cudaMallocAsync(&part, sizeof(double) * 3 * C * nb, c.stream));
    ProfScope prof("bnblock_fwd", 8.0 * 2 * npix * C + 8.0 * npix * C);
    k_stats<<<nb, kT, sizeof(double) * 3 * kT, c.stream>>>(part, x, npix, C, ppb);
    KERNEL_CHECK();
    k_stats_final<<<(C + 63) / 64, 64, 0, c.stream>>>(mu, istd, mean_out, var_out, part, nb, C, npix, mean_in,
                                                       var_in, eps, mom);
    KERNEL_CHECK();
    k_apply<<<grid_ew(npix * C), kT, 0, c.stream>>>(out, x, mu, istd, gamma, beta, npix, C, round_tf32);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(part, c.stream));
}

void bnblock_backward(float* dx, float2* dgamma, float2* dbeta, const float* gout, const float* x, const float2* mu,
                      const float* istd, const float2* gamma, const float2* beta, long npix, int C, bool round_tf32)
{
    auto& c = ctx();
    const int nb = reduce_blocks(npix);
    const long ppb = (npix + nb - 1) / nb;
    double* part;
    float2* gm;
    float* fh;
    CUDA_CHECK(cudaMallocAsync(&part, sizeof(double) * 4 * C * nb, c.stream));
    CUDA_CHECK(cudaMallocAsync(&gm, sizeof(float2) * C, c.stream));
    CUDA_CHECK(cudaMallocAsync(&fh, sizeof(float) * C, c.stream));
    ProfScope prof("bnblock_bwd", 8.0 * 5 * npix * C);
    k_bwd_reduce<<<nb, kT, sizeof(double) * 4 * kT, c.stream>>>(part, gout, x, mu, istd, gamma, beta, npix, C, ppb);
    KERNEL_CHECK();
    k_bwd_final<<<(C + 63) / 64, 64, 0, c.stream>>>(dbeta, dgamma, gm, fh, part, nb, C, npix, gamma, istd);
    KERNEL_CHECK();
    if (dx) {
        k_bwd_apply<<<grid_ew(npix * C), kT, 0, c.stream>>>(dx, gout, x, mu, istd, gamma, beta, gm, fh, npix, C,
                                                            round_tf32);
        KERNEL_CHECK();
    }
    CUDA_CHECK(cudaFreeAsync(part, c.stream));
    CUDA_CHECK(cudaFreeAsync(gm, c.stream));
    CUDA_CHECK(cudaFreeAsync(fh, c.stream));
}

} // namespace mdnn
