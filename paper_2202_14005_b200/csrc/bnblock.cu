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

// Thread mapping for all passes: a thread owns the channel pair (2l, 2l+1),
// l = tid % (C/2), and reads / writes them as float2 from the Re and Im halves
// of the pixel (warp-contiguous 8-byte accesses).  C/2 divides the block, so
// the pair is fixed for a thread across its grid-stride pixel loop.
struct Pair {
    int tpp, l, pl, ppb; // threads per pixel, pair index, pixel lane, pixels per sweep
    __device__ explicit Pair(int C)
    {
        tpp = C / 2;
        l = threadIdx.x % tpp;
        pl = threadIdx.x / tpp;
        ppb = kT / tpp;
    }
};

__device__ __forceinline__ float2 ld2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void st2(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }

// fixed-order reduction of NV doubles per thread over the pixel lanes of each
// pair; the pair's two channels land in part[(blk * C + c) * NV + j]
template<int NV>
__device__ void fold_lanes(double* __restrict__ part, double (&a)[2][NV], const Pair& q, int C)
{
    extern __shared__ double sh[];
#pragma unroll
    for (int k = 0; k < 2; k++)
#pragma unroll
        for (int j = 0; j < NV; j++)
            sh[(threadIdx.x * 2 + k) * NV + j] = a[k][j];
    __syncthreads();
    if (threadIdx.x < C) {
        const int c = threadIdx.x, l = c / 2, k = c % 2;
        double r[NV];
#pragma unroll
        for (int j = 0; j < NV; j++)
            r[j] = 0;
        for (int lane = 0; lane < q.ppb; lane++)
#pragma unroll
            for (int j = 0; j < NV; j++)
                r[j] += sh[((lane * q.tpp + l) * 2 + k) * NV + j];
#pragma unroll
        for (int j = 0; j < NV; j++)
            part[(size_t(blockIdx.x) * C + c) * NV + j] = r[j];
    }
}

// block-per-channel fixed-order tree over the per-block partials
template<int NV>
__device__ void sum_partials(double (&r)[NV], const double* __restrict__ part, int nblocks, int C, int c)
{
    __shared__ double s[NV][kT];
    double a[NV];
#pragma unroll
    for (int j = 0; j < NV; j++)
        a[j] = 0;
    // KU rows' loads in flight per thread (the rows are 2C NV doubles apart: one
    // sector each, latency-bound when issued one at a time), summed in the same
    // order as the one-at-a-time loop
    constexpr int KU = 8;
    for (int k0 = threadIdx.x; k0 < nblocks; k0 += KU * kT) {
        double v[KU][NV];
#pragma unroll
        for (int u = 0; u < KU; u++) {
            const int k = k0 + u * kT;
#pragma unroll
            for (int j = 0; j < NV; j++)
                v[u][j] = k < nblocks ? __ldcg(part + (size_t(k) * C + c) * NV + j) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < KU; u++)
            if (k0 + u * kT < nblocks)
#pragma unroll
                for (int j = 0; j < NV; j++)
                    a[j] += v[u][j];
    }
#pragma unroll
    for (int j = 0; j < NV; j++)
        s[j][threadIdx.x] = a[j];
    __syncthreads();
    for (int h = kT / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h)
#pragma unroll
            for (int j = 0; j < NV; j++)
                s[j][threadIdx.x] += s[j][threadIdx.x + h];
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < NV; j++)
        r[j] = s[j][0];
}

// pass 1 forward: per block partial [Sum Re, Sum Im, Sum |x|^2] per channel
__global__ void __launch_bounds__(kT) k_stats(double* __restrict__ part, const float* __restrict__ x, long npix,
                                              int C, long pix_per_block)
{
    MDNN_PDL_ENTRY();
    const Pair q(C);
    const long p0 = long(blockIdx.x) * pix_per_block, p1 = min(npix, p0 + pix_per_block);
    // fp32 running sums per thread (a few hundred terms each, fixed order),
    // folded across threads and blocks in double: the stream is HBM-bound,
    // a double accumulate per element was not (FP64 + conversions)
    // shifted by the thread's first pixel (re-centred in double below): the
    // sum of squares carries the spread, not the mean
    float f[2][3] = {{0, 0, 0}, {0, 0, 0}};
    float2 shr{0.f, 0.f}, shi{0.f, 0.f};
    long cnt = 0;
    if (p0 + q.pl < p1) {
        shr = ld2(x + (p0 + q.pl) * 2 * C + 2 * q.l);
        shi = ld2(x + (p0 + q.pl) * 2 * C + C + 2 * q.l);
    }
    constexpr int U = 8; // 128 B of loads in flight per thread (latency-bound otherwise)
    for (long p = p0 + q.pl; p < p1; p += U * q.ppb) {
        float2 re[U], im[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const long pp = p + u * q.ppb;
            re[u] = pp < p1 ? ld2(x + pp * 2 * C + 2 * q.l) : shr;
            im[u] = pp < p1 ? ld2(x + pp * 2 * C + C + 2 * q.l) : shi;
            cnt += pp < p1;
        }
#pragma unroll
        for (int u = 0; u < U; u++) { // out-of-range slots hold the shift: zero contribution
            const float2 dr{re[u].x - shr.x, re[u].y - shr.y}, di{im[u].x - shi.x, im[u].y - shi.y};
            f[0][0] += dr.x;
            f[0][1] += di.x;
            f[0][2] = fmaf(dr.x, dr.x, fmaf(di.x, di.x, f[0][2]));
            f[1][0] += dr.y;
            f[1][1] += di.y;
            f[1][2] = fmaf(dr.y, dr.y, fmaf(di.y, di.y, f[1][2]));
        }
    }
    double a[2][3];
    const double n = double(cnt);
    const double sr[2] = {shr.x, shr.y}, si[2] = {shi.x, shi.y};
#pragma unroll
    for (int k = 0; k < 2; k++) {
        a[k][0] = n * sr[k] + f[k][0];
        a[k][1] = n * si[k] + f[k][1];
        a[k][2] = sr[k] * (n * sr[k] + 2.0 * f[k][0]) + si[k] * (n * si[k] + 2.0 * f[k][1]) + f[k][2];
    }
    fold_lanes<3>(part, a, q, C);
}

__device__ void stats_finish(const double (&r)[3], float2* __restrict__ mu, float* __restrict__ istd,
                             float2* __restrict__ mean_out, float2* __restrict__ var_out, int c, long m,
                             const float2* __restrict__ mean_in, const float2* __restrict__ var_in, float eps,
                             float mom);

// final: mean, var (biased), istd, moving statistics; one block per channel
__global__ void __launch_bounds__(kT) k_stats_final(float2* __restrict__ mu, float* __restrict__ istd,
                                                    float2* __restrict__ mean_out, float2* __restrict__ var_out,
                                                    const double* __restrict__ part, int nblocks, int C, long m,
                                                    const float2* __restrict__ mean_in,
                                                    const float2* __restrict__ var_in, float eps, float mom)
{
    MDNN_PDL_ENTRY();
    const int c = blockIdx.x;
    double r[3];
    sum_partials<3>(r, part, nblocks, C, c);
    if (threadIdx.x == 0)
        stats_finish(r, mu, istd, mean_out, var_out, c, m, mean_in, var_in, eps, mom);
}

// final from producer partials (conv epilogue): part[blk][2C real channels][sum, sum of squares]
__global__ void __launch_bounds__(kT) k_stats_final_pre(float2* __restrict__ mu, float* __restrict__ istd,
                                                        float2* __restrict__ mean_out, float2* __restrict__ var_out,
                                                        const double* __restrict__ part, int nblocks, int C, long m,
                                                        const float2* __restrict__ mean_in,
                                                        const float2* __restrict__ var_in, float eps, float mom)
{
    MDNN_PDL_ENTRY();
    const int c = blockIdx.x;
    double re[2], im[2];
    sum_partials<2>(re, part, nblocks, 2 * C, c);
    __syncthreads(); // sum_partials' shared scratch is reused
    sum_partials<2>(im, part, nblocks, 2 * C, C + c);
    const double r[3] = {re[0], im[0], re[1] + im[1]};
    if (threadIdx.x == 0)
        stats_finish(r, mu, istd, mean_out, var_out, c, m, mean_in, var_in, eps, mom);
}

__device__ void stats_finish(const double (&r)[3], float2* __restrict__ mu, float* __restrict__ istd,
                             float2* __restrict__ mean_out, float2* __restrict__ var_out, int c, long m,
                             const float2* __restrict__ mean_in, const float2* __restrict__ var_in, float eps,
                             float mom)
{
    const double mr = r[0] / double(m), mi = r[1] / double(m);
    const double var = r[2] / double(m) - (mr * mr + mi * mi);
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

struct ChanCoef {
    float2 m, g, bb;
    float s;
};

__device__ __forceinline__ ChanCoef coef(const float2* mu, const float* istd, const float2* gamma,
                                         const float2* beta, int c)
{
    return ChanCoef{mu[c], gamma[c], beta[c], istd[c]};
}

// yhat = (x - mu) istd ; z = g yhat + beta
__device__ __forceinline__ void bn_z(const ChanCoef& k, float xr, float xi, float& hr, float& hi, float& zr,
                                     float& zi)
{
    hr = (xr - k.m.x) * k.s;
    hi = (xi - k.m.y) * k.s;
    zr = k.g.x * hr - k.g.y * hi + k.bb.x;
    zi = k.g.x * hi + k.g.y * hr + k.bb.y;
}

// pass 2 forward: out = crelu(g * (x - mu) * istd + beta)
__global__ void __launch_bounds__(kT) k_apply(float* __restrict__ out, const float* __restrict__ x,
                                              const float2* __restrict__ mu, const float* __restrict__ istd,
                                              const float2* __restrict__ gamma, const float2* __restrict__ beta,
                                              long npix, int C, bool rnd)
{
    MDNN_PDL_ENTRY();
    const int tpp = C / 2, l = threadIdx.x % tpp;
    const ChanCoef k0 = coef(mu, istd, gamma, beta, 2 * l), k1 = coef(mu, istd, gamma, beta, 2 * l + 1);
    const long pstride = long(gridDim.x) * kT / tpp;
    constexpr int U = 4;
    for (long p = (long(blockIdx.x) * kT + threadIdx.x) / tpp; p < npix; p += U * pstride) {
        float2 re[U], im[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const long pp = p + u * pstride;
            if (pp < npix) {
                re[u] = ld2(x + pp * 2 * C + 2 * l);
                im[u] = ld2(x + pp * 2 * C + C + 2 * l);
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const long pp = p + u * pstride;
            if (pp >= npix)
                break;
            float hr, hi, z0r, z0i, z1r, z1i;
            bn_z(k0, re[u].x, im[u].x, hr, hi, z0r, z0i);
            bn_z(k1, re[u].y, im[u].y, hr, hi, z1r, z1i);
            st2(out + pp * 2 * C + 2 * l,
                float2{maybe_round(fmaxf(z0r, 0.f), rnd), maybe_round(fmaxf(z1r, 0.f), rnd)});
            st2(out + pp * 2 * C + C + 2 * l,
                float2{maybe_round(fmaxf(z0i, 0.f), rnd), maybe_round(fmaxf(z1i, 0.f), rnd)});
        }
    }
}

// pass 1 backward: per block partial S1 = sum gz, S2 = sum gz * conj(yhat)
__global__ void __launch_bounds__(kT) k_bwd_reduce(double* __restrict__ part, const float* __restrict__ gout,
                                                   const float* __restrict__ x, const float2* __restrict__ mu,
                                                   const float* __restrict__ istd, const float2* __restrict__ gamma,
                                                   const float2* __restrict__ beta, long npix, int C,
                                                   long pix_per_block)
{
    MDNN_PDL_ENTRY();
    const Pair q(C);
    const ChanCoef kc[2] = {coef(mu, istd, gamma, beta, 2 * q.l), coef(mu, istd, gamma, beta, 2 * q.l + 1)};
    const long p0 = long(blockIdx.x) * pix_per_block, p1 = min(npix, p0 + pix_per_block);
    float f[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}}; // fp32 per thread, double across threads (see k_stats)
    constexpr int U = 4; // 128 B of loads in flight per thread
    for (long p = p0 + q.pl; p < p1; p += U * q.ppb) {
        float2 xr[U], xi[U], gr[U], gi[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const long pp = p + u * q.ppb;
            const bool ok = pp < p1;
            xr[u] = ok ? ld2(x + pp * 2 * C + 2 * q.l) : float2{0.f, 0.f};
            xi[u] = ok ? ld2(x + pp * 2 * C + C + 2 * q.l) : float2{0.f, 0.f};
            gr[u] = ok ? ld2(gout + pp * 2 * C + 2 * q.l) : float2{0.f, 0.f};
            gi[u] = ok ? ld2(gout + pp * 2 * C + C + 2 * q.l) : float2{0.f, 0.f};
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
#pragma unroll
            for (int k = 0; k < 2; k++) {
                float hr, hi, zr, zi;
                bn_z(kc[k], k ? xr[u].y : xr[u].x, k ? xi[u].y : xi[u].x, hr, hi, zr, zi);
                const float g_r = zr > 0.f ? (k ? gr[u].y : gr[u].x) : 0.f;
                const float g_i = zi > 0.f ? (k ? gi[u].y : gi[u].x) : 0.f;
                f[k][0] += g_r;
                f[k][1] += g_i;
                // gz * conj(yhat)
                f[k][2] = fmaf(g_r, hr, fmaf(g_i, hi, f[k][2]));
                f[k][3] = fmaf(g_i, hr, fmaf(-g_r, hi, f[k][3]));
            }
        }
    }
    double a[2][4];
#pragma unroll
    for (int k = 0; k < 2; k++)
#pragma unroll
        for (int j = 0; j < 4; j++)
            a[k][j] = f[k][j];
    fold_lanes<4>(part, a, q, C);
}

// final backward (block per channel): dbeta = S1, dgamma = S2, and the coefficients
//   gm = conj(g) S1 / m ;  fh = -Re(conj(g) S2) * istd / m   (dx = (gyh - gm) istd + yhat * fh)
__global__ void __launch_bounds__(kT) k_bwd_final(float2* __restrict__ dbeta, float2* __restrict__ dgamma,
                                                  float2* __restrict__ gm, float* __restrict__ fh,
                                                  const double* __restrict__ part, int nblocks, int C, long m,
                                                  const float2* __restrict__ gamma, const float* __restrict__ istd)
{
    MDNN_PDL_ENTRY();
    const int c = blockIdx.x;
    double r[4];
    sum_partials<4>(r, part, nblocks, C, c);
    if (threadIdx.x != 0)
        return;
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

// final backward from producer partials (conv bwd-data epilogue):
// part[blk][2C real channels][3] = (sum gz_comp, Re S2 contribution, Im S2 contribution)
__global__ void __launch_bounds__(kT) k_bwd_final_pre(float2* __restrict__ dbeta, float2* __restrict__ dgamma,
                                                      float2* __restrict__ gm, float* __restrict__ fh,
                                                      const double* __restrict__ part, int nblocks, int C, long m,
                                                      const float2* __restrict__ gamma,
                                                      const float* __restrict__ istd)
{
    MDNN_PDL_ENTRY();
    const int c = blockIdx.x;
    double re[3], im[3];
    sum_partials<3>(re, part, nblocks, 2 * C, c);
    __syncthreads(); // sum_partials' shared scratch is reused
    sum_partials<3>(im, part, nblocks, 2 * C, C + c);
    if (threadIdx.x != 0)
        return;
    const double r[4] = {re[0], im[0], re[1] + im[1], re[2] + im[2]};
    if (dbeta)
        dbeta[c] = float2{float(r[0]), float(r[1])};
    if (dgamma)
        dgamma[c] = float2{float(r[2]), float(r[3])};
    const double gr = gamma[c].x, gi = gamma[c].y;
    const double c1r = gr * r[0] + gi * r[1], c1i = gr * r[1] - gi * r[0];
    gm[c] = float2{float(c1r / double(m)), float(c1i / double(m))};
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
    MDNN_PDL_ENTRY();
    const int tpp = C / 2, l = threadIdx.x % tpp;
    const ChanCoef kc[2] = {coef(mu, istd, gamma, beta, 2 * l), coef(mu, istd, gamma, beta, 2 * l + 1)};
    const float2 gmc[2] = {gm[2 * l], gm[2 * l + 1]};
    const float fc[2] = {fh[2 * l], fh[2 * l + 1]};
    const long pstride = long(gridDim.x) * kT / tpp;
    constexpr int U = 2; // 64 B of loads in flight per thread
    for (long p0 = (long(blockIdx.x) * kT + threadIdx.x) / tpp; p0 < npix; p0 += U * pstride) {
    float2 xr_[U], xi_[U], gr_[U], gi_[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        const long pp = p0 + u * pstride;
        if (pp < npix) {
            xr_[u] = ld2(x + pp * 2 * C + 2 * l);
            xi_[u] = ld2(x + pp * 2 * C + C + 2 * l);
            gr_[u] = ld2(gout + pp * 2 * C + 2 * l);
            gi_[u] = ld2(gout + pp * 2 * C + C + 2 * l);
        }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        const long p = p0 + u * pstride;
        if (p >= npix)
            break;
        const float2 xr = xr_[u], xi = xi_[u], gr2 = gr_[u], gi2 = gi_[u];
        float o_r[2], o_i[2];
#pragma unroll
        for (int k = 0; k < 2; k++) {
            float hr, hi, zr, zi;
            bn_z(kc[k], k ? xr.y : xr.x, k ? xi.y : xi.x, hr, hi, zr, zi);
            const float g_r = zr > 0.f ? (k ? gr2.y : gr2.x) : 0.f;
            const float g_i = zi > 0.f ? (k ? gi2.y : gi2.x) : 0.f;
            const float2 g = kc[k].g;
            // gyh = gz * conj(g)
            const float yr = g_r * g.x + g_i * g.y, yi = g_i * g.x - g_r * g.y;
            o_r[k] = maybe_round((yr - gmc[k].x) * kc[k].s + hr * fc[k], rnd);
            o_i[k] = maybe_round((yi - gmc[k].y) * kc[k].s + hi * fc[k], rnd);
        }
        st2(dx + p * 2 * C + 2 * l, float2{o_r[0], o_r[1]});
        st2(dx + p * 2 * C + C + 2 * l, float2{o_i[0], o_i[1]});
    }
    }
}

int reduce_blocks(long npix)
{
    long b = long(ctx().sm_count) * 8;
    return int(std::max(1L, std::min(b, (npix + 255) / 256)));
}

int grid_ew(long npix, int C)
{
    long b = (npix * (C / 2) + kT - 1) / kT;
    return int(std::max(1L, std::min(b, long(ctx().sm_count) * 8)));
}

} // namespace

void bnblock_forward(float* out, float2* mu, float* istd, float2* mean_out, float2* var_out, const float* x,
                     const float2* mean_in, const float2* var_in, const float2* gamma, const float2* beta, long npix,
                     int C, float eps, float mom, bool round_tf32, const double* pre_part, int pre_blocks)
{
    auto& c = ctx();
    if (C < 2 || 256 % C != 0)
        throw ConfigError("bnblock: channel count must be >= 2 and divide 256");
    if (pre_part && pre_blocks > 0) {
        // statistics partials came with x from its producer: apply pass only
        ProfScope prof("bnblock_fwd", 8.0 * 2 * npix * C);
        pdl_launch(k_stats_final_pre, C, kT, 0, c.stream, mu, istd, mean_out, var_out, pre_part, pre_blocks, C, npix,
                                                  mean_in, var_in, eps, mom);
        KERNEL_CHECK();
        pdl_launch(k_apply, grid_ew(npix, C), kT, 0, c.stream, out, x, mu, istd, gamma, beta, npix, C, round_tf32);
        KERNEL_CHECK();
        return;
    }
    const int nb = reduce_blocks(npix);
    const long ppb = (npix + nb - 1) / nb;
    double* part;
    CUDA_CHECK(cudaMallocAsync(&part, sizeof(double) * 3 * C * nb, c.stream));
    ProfScope prof("bnblock_fwd", 8.0 * 2 * npix * C + 8.0 * npix * C);
    pdl_launch(k_stats, nb, kT, sizeof(double) * 2 * 3 * kT, c.stream, part, x, npix, C, ppb);
    KERNEL_CHECK();
    pdl_launch(k_stats_final, C, kT, 0, c.stream, mu, istd, mean_out, var_out, part, nb, C, npix, mean_in,
                                                       var_in, eps, mom);
    KERNEL_CHECK();
    pdl_launch(k_apply, grid_ew(npix, C), kT, 0, c.stream, out, x, mu, istd, gamma, beta, npix, C, round_tf32);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(part, c.stream));
}

void bnblock_backward(float* dx, float2* dgamma, float2* dbeta, const float* gout, const float* x, const float2* mu,
                      const float* istd, const float2* gamma, const float2* beta, long npix, int C, bool round_tf32,
                      const double* pre_part, int pre_blocks)
{
    auto& c = ctx();
    const bool pre = pre_part && pre_blocks > 0;
    const int nb = reduce_blocks(npix);
    const long ppb = (npix + nb - 1) / nb;
    double* part = nullptr;
    float2* gm;
    float* fh;
    if (!pre)
        CUDA_CHECK(cudaMallocAsync(&part, sizeof(double) * 4 * C * nb, c.stream));
    CUDA_CHECK(cudaMallocAsync(&gm, sizeof(float2) * C, c.stream));
    CUDA_CHECK(cudaMallocAsync(&fh, sizeof(float) * C, c.stream));
    // algorithmic bytes: reduction pass (x, gout) unless folded into the producer, apply pass (x, gout, dx)
    ProfScope prof("bnblock_bwd", 8.0 * (pre ? 3 : 5) * npix * C);
    if (pre) {
        pdl_launch(k_bwd_final_pre, C, kT, 0, c.stream, dbeta, dgamma, gm, fh, pre_part, pre_blocks, C, npix, gamma, istd);
        KERNEL_CHECK();
    } else {
        pdl_launch(k_bwd_reduce, nb, kT, sizeof(double) * 2 * 4 * kT, c.stream, part, gout, x, mu, istd, gamma, beta, npix, C,
                                                                      ppb);
        KERNEL_CHECK();
        pdl_launch(k_bwd_final, C, kT, 0, c.stream, dbeta, dgamma, gm, fh, part, nb, C, npix, gamma, istd);
        KERNEL_CHECK();
    }
    if (dx) {
        pdl_launch(k_bwd_apply, grid_ew(npix, C), kT, 0, c.stream, dx, gout, x, mu, istd, gamma, beta, gm, fh, npix, C,
                                                            round_tf32);
        KERNEL_CHECK();
    }
    if (part)
        CUDA_CHECK(cudaFreeAsync(part, c.stream));
    CUDA_CHECK(cudaFreeAsync(gm, c.stream));
    CUDA_CHECK(cudaFreeAsync(fh, c.stream));
}

} // namespace mdnn
