// "Thin" complex convolutions: one side has a single channel (MoDL's first
// layer 1 -> F and last layer F -> 1, conv_layer nn.hpp:344-426).  The wide
// side is channels-last (CHLAST), the thin side is a plain image (for one
// channel the two layouts coincide).  These passes are memory-bound (9 complex
// MACs per wide element), so every kernel streams the wide tensor once with
// warp-contiguous channel accesses and keeps the thin image tile in smem.
//
//   expand  out[p, f] = sum_t thin[p + dir (t - c0)] * U[t, f]
//   reduce  out[q]    = sum_{t, c} wide[q + dir (t - c0), c] * U[t, c]
//   wgrad   dw[t, f]  = sum_p g[p, f] * conj(h[p + t - c0])   (one of g/h wide)
// with U a per-launch packing of w (or its flipped conjugate for adjoints).
#include "kernels.h"
#include "profile.h"

#include <algorithm>

namespace mdnn {

namespace {

constexpr int TX = 32, TY = 8, MAXK = 5, MAXF = 256;

__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }

// U[t][f] for the 4 uses; w has dims [KX, KY, Cin, Cout]
//   mode 0: fwd 1 -> F           U[t][f] = w[t, 0, f]
//   mode 1: bwd-data of F -> 1   U[t][c] = conj(w[flip t, c, 0])   (expand with dir +1 on flipped taps)
//   mode 2: fwd F -> 1           U[t][c] = w[t, c, 0]
//   mode 3: bwd-data of 1 -> F   U[t][f] = conj(w[flip t, 0, f])
__global__ void k_pack_thin(float2* U, const float2* w, int KX, int KY, int F, int mode)
{
    const int KK = KX * KY;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < KK * F; i += gridDim.x * blockDim.x) {
        const int t = i % KK, f = i / KK;
        const int tx = t % KX, ty = t / KX;
        const int tf = (KX - 1 - tx) + KX * (KY - 1 - ty);
        float2 v;
        if (mode == 0 || mode == 2)
            v = w[t + KK * f];
        else {
            float2 ww = w[tf + KK * f];
            v = float2{ww.x, -ww.y};
        }
        U[t * F + f] = v;
    }
}

// thin -> wide, block = TX x TY pixel tile of one item; thread (f, pixel lane)
__global__ void __launch_bounds__(256) k_thin_expand(float* __restrict__ out, const float2* __restrict__ in,
                                                     const float2* __restrict__ U, int X, int Y, int F, int KX, int KY,
                                                     int ox, int oy)
{
    __shared__ float2 tile[(TY + MAXK - 1) * (TX + MAXK - 1)];
    extern __shared__ float2 su[]; // [KK][F]
    const int KK = KX * KY;
    const int HX = TX + KX - 1, HY = TY + KY - 1;
    const long b = blockIdx.z;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const long XY = long(X) * Y;
    for (int e = threadIdx.x; e < HX * HY; e += blockDim.x) {
        const int hx = e % HX, hy = e / HX;
        const int gx = x0 + hx - ox, gy = y0 + hy - oy;
        tile[e] = (gx >= 0 && gx < X && gy >= 0 && gy < Y) ? in[gx + long(X) * gy + XY * b] : float2{0.f, 0.f};
    }
    for (int e = threadIdx.x; e < KK * F; e += blockDim.x)
        su[e] = U[e];
    __syncthreads();
    const int lanes = blockDim.x / F; // pixels processed concurrently
    const int f = threadIdx.x % F, pl = threadIdx.x / F;
    if (pl >= lanes)
        return;
    for (int pix = pl; pix < TX * TY; pix += lanes) {
        const int px = pix % TX, py = pix / TX;
        const int gx = x0 + px, gy = y0 + py;
        if (gx >= X || gy >= Y)
            continue;
        float2 acc{0.f, 0.f};
        for (int ky = 0; ky < KY; ky++)
            for (int kx = 0; kx < KX; kx++) {
                const float2 t = cmul(tile[(py + ky) * HX + px + kx], su[(kx + KX * ky) * F + f]);
                acc.x += t.x;
                acc.y += t.y;
            }
        float* dst = out + ((b * XY) + gx + long(X) * gy) * 2 * F;
        dst[f] = acc.x;
        dst[F + f] = acc.y;
    }
}

// wide -> thin, one output pixel per thread; channels streamed in chunks of CC
constexpr int CC = 8;
__global__ void __launch_bounds__(TX* TY) k_thin_reduce(float2* __restrict__ out, const float* __restrict__ in,
                                                        const float2* __restrict__ U, int X, int Y, int F, int KX,
                                                        int KY, int ox, int oy)
{
    __shared__ float2 tile[(TY + MAXK - 1) * (TX + MAXK - 1) * CC];
    __shared__ float2 su[MAXK * MAXK * CC];
    const int KK = KX * KY;
    const int HX = TX + KX - 1, HY = TY + KY - 1;
    const long b = blockIdx.z;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const long XY = long(X) * Y;
    const int px = threadIdx.x % TX, py = threadIdx.x / TX;
    float2 acc{0.f, 0.f};
    for (int c0 = 0; c0 < F; c0 += CC) {
        const int nc = min(CC, F - c0);
        __syncthreads();
        for (int e = threadIdx.x; e < HX * HY * CC; e += blockDim.x) {
            const int cc = e % CC, hp = e / CC;
            const int hx = hp % HX, hy = hp / HX;
            const int gx = x0 + hx - ox, gy = y0 + hy - oy;
            float2 v{0.f, 0.f};
            if (cc < nc && gx >= 0 && gx < X && gy >= 0 && gy < Y) {
                const float* src = in + ((b * XY) + gx + long(X) * gy) * 2 * F;
                v = float2{src[c0 + cc], src[F + c0 + cc]};
            }
            tile[hp * CC + cc] = v;
        }
        for (int e = threadIdx.x; e < KK * CC; e += blockDim.x) {
            const int cc = e % CC, t = e / CC;
            su[e] = cc < nc ? U[t * F + c0 + cc] : float2{0.f, 0.f};
        }
        __syncthreads();
        for (int ky = 0; ky < KY; ky++)
            for (int kx = 0; kx < KX; kx++) {
                const float2* tp = tile + ((py + ky) * HX + px + kx) * CC;
                const float2* up = su + (kx + KX * ky) * CC;
#pragma unroll
                for (int cc = 0; cc < CC; cc++) {
                    const float2 t = cmul(tp[cc], up[cc]);
                    acc.x += t.x;
                    acc.y += t.y;
                }
            }
    }
    const int gx = x0 + px, gy = y0 + py;
    if (gx < X && gy < Y)
        out[(b * XY) + gx + long(X) * gy] = acc;
}

// weight gradient with one thin operand.  g is the "dy" side, h the "x" side:
//   dw[t, f] = sum_p g[p, f] conj(h[p + t - c0, f])   (the wide side carries f)
// thin_is_h: h is the 1-channel image (1 -> F layer), else g is (F -> 1 layer).
// Block = pixel tile; thread (f, lane); K^2 accumulators per thread; partials
// per block [block][t][f] reduced in fixed order by k_thin_wsum.
__global__ void __launch_bounds__(256) k_thin_wgrad(float2* __restrict__ part, const float2* __restrict__ g_thin,
                                                    const float* __restrict__ g_wide, const float2* __restrict__ h_thin,
                                                    const float* __restrict__ h_wide, int X, int Y, int F, int KX,
                                                    int KY, int c0x, int c0y, bool thin_is_h)
{
    __shared__ float2 tile[(TY + MAXK - 1) * (TX + MAXK - 1)];
    const int KK = KX * KY;
    const int HX = TX + KX - 1, HY = TY + KY - 1;
    const long b = blockIdx.z;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const long XY = long(X) * Y;
    // thin operand tile: for thin h, the halo of h; for thin g, just the tile (no halo)
    if (thin_is_h) {
        for (int e = threadIdx.x; e < HX * HY; e += blockDim.x) {
            const int hx = e % HX, hy = e / HX;
            const int gx = x0 + hx - c0x, gy = y0 + hy - c0y;
            tile[e] = (gx >= 0 && gx < X && gy >= 0 && gy < Y) ? h_thin[gx + long(X) * gy + XY * b] : float2{0.f, 0.f};
        }
    } else {
        for (int e = threadIdx.x; e < TX * TY; e += blockDim.x) {
            const int gx = x0 + e % TX, gy = y0 + e / TX;
            tile[e] = (gx < X && gy < Y) ? g_thin[gx + long(X) * gy + XY * b] : float2{0.f, 0.f};
        }
    }
    __syncthreads();
    const int lanes = blockDim.x / F;
    const int f = threadIdx.x % F, pl = threadIdx.x / F;
    constexpr int NA = MAXK * MAXK;
    float2 acc[NA];
#pragma unroll
    for (int t = 0; t < NA; t++)
        acc[t] = float2{0.f, 0.f};
    if (pl < lanes) {
        for (int pix = pl; pix < TX * TY; pix += lanes) {
            const int px = pix % TX, py = pix / TX;
            const int gx = x0 + px, gy = y0 + py;
            if (gx >= X || gy >= Y)
                continue;
            if (thin_is_h) {
                const float* gw = g_wide + ((b * XY) + gx + long(X) * gy) * 2 * F;
                const float2 gv{gw[f], gw[F + f]};
#pragma unroll
                for (int t = 0; t < NA; t++) {
                    if (t >= KK)
                        break;
                    const int kx = t % KX, ky = t / KX;
                    const float2 hv = tile[(py + ky) * HX + px + kx];
                    acc[t].x += gv.x * hv.x + gv.y * hv.y;
                    acc[t].y += gv.y * hv.x - gv.x * hv.y;
                }
            } else {
                const float2 gv = tile[py * TX + px];
#pragma unroll
                for (int t = 0; t < NA; t++) {
                    if (t >= KK)
                        break;
                    const int kx = t % KX, ky = t / KX;
                    const int hx = gx + kx - c0x, hy = gy + ky - c0y;
                    if (hx < 0 || hx >= X || hy < 0 || hy >= Y)
                        continue;
                    const float* hw = h_wide + ((b * XY) + hx + long(X) * hy) * 2 * F;
                    const float2 hv{hw[f], hw[F + f]};
                    acc[t].x += gv.x * hv.x + gv.y * hv.y;
                    acc[t].y += gv.y * hv.x - gv.x * hv.y;
                }
            }
        }
    }
    // reduce the pixel lanes of each f in fixed order through smem
    extern __shared__ float2 sred[]; // [lanes][KK][F]
    if (pl < lanes)
        for (int t = 0; t < KK && t < NA; t++)
            sred[(pl * KK + t) * F + f] = acc[t];
    __syncthreads();
    const long blk = (long(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    for (int e = threadIdx.x; e < KK * F; e += blockDim.x) {
        float2 s{0.f, 0.f};
        for (int l = 0; l < lanes; l++) {
            s.x += sred[l * KK * F + e].x;
            s.y += sred[l * KK * F + e].y;
        }
        part[blk * KK * F + e] = s;
    }
}

__global__ void k_thin_wsum(float2* __restrict__ dw, const float2* __restrict__ part, long nblk, int KK, int F,
                            bool f_is_cout)
{
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < KK * F; e += gridDim.x * blockDim.x) {
        double sr = 0, si = 0;
        for (long k = 0; k < nblk; k++) {
            sr += part[k * KK * F + e].x;
            si += part[k * KK * F + e].y;
        }
        const int t = e / F, f = e % F;
        // w dims [KX, KY, Cin, Cout]: 1 -> F: index t + KK * f; F -> 1: t + KK * c
        (void)f_is_cout;
        dw[t + long(KK) * f] = float2{float(sr), float(si)};
    }
}

} // namespace

bool conv_thin_supported(const ConvGeom& g)
{
    const bool one_in = g.Cin == 1, one_out = g.Cout == 1;
    const long F = one_in ? g.Cout : g.Cin;
    if (one_in == one_out || F > MAXF || 256 % F != 0 || g.KX > MAXK || g.KY > MAXK || g.KX * g.KY > 25)
        return false;
    // the wide side must be channels-last (the thin side is layout-free)
    return one_in ? g.out_chlast : g.in_chlast;
}

// mode: 0 fwd, 1 bwd-data
void conv_thin_run(cfloat* outp, const cfloat* inp, const cfloat* w, const ConvGeom& g, int mode)
{
    auto& c = ctx();
    const bool one_in = g.Cin == 1;
    const int F = int(one_in ? g.Cout : g.Cin);
    const int KK = int(g.KX * g.KY);
    // expand (thin -> wide): fwd of 1->F, bwd-data of F->1; reduce otherwise
    const bool expand = (mode == 0) == one_in;
    const int pmode = mode == 0 ? (one_in ? 0 : 2) : (one_in ? 3 : 1);
    float2* U;
    CUDA_CHECK(cudaMallocAsync(&U, sizeof(float2) * KK * F, c.stream));
    k_pack_thin<<<std::max(1, (KK * F + 255) / 256), 256, 0, c.stream>>>(U, w, int(g.KX), int(g.KY), F, pmode);
    KERNEL_CHECK();
    // window offset: forward reads p + t - c0; adjoints use flipped taps with offset K-1-c0
    const int ox = mode == 0 ? int(g.px) : int(g.KX - 1 - g.px);
    const int oy = mode == 0 ? int(g.py) : int(g.KY - 1 - g.py);
    dim3 grid(unsigned((g.X + TX - 1) / TX), unsigned((g.Y + TY - 1) / TY), unsigned(g.B));
    // HBM-bound: algorithmic bytes = wide side once + thin side once
    ProfScope prof(mode == 0 ? "conv_thin_fwd" : "conv_thin_bwd_data", 8.0 * double(g.X) * g.Y * g.B * (F + 1));
    if (expand)
        k_thin_expand<<<grid, 256, sizeof(float2) * KK * F, c.stream>>>(reinterpret_cast<float*>(outp), inp, U,
                                                                       int(g.X), int(g.Y), F, int(g.KX), int(g.KY), ox,
                                                                       oy);
    else
        k_thin_reduce<<<grid, TX * TY, 0, c.stream>>>(outp, reinterpret_cast<const float*>(inp), U, int(g.X),
                                                      int(g.Y), F, int(g.KX), int(g.KY), ox, oy);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(U, c.stream));
}

// dw[t, c, f] = sum_p dy[p, f] conj(x[p + t - c0, c]) with one thin side
void conv_thin_wgrad(cfloat* dw, const cfloat* x, const cfloat* dy, const ConvGeom& g)
{
    auto& c = ctx();
    const bool one_in = g.Cin == 1;
    const int F = int(one_in ? g.Cout : g.Cin);
    const int KK = int(g.KX * g.KY);
    dim3 grid(unsigned((g.X + TX - 1) / TX), unsigned((g.Y + TY - 1) / TY), unsigned(g.B));
    const long nblk = long(grid.x) * grid.y * grid.z;
    const int lanes = 256 / F;
    float2* part;
    CUDA_CHECK(cudaMallocAsync(&part, sizeof(float2) * nblk * KK * F, c.stream));
    ProfScope prof("conv_thin_bwd_weight", 8.0 * double(g.X) * g.Y * g.B * (F + 1));
    const size_t smem = sizeof(float2) * size_t(lanes) * KK * F;
    if (one_in) // h = x thin, g = dy wide
        k_thin_wgrad<<<grid, 256, smem, c.stream>>>(part, nullptr, reinterpret_cast<const float*>(dy), x, nullptr,
                                                     int(g.X), int(g.Y), F, int(g.KX), int(g.KY), int(g.px),
                                                     int(g.py), true);
    else // g = dy thin, h = x wide
        k_thin_wgrad<<<grid, 256, smem, c.stream>>>(part, dy, nullptr, nullptr, reinterpret_cast<const float*>(x),
                                                     int(g.X), int(g.Y), F, int(g.KX), int(g.KY), int(g.px),
                                                     int(g.py), false);
    KERNEL_CHECK();
    k_thin_wsum<<<std::max(1, (KK * F + 255) / 256), 256, 0, c.stream>>>(dw, part, nblk, KK, F, one_in);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(part, c.stream));
}

} // namespace mdnn
