// Complex "same" cross-correlation layers (conv_layer, nn.hpp:344-426; the
// TenMul wiring of conv_tenmul, nn.hpp:305-337) on CUDA cores.
//
//   fwd        y[p,f]  = sum_{t,c} x[p+t-c0, c] w[t,c,f]
//   bwd-data   dx[q,c] = sum_{t,f} dy[q-t+c0, f] conj(w[t,c,f])
//   bwd-weight dw[t,c,f] = sum_p dy[p,f] conj(x[p+t-c0, c])
//
// Each activation operand may be stored CANON (reference layout) or CHLAST
// (channels-last planar, core.h).  These kernels serve every channel count
// and kernel size (MoDL 1->F / F->1, VarNet 2->24 / 24->2 at 11x11); 3x3
// layers with 32/64 channels go to the tcgen05 path (conv_tc.cu).
// Reductions are fixed-order (no atomics): bitwise run-to-run stable.
#include "kernels.h"
#include "profile.h"

#include <algorithm>

namespace mdnn {

namespace {

constexpr int TX = 32, TY = 8;   // output tile (pixels)
constexpr int MAXK = 11;
// output channels per block: 8, or exactly 2 for the VarNet 24 -> 2 adjoint
inline int fg_for(long nout) { return nout <= 2 ? 2 : 8; }

// element (item b, pixel xy = x + X*y, channel c) of a C-channel tensor
struct Acc {
    const cfloat* p;
    long C, XY;
    bool chl;
    __device__ __forceinline__ float2 ld(long b, long xy, long c) const
    {
        if (chl) {
            const float* f = reinterpret_cast<const float*>(p) + (b * XY + xy) * 2 * C;
            return float2{f[c], f[C + c]};
        }
        return p[xy + XY * (c + C * b)];
    }
};
struct Out {
    cfloat* p;
    long C, XY;
    bool chl;
    __device__ __forceinline__ void st(long b, long xy, long c, float2 v) const
    {
        if (chl) {
            float* f = reinterpret_cast<float*>(p) + (b * XY + xy) * 2 * C;
            f[c] = v.x;
            f[C + c] = v.y;
        } else {
            p[xy + XY * (c + C * b)] = v;
        }
    }
};

// Real-operand fast path.  VarNet's convolutions see real data throughout
// (RealChan output, RBF output, real-valued weights by the real_weights flag):
// a complex MAC with Im = 0 on both sides reduces to one real FMA whose
// result is bitwise the real part the complex formula produces (the extra
// products are exact zeros), and the imaginary part is zero.  A tiny kernel
// raises a device flag if any operand element has a nonzero imaginary part;
// the conv kernels read it (block-uniform) and pick the complex or the real
// inner loop — no host synchronisation, any complex input takes the full path.
__global__ void k_imag_any(const float2* __restrict__ a, long n, unsigned* flag)
{
    MDNN_PDL_ENTRY();
    int any = 0;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        any |= a[i].y != 0.f;
    any = __syncthreads_or(any);
    if (any && threadIdx.x == 0)
        atomicOr(flag, 1u);
}

// mode 0: fwd (in = x, Cin in, weights w[t,c,f]); mode 1: bwd-data (in = dy,
// channels Cout, weights conj(w[t,c,f]) flipped, output channel c)
template<int MODE, int FG>
__global__ void __launch_bounds__(TX* TY) k_conv_direct(Out out, Acc in, const cfloat* __restrict__ w, ConvGeom g,
                                                        const unsigned* __restrict__ imag_flag, int skip_real)
{
    MDNN_PDL_ENTRY();
    const bool real = imag_flag && *imag_flag == 0;
    if (real && skip_real)
        return; // real operands: k_conv_direct_real computed this launch
    __shared__ float2 tile[TY + MAXK - 1][TX + MAXK - 1];
    __shared__ float2 wsh[MAXK * MAXK][FG];
    // real parts of the taps' weights, FG contiguous floats per tap (16-B aligned rows):
    // the real-operand loop reads them as float4 / float2 (3 loads per 8 FMAs instead of 9)
    __shared__ __align__(16) float wre[MAXK * MAXK][FG];
    const long nin = MODE == 0 ? g.Cin : g.Cout;
    const long nout = MODE == 0 ? g.Cout : g.Cin;
    const long ngrp = (nout + FG - 1) / FG;
    const long b = blockIdx.z / ngrp;
    const long f0 = (blockIdx.z % ngrp) * FG;
    const long x0 = long(blockIdx.x) * TX, y0 = long(blockIdx.y) * TY;
    const int KX = int(g.KX), KY = int(g.KY);
    // input window offset: fwd in[p + t - c0]; bwd in[q - t + c0] = in[q + t' - (K-1-c0)]
    const long ox = MODE == 0 ? g.px : (g.KX - 1 - g.px);
    const long oy = MODE == 0 ? g.py : (g.KY - 1 - g.py);
    const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
    float2 acc[FG];
#pragma unroll
    for (int f = 0; f < FG; f++)
        acc[f] = float2{0.f, 0.f};
    const int HX = TX + KX - 1, HY = TY + KY - 1;
    for (long c = 0; c < nin; c++) {
        for (int e = threadIdx.x; e < HX * HY; e += blockDim.x) {
            int hx = e % HX, hy = e / HX;
            long gx = x0 + hx - ox, gy = y0 + hy - oy;
            tile[hy][hx] = (gx >= 0 && gx < g.X && gy >= 0 && gy < g.Y) ? in.ld(b, gx + g.X * gy, c)
                                                                       : float2{0.f, 0.f};
        }
        for (int e = threadIdx.x; e < KX * KY * FG; e += blockDim.x) {
            int t = e % (KX * KY), f = e / (KX * KY);
            long fo = f0 + f;
            float2 v{0.f, 0.f};
            if (fo < nout) {
                if (MODE == 0) {
                    v = w[t + g.KX * g.KY * (c + g.Cin * fo)];
                } else {
                    int tpx = t % KX, tpy = t / KX;
                    long tt = (KX - 1 - tpx) + g.KX * (KY - 1 - tpy);
                    float2 ww = w[tt + g.KX * g.KY * (fo + g.Cin * c)];
                    v = float2{ww.x, -ww.y};
                }
            }
            wsh[t][f] = v;
            wre[t][f] = v.x;
        }
        __syncthreads();
        if (real) {
            for (int ky = 0; ky < KY; ky++)
                for (int kx = 0; kx < KX; kx++) {
                    const float xr = tile[ty + ky][tx + kx].x;
                    const int t = kx + KX * ky;
                    float wv[FG];
                    if constexpr (FG % 4 == 0) {
#pragma unroll
                        for (int f = 0; f < FG; f += 4) {
                            const float4 q = *reinterpret_cast<const float4*>(&wre[t][f]);
                            wv[f] = q.x;
                            wv[f + 1] = q.y;
                            wv[f + 2] = q.z;
                            wv[f + 3] = q.w;
                        }
                    } else if constexpr (FG % 2 == 0) {
#pragma unroll
                        for (int f = 0; f < FG; f += 2) {
                            const float2 q = *reinterpret_cast<const float2*>(&wre[t][f]);
                            wv[f] = q.x;
                            wv[f + 1] = q.y;
                        }
                    } else {
#pragma unroll
                        for (int f = 0; f < FG; f++)
                            wv[f] = wre[t][f];
                    }
#pragma unroll
                    for (int f = 0; f < FG; f++)
                        acc[f].x = fmaf(xr, wv[f], acc[f].x);
                }
        } else {
            for (int ky = 0; ky < KY; ky++)
                for (int kx = 0; kx < KX; kx++) {
                    float2 xv = tile[ty + ky][tx + kx];
                    const int t = kx + KX * ky;
#pragma unroll
                    for (int f = 0; f < FG; f++) {
                        float2 wv = wsh[t][f];
                        acc[f].x = fmaf(xv.x, wv.x, fmaf(-xv.y, wv.y, acc[f].x));
                        acc[f].y = fmaf(xv.x, wv.y, fmaf(xv.y, wv.x, acc[f].y));
                    }
                }
        }
        __syncthreads();
    }
    const long px = x0 + tx, py = y0 + ty;
    if (px < g.X && py < g.Y)
#pragma unroll
        for (int f = 0; f < FG; f++)
            if (f0 + f < nout)
                out.st(b, px + g.X * py, f0 + f, acc[f]);
}

// Real-operand path (VarNet: real images and real-valued weights stored complex)
// register-blocked along x: a thread owns RPX consecutive output pixels and FG
// output channels; per (channel, kernel row) it loads a window of RPX + KX - 1
// real inputs once and slides over the KX taps with float4 weight rows, so a
// tap costs (RPX + FG/4 + ...)/(RPX * FG) loads per FMA instead of ~1.
// Launched alongside k_conv_direct; exactly one of the two does the work
// (device-side imaginary-part flag, no host synchronisation).
constexpr int RTX = 16, RTY = 16; // 16 x 16 threads; RPX x 16 pixels... per block: (16 RPX) x 16 outputs
// RPX pixels per thread (8 for FG = 2 measured no faster than 4)
template<int FG>
constexpr int rpx_for() { return 4; }

template<int MODE, int FG, int RPX = rpx_for<FG>()>
__global__ void __launch_bounds__(RTX* RTY) k_conv_direct_real(Out out, Acc in, const cfloat* __restrict__ w,
                                                              ConvGeom g, const unsigned* __restrict__ imag_flag)
{
    MDNN_PDL_ENTRY();
    if (*imag_flag != 0)
        return; // complex operands: k_conv_direct computes this launch
    constexpr int OX = RTX * RPX, OY = RTY;
    // row pitch rounded up to a float4 multiple (+4): the sliding window of
    // RPX + KX - 1 values is read as 16-B vectors (scalar reads 4 words apart
    // were bank-conflicted and issue-bound)
    constexpr int HXP = ((OX + MAXK - 1 + 3) / 4) * 4 + 4;
    constexpr int NV4 = (RPX + MAXK - 1 + 3) / 4;
    static_assert(RPX % 4 == 0, "the window is read as 16-B vectors from tx * RPX");
    __shared__ __align__(16) float tile[OY + MAXK - 1][HXP];
    __shared__ __align__(16) float wre[MAXK * MAXK][FG];
    const long nin = MODE == 0 ? g.Cin : g.Cout;
    const long nout = MODE == 0 ? g.Cout : g.Cin;
    const long ngrp = (nout + FG - 1) / FG;
    const long b = blockIdx.z / ngrp;
    const long f0 = (blockIdx.z % ngrp) * FG;
    const long x0 = long(blockIdx.x) * OX, y0 = long(blockIdx.y) * OY;
    const int KX = int(g.KX), KY = int(g.KY);
    const long ox = MODE == 0 ? g.px : (g.KX - 1 - g.px);
    const long oy = MODE == 0 ? g.py : (g.KY - 1 - g.py);
    const int tx = threadIdx.x % RTX, ty = threadIdx.x / RTX;
    float acc[RPX][FG];
#pragma unroll
    for (int p = 0; p < RPX; p++)
#pragma unroll
        for (int f = 0; f < FG; f++)
            acc[p][f] = 0.f;
    const int HX = OX + KX - 1, HY = OY + KY - 1;
    for (long c = 0; c < nin; c++) {
        __syncthreads();
        for (int e = threadIdx.x; e < HX * HY; e += blockDim.x) {
            const int hx = e % HX, hy = e / HX;
            const long gx = x0 + hx - ox, gy = y0 + hy - oy;
            tile[hy][hx] = (gx >= 0 && gx < g.X && gy >= 0 && gy < g.Y) ? in.ld(b, gx + g.X * gy, c).x : 0.f;
        }
        for (int e = threadIdx.x; e < KX * KY * FG; e += blockDim.x) {
            const int t = e % (KX * KY), f = e / (KX * KY);
            const long fo = f0 + f;
            float v = 0.f;
            if (fo < nout) {
                if (MODE == 0) {
                    v = w[t + g.KX * g.KY * (c + g.Cin * fo)].x;
                } else {
                    const int tpx = t % KX, tpy = t / KX;
                    const long tt = (KX - 1 - tpx) + g.KX * (KY - 1 - tpy);
                    v = w[tt + g.KX * g.KY * (fo + g.Cin * c)].x; // conj: real part unchanged
                }
            }
            wre[t][f] = v;
        }
        __syncthreads();
        for (int ky = 0; ky < KY; ky++) {
            float win[4 * NV4];
            const float4* trow = reinterpret_cast<const float4*>(&tile[ty + ky][tx * RPX]);
#pragma unroll
            for (int v4 = 0; v4 < NV4; v4++) {
                const float4 q4 = trow[v4];
                win[4 * v4] = q4.x;
                win[4 * v4 + 1] = q4.y;
                win[4 * v4 + 2] = q4.z;
                win[4 * v4 + 3] = q4.w;
            }
#pragma unroll
            for (int kx = 0; kx < MAXK; kx++) {
                if (kx >= KX)
                    break;
                const int t = kx + KX * ky;
                float wv[FG];
                if constexpr (FG % 4 == 0) {
#pragma unroll
                    for (int f = 0; f < FG; f += 4) {
                        const float4 q4 = *reinterpret_cast<const float4*>(&wre[t][f]);
                        wv[f] = q4.x;
                        wv[f + 1] = q4.y;
                        wv[f + 2] = q4.z;
                        wv[f + 3] = q4.w;
                    }
                } else {
#pragma unroll
                    for (int f = 0; f < FG; f += 2) {
                        const float2 q2 = *reinterpret_cast<const float2*>(&wre[t][f]);
                        wv[f] = q2.x;
                        wv[f + 1] = q2.y;
                    }
                }
#pragma unroll
                for (int p = 0; p < RPX; p++)
#pragma unroll
                    for (int f = 0; f < FG; f++)
                        acc[p][f] = fmaf(win[p + kx], wv[f], acc[p][f]);
            }
        }
    }
    const long py = y0 + ty;
    if (py >= g.Y)
        return;
#pragma unroll
    for (int p = 0; p < RPX; p++) {
        const long px = x0 + tx * RPX + p;
        if (px < g.X)
#pragma unroll
            for (int f = 0; f < FG; f++)
                if (f0 + f < nout)
                    out.st(b, px + g.X * py, f0 + f, float2{acc[p][f], 0.f});
    }
}

// bwd-weight: block = (c-group x f-group, split); loops over its share of
// pixel tiles; thread owns combos (t, c, f) accumulated in registers.
constexpr int WTX = 32, WTY = 8;          // pixel tile
constexpr int WMAXC = 4;                  // combos per thread

// WG_C x WG_F channel pairs per block; (4, 8) for 3x3-5x5 kernels, (1, 8) up to 11x11
template<int WG_C, int WG_F>
__global__ void __launch_bounds__(256) k_conv_wgrad(float2* __restrict__ part, Acc x, Acc dy, ConvGeom g, int nsplit)
{
    MDNN_PDL_ENTRY();
    __shared__ float2 xt[WG_C][WTY + MAXK - 1][WTX + MAXK - 1];
    __shared__ float2 dyt[WG_F][WTY][WTX];
    const int KX = int(g.KX), KY = int(g.KY), KK = KX * KY;
    const long ncg = (g.Cin + WG_C - 1) / WG_C;
    const long c0 = (blockIdx.x % ncg) * WG_C;
    const long f0 = (blockIdx.x / ncg) * WG_F;
    const int split = blockIdx.y;
    const long ntx = (g.X + WTX - 1) / WTX, nty = (g.Y + WTY - 1) / WTY;
    const long ntiles = ntx * nty * g.B;
    const int ncombo = KK * WG_C * WG_F;
    const int HX = WTX + KX - 1, HY = WTY + KY - 1;
    float2 acc[WMAXC];
#pragma unroll
    for (int i = 0; i < WMAXC; i++)
        acc[i] = float2{0.f, 0.f};
    for (long tile = split; tile < ntiles; tile += nsplit) {
        const long b = tile / (ntx * nty);
        const long tr = tile % (ntx * nty);
        const long x0 = (tr % ntx) * WTX, y0 = (tr / ntx) * WTY;
        for (int e = threadIdx.x; e < WG_C * HX * HY; e += blockDim.x) {
            int hx = e % HX, hy = (e / HX) % HY, cc = e / (HX * HY);
            long gx = x0 + hx - g.px, gy = y0 + hy - g.py, c = c0 + cc;
            xt[cc][hy][hx] = (c < g.Cin && gx >= 0 && gx < g.X && gy >= 0 && gy < g.Y) ? x.ld(b, gx + g.X * gy, c)
                                                                                        : float2{0.f, 0.f};
        }
        for (int e = threadIdx.x; e < WG_F * WTX * WTY; e += blockDim.x) {
            int px = e % WTX, py = (e / WTX) % WTY, ff = e / (WTX * WTY);
            long gx = x0 + px, gy = y0 + py, f = f0 + ff;
            dyt[ff][py][px] = (f < g.Cout && gx < g.X && gy < g.Y) ? dy.ld(b, gx + g.X * gy, f) : float2{0.f, 0.f};
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < WMAXC; i++) {
            int combo = threadIdx.x + i * blockDim.x;
            if (combo >= ncombo)
                break;
            int t = combo % KK, cc = (combo / KK) % WG_C, ff = combo / (KK * WG_C);
            int kx = t % KX, ky = t / KX;
            float ar = acc[i].x, ai = acc[i].y;
            for (int py = 0; py < WTY; py++)
                for (int px = 0; px < WTX; px++) {
                    float2 d = dyt[ff][py][px];
                    float2 xv = xt[cc][py + ky][px + kx];
                    // d * conj(xv)
                    ar = fmaf(d.x, xv.x, fmaf(d.y, xv.y, ar));
                    ai = fmaf(d.y, xv.x, fmaf(-d.x, xv.y, ai));
                }
            acc[i] = float2{ar, ai};
        }
        __syncthreads();
    }
    for (int i = 0; i < WMAXC; i++) {
        int combo = threadIdx.x + i * blockDim.x;
        if (combo >= ncombo)
            break;
        int t = combo % KK, cc = (combo / KK) % WG_C, ff = combo / (KK * WG_C);
        long c = c0 + cc, f = f0 + ff;
        if (c < g.Cin && f < g.Cout)
            part[size_t(split) * KK * g.Cin * g.Cout + t + KK * (c + g.Cin * f)] = acc[i];
    }
}

// bwd-weight, register-blocked along kx: thread (ky, c, f) keeps the K
// accumulators of one kernel row and slides a K-wide window of x along each
// pixel row (1 dy + 1 x smem load per K complex MACs).  Block = all
// (ky, c, f) combos (K * Cin * Cout <= 576 threads: the VarNet 2 <-> 24
// 11x11 layers); grid = pixel-tile splits, partials folded by k_sum_splits.
// FP output channels per thread share the sliding x window (FP = 2: 3 loads per
// 2K real FMAs instead of 2 per K)
template<int K, int FP>
__global__ void __launch_bounds__(576) k_conv_wgrad_rb(float2* __restrict__ part, Acc x, Acc dy, ConvGeom g,
                                                        int nsplit, const unsigned* __restrict__ imag_flag,
                                                        bool complex_only = false)
{
    MDNN_PDL_ENTRY();
    const bool real = imag_flag && *imag_flag == 0;
    if (complex_only && real) // the tensor-core kernel of this launch pair handles real operands
        return;
    constexpr int HX = WTX + K - 1, HY = WTY + K - 1;
    // odd float2 row pitch: the K kernel-row lanes of a warp read K different rows
    // at the same column; an even pitch (42) mapped several of them to one bank
    constexpr int HXP = HX | 1;
    extern __shared__ float2 wsm[];
    const int Cin = int(g.Cin), Cout = int(g.Cout);
    float2* xt = wsm;                          // [Cin][HY][HX]
    float2* dyt = wsm + Cin * HY * HXP;        // [Cout][WTY][WTX]
    const int nthr = K * Cin * (Cout / FP);
    const int tid = threadIdx.x;
    const int ky = tid % K, c = (tid / K) % Cin, f = (tid / (K * Cin)) * FP;
    const bool act = tid < nthr;
    const long ntx = (g.X + WTX - 1) / WTX, nty = (g.Y + WTY - 1) / WTY;
    const long ntiles = ntx * nty * g.B;
    float2 acc[FP][K];
#pragma unroll
    for (int q = 0; q < FP; q++)
#pragma unroll
        for (int k = 0; k < K; k++)
            acc[q][k] = float2{0.f, 0.f};
    for (long tile = blockIdx.x; tile < ntiles; tile += nsplit) {
        const long b = tile / (ntx * nty);
        const long tr = tile % (ntx * nty);
        const long x0 = (tr % ntx) * WTX, y0 = (tr / ntx) * WTY;
        __syncthreads();
        for (int e = tid; e < Cin * HX * HY; e += blockDim.x) {
            const int hx = e % HX, hy = (e / HX) % HY, cc = e / (HX * HY);
            const long gx = x0 + hx - g.px, gy = y0 + hy - g.py;
            xt[(cc * HY + hy) * HXP + hx] =
                (gx >= 0 && gx < g.X && gy >= 0 && gy < g.Y) ? x.ld(b, gx + g.X * gy, cc) : float2{0.f, 0.f};
        }
        for (int e = tid; e < Cout * WTX * WTY; e += blockDim.x) {
            const int px = e % WTX, py = (e / WTX) % WTY, ff = e / (WTX * WTY);
            const long gx = x0 + px, gy = y0 + py;
            dyt[e] = (gx < g.X && gy < g.Y) ? dy.ld(b, gx + g.X * gy, ff) : float2{0.f, 0.f};
        }
        __syncthreads();
        if (!act)
            continue;
        for (int py = 0; py < WTY; py++) {
            const float2* xr = xt + (c * HY + py + ky) * HXP;
            const float2* dr = dyt + (f * WTY + py) * WTX;
            float2 win[K];
#pragma unroll
            for (int k = 0; k < K - 1; k++)
                win[k] = xr[k];
            if (real) {
#pragma unroll 4
                for (int px = 0; px < WTX; px++) {
                    win[K - 1] = xr[px + K - 1];
#pragma unroll
                    for (int q = 0; q < FP; q++) {
                        const float d = dr[q * WTY * WTX + px].x;
#pragma unroll
                        for (int kx = 0; kx < K; kx++)
                            acc[q][kx].x = fmaf(d, win[kx].x, acc[q][kx].x);
                    }
#pragma unroll
                    for (int k = 0; k < K - 1; k++)
                        win[k] = win[k + 1];
                }
            } else {
#pragma unroll 4
                for (int px = 0; px < WTX; px++) {
                    win[K - 1] = xr[px + K - 1];
#pragma unroll
                    for (int q = 0; q < FP; q++) {
                        const float2 d = dr[q * WTY * WTX + px];
#pragma unroll
                        for (int kx = 0; kx < K; kx++) { // acc[kx] += d * conj(x[px + kx])
                            acc[q][kx].x = fmaf(d.x, win[kx].x, acc[q][kx].x);
                            acc[q][kx].y = fmaf(d.y, win[kx].x, acc[q][kx].y);
                            acc[q][kx].x = fmaf(d.y, win[kx].y, acc[q][kx].x);
                            acc[q][kx].y = fmaf(-d.x, win[kx].y, acc[q][kx].y);
                        }
                    }
#pragma unroll
                    for (int k = 0; k < K - 1; k++)
                        win[k] = win[k + 1];
                }
            }
        }
    }
    if (act) {
        const long KK = long(K) * K;
#pragma unroll
        for (int q = 0; q < FP; q++)
#pragma unroll
            for (int kx = 0; kx < K; kx++)
                part[size_t(blockIdx.x) * KK * Cin * Cout + (kx + K * ky) + KK * (c + long(Cin) * (f + q))] =
                    acc[q][kx];
    }
}

// out[i] = sum_s part[s][i]: block = 64 outputs x 4 split groups (group g sums
// splits g, g + 4, ... in order; the groups are added in order): the serial
// per-output loop over ~300 splits was latency-bound
__global__ void __launch_bounds__(256) k_sum_splits(cfloat* out, const float2* part, long n, int nsplit,
                                                    const unsigned* __restrict__ complex_only = nullptr)
{
    MDNN_PDL_ENTRY();
    if (complex_only && *complex_only == 0)
        return;
    __shared__ double2 red[4][64];
    const int o = threadIdx.x & 63, gq = threadIdx.x >> 6;
    const long i = long(blockIdx.x) * 64 + o;
    double ar = 0, ai = 0;
    if (i < n) {
#pragma unroll 4
        for (int s = gq; s < nsplit; s += 4) {
            const float2 v = part[size_t(s) * n + i];
            ar += v.x;
            ai += v.y;
        }
    }
    red[gq][o] = double2{ar, ai};
    __syncthreads();
    if (gq == 0 && i < n) {
        double2 r = red[0][o];
        for (int k = 1; k < 4; k++) {
            r.x += red[k][o].x;
            r.y += red[k][o].y;
        }
        out[i] = float2{float(r.x), float(r.y)};
    }
}

// algorithmic flops of one pass: 8 per complex MAC, or 2 per
// real MAC when the host knows both operands are real (VarNet)
double conv_flops(const ConvGeom& g, bool real = false)
{
    return (real ? 2.0 : 8.0) * double(g.X) * g.Y * g.B * g.Cin * g.Cout * g.KX * g.KY;
}

void check_geom(const ConvGeom& g)
{
    if (g.KX > MAXK || g.KY > MAXK)
        throw ConfigError("conv: kernel extent > 11 not supported on device");
}

// device flag: 1 if any of the operands has a nonzero imaginary part
unsigned* imag_flag(std::initializer_list<std::pair<const cfloat*, long>> ops)
{
    auto& c = ctx();
    unsigned* f;
    CUDA_CHECK(cudaMallocAsync(&f, sizeof(unsigned), c.stream));
    CUDA_CHECK(cudaMemsetAsync(f, 0, sizeof(unsigned), c.stream));
    for (auto [p, n] : ops) {
        pdl_launch(k_imag_any, int(std::min<long>((n + 255) / 256, 2L * c.sm_count)), 256, 0, c.stream, p, n, f);
        KERNEL_CHECK();
    }
    return f;
}

} // namespace

long conv_epi_blocks(const ConvGeom& g, int mode)
{
    if (conv_tc_supported(g.Cin, g.Cout, g.KX, g.KY))
        return long(ctx().sm_count) * conv_tc_stat_slots();
    if (conv_thin_supported(g))
        return conv_thin_epi_blocks(g, mode);
    return 0;
}

void conv_fwd(cfloat* y, const cfloat* x, const cfloat* w, const ConvGeom& g)
{
    check_geom(g);
    if (conv_tc_supported(g.Cin, g.Cout, g.KX, g.KY)) {
        conv_tc_run(y, x, w, g, 0);
        return;
    }
    if (conv_thin_supported(g)) {
        conv_thin_run(y, x, w, g, 0);
        return;
    }
    const int FGv = fg_for(g.Cout);
    dim3 grid(unsigned((g.X + TX - 1) / TX), unsigned((g.Y + TY - 1) / TY),
              unsigned(g.B * ((g.Cout + FGv - 1) / FGv)));
    const long XY = g.X * g.Y;
    const bool known = (g.real_known & 3) == 3;
    ProfScope prof("conv_fwd", conv_flops(g, known));
    unsigned* fl = known ? ctx().d_zero : imag_flag({{x, XY * g.Cin * g.B}, {w, g.KX * g.KY * g.Cin * g.Cout}});
    if (conv_vn_tc_supported(g)) {
        conv_vn_tc_run(y, x, w, g, 0, fl);
    } else {
        const int RP = FGv == 2 ? rpx_for<2>() : rpx_for<8>();
        dim3 rgrid(unsigned((g.X + RTX * RP - 1) / (RTX * RP)), unsigned((g.Y + RTY - 1) / RTY),
                   unsigned(g.B * ((g.Cout + FGv - 1) / FGv)));
        if (FGv == 2)
            pdl_launch(k_conv_direct_real<0, 2>, rgrid, RTX * RTY, 0, ctx().stream, Out{y, g.Cout, XY, g.out_chlast},
                                                                          Acc{x, g.Cin, XY, g.in_chlast}, w, g, fl);
        else
            pdl_launch(k_conv_direct_real<0, 8>, rgrid, RTX * RTY, 0, ctx().stream, Out{y, g.Cout, XY, g.out_chlast},
                                                                          Acc{x, g.Cin, XY, g.in_chlast}, w, g, fl);
        KERNEL_CHECK();
    }
    if (FGv == 2)
        pdl_launch(k_conv_direct<0, 2>, grid, TX * TY, 0, ctx().stream, Out{y, g.Cout, XY, g.out_chlast},
                                                                Acc{x, g.Cin, XY, g.in_chlast}, w, g, fl, 1);
    else
        pdl_launch(k_conv_direct<0, 8>, grid, TX * TY, 0, ctx().stream, Out{y, g.Cout, XY, g.out_chlast},
                                                                Acc{x, g.Cin, XY, g.in_chlast}, w, g, fl, 1);
    KERNEL_CHECK();
    if (!known)
        CUDA_CHECK(cudaFreeAsync(fl, ctx().stream));
}

void conv_bwd_data(cfloat* dx, const cfloat* dy, const cfloat* w, const ConvGeom& g)
{
    check_geom(g);
    if (conv_tc_supported(g.Cin, g.Cout, g.KX, g.KY)) {
        conv_tc_run(dx, dy, w, g, 1);
        return;
    }
    if (conv_thin_supported(g)) {
        conv_thin_run(dx, dy, w, g, 1);
        return;
    }
    const int FGv = fg_for(g.Cin);
    dim3 grid(unsigned((g.X + TX - 1) / TX), unsigned((g.Y + TY - 1) / TY),
              unsigned(g.B * ((g.Cin + FGv - 1) / FGv)));
    const long XY = g.X * g.Y;
    const bool known = (g.real_known & 6) == 6;
    ProfScope prof("conv_bwd_data", conv_flops(g, known));
    unsigned* fl = known ? ctx().d_zero : imag_flag({{dy, XY * g.Cout * g.B}, {w, g.KX * g.KY * g.Cin * g.Cout}});
    if (conv_vn_tc_supported(g)) {
        conv_vn_tc_run(dx, dy, w, g, 1, fl);
    } else {
        const int RP = FGv == 2 ? rpx_for<2>() : rpx_for<8>();
        dim3 rgrid(unsigned((g.X + RTX * RP - 1) / (RTX * RP)), unsigned((g.Y + RTY - 1) / RTY),
                   unsigned(g.B * ((g.Cin + FGv - 1) / FGv)));
        if (FGv == 2)
            pdl_launch(k_conv_direct_real<1, 2>, rgrid, RTX * RTY, 0, ctx().stream, Out{dx, g.Cin, XY, g.in_chlast},
                                                                          Acc{dy, g.Cout, XY, g.out_chlast}, w, g, fl);
        else
            pdl_launch(k_conv_direct_real<1, 8>, rgrid, RTX * RTY, 0, ctx().stream, Out{dx, g.Cin, XY, g.in_chlast},
                                                                          Acc{dy, g.Cout, XY, g.out_chlast}, w, g, fl);
        KERNEL_CHECK();
    }
    if (FGv == 2)
        pdl_launch(k_conv_direct<1, 2>, grid, TX * TY, 0, ctx().stream, Out{dx, g.Cin, XY, g.in_chlast},
                                                                Acc{dy, g.Cout, XY, g.out_chlast}, w, g, fl, 1);
    else
        pdl_launch(k_conv_direct<1, 8>, grid, TX * TY, 0, ctx().stream, Out{dx, g.Cin, XY, g.in_chlast},
                                                                Acc{dy, g.Cout, XY, g.out_chlast}, w, g, fl, 1);
    KERNEL_CHECK();
    if (!known)
        CUDA_CHECK(cudaFreeAsync(fl, ctx().stream));
}

void conv_bwd_weight(cfloat* dw, const cfloat* x, const cfloat* dy, const ConvGeom& g)
{
    check_geom(g);
    if (conv_tc_wgrad_supported(g.Cin, g.Cout, g.KX, g.KY)) {
        conv_tc_wgrad(dw, x, dy, g);
        return;
    }
    if (conv_thin_supported(g)) {
        conv_thin_wgrad(dw, x, dy, g);
        return;
    }
    const long KK = g.KX * g.KY;
    if (g.KX == 11 && g.KY == 11 && 11 * g.Cin * g.Cout <= 576) {
        // VarNet K = 11 layers: tensor cores for real operands (conv_vn_tc.cu),
        // the register-blocked CUDA-core kernel for complex ones; with operands not
        // known real on the host both are launched and the device imag flag picks
        auto& c = ctx();
        const long XY = g.X * g.Y;
        const bool known = (g.real_known & 5) == 5;
        const bool tc = conv_vn_tc_supported(g);
        unsigned* fl = known ? c.d_zero : imag_flag({{x, XY * g.Cin * g.B}, {dy, XY * g.Cout * g.B}});
        if (tc)
            conv_vn_tc_wgrad(dw, x, dy, g, fl);
        if (!tc || !known) {
            const long ntiles = ((g.X + WTX - 1) / WTX) * ((g.Y + WTY - 1) / WTY) * g.B;
            const int nsplit = int(std::min<long>(ntiles, 2L * c.sm_count));
            const long n = KK * g.Cin * g.Cout;
            const size_t smem = sizeof(float2) * (g.Cin * (WTY + 10) * ((WTX + 10) | 1) + g.Cout * WTX * WTY);
            float2* part;
            CUDA_CHECK(cudaMallocAsync(&part, sizeof(float2) * n * nsplit, c.stream));
            ProfScope prof("conv_bwd_weight", conv_flops(g, known));
            const bool fp2 = g.Cout % 2 == 0;
            auto kern = fp2 ? k_conv_wgrad_rb<11, 2> : k_conv_wgrad_rb<11, 1>;
            allow_max_dyn_smem(reinterpret_cast<const void*>(kern));
            const int nthr = int(((11 * g.Cin * (fp2 ? g.Cout / 2 : g.Cout) + 31) / 32) * 32);
            pdl_launch(kern, nsplit, nthr, smem, c.stream, part, Acc{x, g.Cin, XY, g.in_chlast},
                                                  Acc{dy, g.Cout, XY, g.out_chlast}, g, nsplit, fl, tc);
            KERNEL_CHECK();
            pdl_launch(k_sum_splits, int((n + 63) / 64), 256, 0, c.stream, dw, part, n, nsplit, tc ? fl : nullptr);
            KERNEL_CHECK();
            CUDA_CHECK(cudaFreeAsync(part, c.stream));
        }
        if (!known)
            CUDA_CHECK(cudaFreeAsync(fl, c.stream));
        return;
    }
    const bool small_k = KK * 4 * 8 <= 256 * WMAXC;
    const int WG_C = small_k ? 4 : 1, WG_F = 8;
    if (KK * WG_C * WG_F > 256 * WMAXC)
        throw ConfigError("conv: kernel too large for the weight-gradient kernel");
    const long ngroups = ((g.Cin + WG_C - 1) / WG_C) * ((g.Cout + WG_F - 1) / WG_F);
    const long ntiles = ((g.X + WTX - 1) / WTX) * ((g.Y + WTY - 1) / WTY) * g.B;
    long target = long(ctx().sm_count) * 4;
    int nsplit = int(std::max(1L, std::min(ntiles, (target + ngroups - 1) / ngroups)));
    const long n = KK * g.Cin * g.Cout;
    const long XY = g.X * g.Y;
    auto& c = ctx();
    float2* part;
    CUDA_CHECK(cudaMallocAsync(&part, sizeof(float2) * n * nsplit, c.stream));
    dim3 grid{unsigned(ngroups), unsigned(nsplit)};
    ProfScope prof("conv_bwd_weight", conv_flops(g));
    Acc ax{x, g.Cin, XY, g.in_chlast}, ad{dy, g.Cout, XY, g.out_chlast};
    if (small_k)
        pdl_launch(k_conv_wgrad<4, 8>, grid, 256, 0, c.stream, part, ax, ad, g, nsplit);
    else
        pdl_launch(k_conv_wgrad<1, 8>, grid, 256, 0, c.stream, part, ax, ad, g, nsplit);
    KERNEL_CHECK();
    pdl_launch(k_sum_splits, int((n + 63) / 64), 256, 0, c.stream, dw, part, n, nsplit, nullptr);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(part, c.stream));
}

} // namespace mdnn
