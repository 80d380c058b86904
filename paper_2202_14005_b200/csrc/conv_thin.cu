// "Thin" complex convolutions: one side has a single channel (MoDL's first
// layer 1 -> F and last layer F -> 1, conv_layer nn.hpp:344-426).  The wide
// side is channels-last (CHLAST), the thin side is a plain image (for one
// channel the two layouts coincide).  With 9 complex MACs per wide element
// these passes sit between the HBM and the FP32 roofline, so every kernel
// streams the wide tensor exactly once, coalesced, and keeps the thin image in
// shared memory:
//
//   expand  out[p, f] = sum_t thin[p + t - o] * U[t, f]
//           thread = (channel f, row segment); U[., f] in registers; a K x K
//           register window slides along x (K smem loads per output pixel).
//   reduce  out[q]    = sum_t z_t[q + t - o],  z_t[h] = sum_c wide[h, c] U[t, c]
//           per halo pixel the K^2 tap projections over all channels (channel
//           chunks staged through smem, U broadcast), then a K^2 gather.
//   wgrad   dw[t, f]  = sum_p g[p, f] conj(h[p + t - c0])  (one of g / h wide)
//           persistent CTAs, thread = (channel, row segment), K^2 register
//           accumulators, the thin operand as a sliding register window; per-CTA
//           partials folded in a fixed order (bitwise run-to-run stable).
// U is a per-launch packing of w (or its flipped conjugate for the adjoints).
#include "kernels.h"
#include "profile.h"

#include <algorithm>

namespace mdnn {

namespace {

constexpr int TX = 32, NT = 256, MAXF = 256;
// CTAs per SM the 3x3 weight-gradient kernels are built for: 3 (80 registers, ~100 B
// spilled) beat 2 (128 registers): 3.61 -> 3.37 ms per two C2 steps; the expand
// kernel at 3 lost more (2.66 -> 2.85 ms) and keeps 2
#define THIN_WG_MINB(K) ((K) == 3 ? 3 : 1)

// U[t][f] for the 4 uses; w has dims [KX, KY, Cin, Cout]
//   mode 0: fwd 1 -> F           U[t][f] = w[t, 0, f]
//   mode 1: bwd-data of F -> 1   U[t][c] = conj(w[flip t, c, 0])   (expand on flipped taps)
//   mode 2: fwd F -> 1           U[t][c] = w[t, c, 0]
//   mode 3: bwd-data of 1 -> F   U[t][f] = conj(w[flip t, 0, f])
__global__ void k_pack_thin(float2* U, const float2* w, int KX, int KY, int F, int mode)
{
    MDNN_PDL_ENTRY();
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

// zero-padded halo of a one-channel image: tile[hy][hx] = img[x0 + hx - ox, y0 + hy - oy]
template<int HX, int HY>
__device__ __forceinline__ void load_halo(float2* tile, const float2* __restrict__ img, int X, int Y, long b, int x0,
                                          int y0, int ox, int oy)
{
    const long XY = long(X) * Y;
    for (int e = threadIdx.x; e < HX * HY; e += blockDim.x) {
        const int hx = e % HX, hy = e / HX;
        const int gx = x0 + hx - ox, gy = y0 + hy - oy;
        tile[e] = (gx >= 0 && gx < X && gy >= 0 && gy < Y) ? img[gx + long(X) * gy + XY * b] : float2{0.f, 0.f};
    }
}

// thin -> wide.  Block = TX x TY pixel tile of one item.  P output channels
// per thread (P = 2 when F is even: the window loads and the loop overhead are
// shared by two channels and the stores are 8-byte channel pairs -- the P = 1
// form was issue-bound with the FMA pipe half busy).
// Optional epilogue work on the produced wide tensor (P = 2, F = 64): per
// block forward BN statistics [blk][2F real channels][sum, sum of squares] in
// the layout of bnblock.cu's final kernels.  (The last BN block's backward
// reduction is emitted by the tensor-core expand of conv_thin_tc.cu.)
struct ThinEpi {
    double* stats = nullptr;
};

template<int K, int P>
__global__ void __launch_bounds__(NT) k_thin_expand(float* __restrict__ out, const float2* __restrict__ in,
                                                    const float2* __restrict__ U, int X, int Y, int F, int ox, int oy,
                                                    const ThinEpi ep)
{
    MDNN_PDL_ENTRY();
    constexpr int TY = 8, HX = TX + K - 1, HY = TY + K - 1;
    __shared__ float2 tile[HX * HY];
    const long b = blockIdx.z;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const long XY = long(X) * Y;
    load_halo<HX, HY>(tile, in, X, Y, b, x0, y0, ox, oy);
    const int FP = F / P;
    const int f = (threadIdx.x % FP) * P, lane = threadIdx.x / FP, lanes = NT / FP;
    float2 u[P][K * K];
#pragma unroll
    for (int q = 0; q < P; q++)
#pragma unroll
        for (int t = 0; t < K * K; t++)
            u[q][t] = U[t * F + f + q];
    __syncthreads();
    // epilogue accumulators: per channel q of the pair, Re lane and Im lane:
    // (sum, sum sq) of the values shifted by this thread's first value (esh),
    // re-centred in double at the fold -- the sum of squares carries the
    // spread, not the mean (no E|x|^2 - |mu|^2 cancellation)
    float es[P][2][2] = {};
    float esh[P][2] = {};
    int ecount = 0;
    const int nseg = max(1, lanes / TY), seglen = TX / nseg;
    for (int it = lane; it < TY * nseg; it += lanes) {
        const int row = it / nseg, xs = (it % nseg) * seglen;
        const int gy = y0 + row;
        if (gy >= Y)
            continue;
        float2 win[K][K];
#pragma unroll
        for (int ky = 0; ky < K; ky++)
#pragma unroll
            for (int kx = 0; kx < K - 1; kx++)
                win[ky][kx] = tile[(row + ky) * HX + xs + kx];
        float* op = out + (b * XY + long(X) * gy + x0 + xs) * 2 * F + f;
        // unrolled: the window shifts become register renames
#pragma unroll 8
        for (int i = 0; i < seglen; i++, op += 2 * F) {
            const int px = xs + i;
#pragma unroll
            for (int ky = 0; ky < K; ky++)
                win[ky][K - 1] = tile[(row + ky) * HX + px + K - 1];
            float2 acc[P];
#pragma unroll
            for (int q = 0; q < P; q++) {
                // two accumulator pairs (even / odd taps): 4 FFMA per complex MAC, short chains
                float2 a0{0.f, 0.f}, a1{0.f, 0.f};
#pragma unroll
                for (int ky = 0; ky < K; ky++)
#pragma unroll
                    for (int kx = 0; kx < K; kx++) {
                        const float2 w_ = win[ky][kx], uu = u[q][kx + K * ky];
                        float2& a_ = ((kx + K * ky) & 1) ? a1 : a0;
                        a_.x = fmaf(w_.x, uu.x, a_.x);
                        a_.y = fmaf(w_.x, uu.y, a_.y);
                        a_.x = fmaf(-w_.y, uu.y, a_.x);
                        a_.y = fmaf(w_.y, uu.x, a_.y);
                    }
                acc[q] = float2{a0.x + a1.x, a0.y + a1.y};
            }
            if (x0 + px < X) {
                if constexpr (P == 2) {
                    *reinterpret_cast<float2*>(op) = float2{acc[0].x, acc[1].x};
                    *reinterpret_cast<float2*>(op + F) = float2{acc[0].y, acc[1].y};
                    if (ep.stats) {
                        if (ecount++ == 0) {
#pragma unroll
                            for (int q = 0; q < P; q++)
                                esh[q][0] = acc[q].x, esh[q][1] = acc[q].y;
                        }
#pragma unroll
                        for (int q = 0; q < P; q++) {
                            const float dr = acc[q].x - esh[q][0], di = acc[q].y - esh[q][1];
                            es[q][0][0] += dr;
                            es[q][0][1] = fmaf(dr, dr, es[q][0][1]);
                            es[q][1][0] += di;
                            es[q][1][1] = fmaf(di, di, es[q][1][1]);
                        }
                    }
                } else {
                    op[0] = acc[0].x;
                    op[F] = acc[0].y;
                }
            }
#pragma unroll
            for (int ky = 0; ky < K; ky++)
#pragma unroll
                for (int kx = 0; kx < K - 1; kx++)
                    win[ky][kx] = win[ky][kx + 1];
        }
    }
    if constexpr (P == 2) {
        if (ep.stats) {
            // fixed-order fold over the `lanes` threads of each channel pair
            constexpr int NV = P * 2 * 2;
            __shared__ double red[NT * NV];
            __syncthreads();
#pragma unroll
            for (int q = 0; q < P; q++)
#pragma unroll
                for (int c2 = 0; c2 < 2; c2++) {
                    const double sh = esh[q][c2], n = ecount;
                    red[threadIdx.x * NV + (q * 2 + c2) * 2] = n * sh + es[q][c2][0];
                    red[threadIdx.x * NV + (q * 2 + c2) * 2 + 1] = sh * (n * sh + 2.0 * es[q][c2][0]) + es[q][c2][1];
                }
            __syncthreads();
            const long blk = blockIdx.x + long(gridDim.x) * (blockIdx.y + long(gridDim.y) * blockIdx.z);
            constexpr int nv = 2;
            double* dst = ep.stats;
            for (int e = threadIdx.x; e < FP * P * 2 * nv; e += NT) {
                const int v = e % nv, qc = (e / nv) % (P * 2), fp = e / (nv * P * 2);
                double acc = 0;
                for (int l = 0; l < lanes; l++)
                    acc += red[(l * FP + fp) * NV + qc * 2 + v];
                const int q = qc >> 1, c2 = qc & 1;
                const int n = c2 * F + fp * P + q; // real channel: Re part c, Im part F + c
                dst[(blk * 2 * F + n) * nv + v] = acc;
            }
        }
    }
}

// wide -> thin.  Output tile TX x TY; halo pixel h is owned by thread h % NT,
// which streams its own channel rows (8 channels = 2 x 16 B of Re and of Im
// per chunk) into private shared-memory slots with cp.async, double-buffered,
// so the channel loop needs no block barrier; U[t][c] is staged once and read
// as broadcasts.  The K^2 tap projections z_t[h] then meet in shared memory
// for the final K^2 gather.
constexpr int RCC = 8; // channels per chunk
template<int K>
struct ReduceCfg {
    static constexpr int TY = K == 3 ? 16 : 8;
    static constexpr int HX = TX + K - 1, HY = TY + K - 1, NH = HX * HY, KK = K * K;
    static constexpr int PP = (NH + NT - 1) / NT; // halo pixels per thread
    // staging: [buf][PP][quad 0..3][NT] float4   (quad: Re lo, Re hi, Im lo, Im hi)
    static constexpr int STAGE_F4 = 2 * PP * 4 * NT;
    static constexpr int Z_F2 = NH * KK;
    static constexpr size_t stage_bytes() { return sizeof(float4) * STAGE_F4; }
    static constexpr size_t z_bytes() { return sizeof(float2) * Z_F2; }
    static constexpr size_t smem(int F)
    {
        return (stage_bytes() > z_bytes() ? stage_bytes() : z_bytes()) + sizeof(float2) * KK * F;
    }
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid)
{
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template<int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template<int K>
__global__ void __launch_bounds__(NT, K == 3 ? 2 : 1) k_thin_reduce(float2* __restrict__ out, const float* __restrict__ in,
                                                       const float2* __restrict__ U, int X, int Y, int F, int ox,
                                                       int oy)
{
    MDNN_PDL_ENTRY();
    using Cfg = ReduceCfg<K>;
    constexpr int HX = Cfg::HX, NH = Cfg::NH, KK = Cfg::KK, PP = Cfg::PP, TY = Cfg::TY;
    extern __shared__ float4 smr4[];
    float4* stage = smr4;                                  // [2][PP][4][NT]
    float2* z = reinterpret_cast<float2*>(smr4);           // [NH][KK] after the channel loop
    constexpr size_t ZOFF = (Cfg::stage_bytes() > Cfg::z_bytes() ? Cfg::stage_bytes() : Cfg::z_bytes());
    float2* su = reinterpret_cast<float2*>(reinterpret_cast<char*>(smr4) + ZOFF); // [KK][F]
    const int tid = threadIdx.x;
    const long b = blockIdx.z;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const long XY = long(X) * Y;
    for (int e = tid; e < KK * F; e += NT)
        su[e] = U[e];

    // per owned halo pixel: source row (or null when outside the image)
    const float* src[PP];
#pragma unroll
    for (int k = 0; k < PP; k++) {
        const int h = tid + k * NT;
        const int hx = h % HX, hy = h / HX;
        const int gx = x0 + hx - ox, gy = y0 + hy - oy;
        src[k] = (h < NH && gx >= 0 && gx < X && gy >= 0 && gy < Y) ? in + (b * XY + gx + long(X) * gy) * 2 * F
                                                                     : nullptr;
    }
    auto issue = [&](int chunk, int buf) {
        const int c0 = chunk * RCC;
#pragma unroll
        for (int k = 0; k < PP; k++)
#pragma unroll
            for (int qd = 0; qd < 4; qd++) {
                const bool ok = src[k] != nullptr;
                const float* g = ok ? src[k] + (qd >> 1) * F + c0 + (qd & 1) * 4 : in;
                cp_async16(&stage[((buf * PP + k) * 4 + qd) * NT + tid], g, ok);
            }
        cp_commit();
    };
    const int nchunk = F / RCC;
    issue(0, 0);
    __syncthreads(); // su visible

    float2 acc[PP][KK];
#pragma unroll
    for (int k = 0; k < PP; k++)
#pragma unroll
        for (int t = 0; t < KK; t++)
            acc[k][t] = float2{0.f, 0.f};
    for (int ch = 0; ch < nchunk; ch++) {
        const int buf = ch & 1;
        if (ch + 1 < nchunk) {
            issue(ch + 1, buf ^ 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        float re[PP][RCC], im[PP][RCC];
#pragma unroll
        for (int k = 0; k < PP; k++) {
            const float4 a0 = stage[((buf * PP + k) * 4 + 0) * NT + tid];
            const float4 a1 = stage[((buf * PP + k) * 4 + 1) * NT + tid];
            const float4 b0 = stage[((buf * PP + k) * 4 + 2) * NT + tid];
            const float4 b1 = stage[((buf * PP + k) * 4 + 3) * NT + tid];
            re[k][0] = a0.x, re[k][1] = a0.y, re[k][2] = a0.z, re[k][3] = a0.w;
            re[k][4] = a1.x, re[k][5] = a1.y, re[k][6] = a1.z, re[k][7] = a1.w;
            im[k][0] = b0.x, im[k][1] = b0.y, im[k][2] = b0.z, im[k][3] = b0.w;
            im[k][4] = b1.x, im[k][5] = b1.y, im[k][6] = b1.z, im[k][7] = b1.w;
        }
        const float2* uc = su + ch * RCC;
#pragma unroll
        for (int cc = 0; cc < RCC; cc++)
#pragma unroll
            for (int t = 0; t < KK; t++) {
                const float2 uu = uc[t * F + cc];
#pragma unroll
                for (int k = 0; k < PP; k++) {
                    acc[k][t].x = fmaf(re[k][cc], uu.x, acc[k][t].x);
                    acc[k][t].y = fmaf(re[k][cc], uu.y, acc[k][t].y);
                    acc[k][t].x = fmaf(-im[k][cc], uu.y, acc[k][t].x);
                    acc[k][t].y = fmaf(im[k][cc], uu.x, acc[k][t].y);
                }
            }
    }
    __syncthreads(); // all staging reads done before z overwrites it
#pragma unroll
    for (int k = 0; k < PP; k++) {
        const int h = tid + k * NT;
        if (h < NH)
#pragma unroll
            for (int t = 0; t < KK; t++)
                z[h * KK + t] = acc[k][t];
    }
    __syncthreads();
    for (int q = tid; q < TX * TY; q += NT) {
        const int px = q % TX, py = q / TX;
        const int gx = x0 + px, gy = y0 + py;
        float2 s{0.f, 0.f};
#pragma unroll
        for (int ky = 0; ky < K; ky++)
#pragma unroll
            for (int kx = 0; kx < K; kx++) {
                const float2 v = z[((py + ky) * HX + px + kx) * KK + kx + K * ky];
                s.x += v.x;
                s.y += v.y;
            }
        if (gx < X && gy < Y)
            out[b * XY + gx + long(X) * gy] = s;
    }
}

// Weight gradient with one thin operand; persistent CTAs over TX x 8 tiles.
//   WIDE_IS_G (1 -> F layer, g = dy wide, h = x thin):
//       acc[t] += g[p, f] conj(h[p + t - c0]),  window over h with offset c0
//   else (F -> 1 layer, g = dy thin, h = x wide), substituting p' = p + t - c0:
//       acc[t] += g[p' - t + c0] conj(h[p', c]), window over g with offset K-1-c0
//       and flipped tap index.
// P channels per thread (P = 2: 8-byte channel-pair loads, the window loads and
// the loop overhead shared by two channels -- as in k_thin_expand)
template<int K, bool WIDE_IS_G, int P>
__global__ void __launch_bounds__(NT, THIN_WG_MINB(K)) k_thin_wgrad(float2* __restrict__ part, const float* __restrict__ wide,
                                                   const float2* __restrict__ thin, int X, int Y, int B, int F,
                                                   int ox, int oy)
{
    MDNN_PDL_ENTRY();
    constexpr int TY = 8, HX = TX + K - 1, HY = TY + K - 1, KK = K * K;
    __shared__ float2 tile[HX * HY];
    extern __shared__ float2 sred[]; // [lanes][KK][F] = NT * KK float2
    const long XY = long(X) * Y;
    const int ntx = (X + TX - 1) / TX, nty = (Y + TY - 1) / TY;
    const long ntiles = long(ntx) * nty * B;
    const int FP = F / P;
    const int f = (threadIdx.x % FP) * P, lane = threadIdx.x / FP, lanes = NT / FP;
    const int nseg = max(1, lanes / TY), seglen = TX / nseg;
    float2 acc[P][KK];
#pragma unroll
    for (int q = 0; q < P; q++)
#pragma unroll
        for (int t = 0; t < KK; t++)
            acc[q][t] = float2{0.f, 0.f};
    for (long tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
        const int x0 = int(tl % ntx) * TX, y0 = int((tl / ntx) % nty) * TY;
        const long b = tl / (long(ntx) * nty);
        __syncthreads();
        load_halo<HX, HY>(tile, thin, X, Y, b, x0, y0, ox, oy);
        __syncthreads();
        for (int it = lane; it < TY * nseg; it += lanes) {
            const int row = it / nseg, xs = (it % nseg) * seglen;
            const int gy = y0 + row;
            if (gy >= Y)
                continue;
            float2 win[K][K];
#pragma unroll
            for (int ky = 0; ky < K; ky++)
#pragma unroll
                for (int kx = 0; kx < K - 1; kx++)
                    win[ky][kx] = tile[(row + ky) * HX + xs + kx];
            const int xend = min(seglen, X - x0 - xs);
            // wide operand walked with a pointer (2F floats per pixel), PD pixels
            // of loads in flight ahead of the taps
            constexpr int PD = 4;
            const float* wp = wide + (b * XY + long(X) * gy + x0 + xs) * 2 * F + f;
            // pre[d][q] = (Re, Im) of channel f + q at pixel i + d
            float2 pre[PD][P];
            auto ldpix = [&](const float* ptr, float2 (&o)[P]) {
                if constexpr (P == 2) {
                    const float2 re = __ldg(reinterpret_cast<const float2*>(ptr));
                    const float2 im = __ldg(reinterpret_cast<const float2*>(ptr + F));
                    o[0] = float2{re.x, im.x};
                    o[1] = float2{re.y, im.y};
                } else {
                    o[0] = float2{__ldg(ptr), __ldg(ptr + F)};
                }
            };
#pragma unroll
            for (int d = 0; d < PD; d++) {
                if (d < xend)
                    ldpix(wp + d * 2 * F, pre[d]);
                else
#pragma unroll
                    for (int q = 0; q < P; q++)
                        pre[d][q] = float2{0.f, 0.f};
            }
            wp += PD * 2 * F;
#pragma unroll 8
            for (int i = 0; i < xend; i++) {
                const int px = xs + i;
                float2 vv[P];
#pragma unroll
                for (int q = 0; q < P; q++)
                    vv[q] = pre[0][q];
#pragma unroll
                for (int d = 0; d < PD - 1; d++)
#pragma unroll
                    for (int q = 0; q < P; q++)
                        pre[d][q] = pre[d + 1][q];
                if (i + PD < xend)
                    ldpix(wp, pre[PD - 1]);
                else
#pragma unroll
                    for (int q = 0; q < P; q++)
                        pre[PD - 1][q] = float2{0.f, 0.f};
                wp += 2 * F;
#pragma unroll
                for (int ky = 0; ky < K; ky++)
                    win[ky][K - 1] = tile[(row + ky) * HX + px + K - 1];
#pragma unroll
                for (int q = 0; q < P; q++) {
                    const float2 v = vv[q];
#pragma unroll
                    for (int ky = 0; ky < K; ky++)
#pragma unroll
                        for (int kx = 0; kx < K; kx++) {
                            const float2 s = win[ky][kx];
                            if (WIDE_IS_G) {
                                // v * conj(s)
                                float2& a_ = acc[q][kx + K * ky];
                                a_.x = fmaf(v.x, s.x, a_.x);
                                a_.y = fmaf(v.y, s.x, a_.y);
                                a_.x = fmaf(v.y, s.y, a_.x);
                                a_.y = fmaf(-v.x, s.y, a_.y);
                            } else {
                                // s * conj(v)
                                float2& a_ = acc[q][(K - 1 - kx) + K * (K - 1 - ky)];
                                a_.x = fmaf(s.x, v.x, a_.x);
                                a_.y = fmaf(s.y, v.x, a_.y);
                                a_.x = fmaf(s.y, v.y, a_.x);
                                a_.y = fmaf(-s.x, v.y, a_.y);
                            }
                        }
                }
#pragma unroll
                for (int ky = 0; ky < K; ky++)
#pragma unroll
                    for (int kx = 0; kx < K - 1; kx++)
                        win[ky][kx] = win[ky][kx + 1];
            }
        }
    }
    // fold the lanes of each channel in a fixed order
#pragma unroll
    for (int q = 0; q < P; q++)
#pragma unroll
        for (int t = 0; t < KK; t++)
            sred[(lane * KK + t) * F + f + q] = acc[q][t];
    __syncthreads();
    for (int e = threadIdx.x; e < KK * F; e += NT) {
        float2 s{0.f, 0.f};
        for (int l = 0; l < lanes; l++) {
            s.x += sred[l * KK * F + e].x;
            s.y += sred[l * KK * F + e].y;
        }
        part[long(blockIdx.x) * KK * F + e] = s;
    }
}

// dw[t + KK f] = sum over CTAs of part[blk][t * F + f]; one block per output,
// fixed-order tree in double
__global__ void __launch_bounds__(NT) k_thin_wsum(float2* __restrict__ dw, const float2* __restrict__ part, int nblk,
                                                  int KK, int F)
{
    MDNN_PDL_ENTRY();
    __shared__ double sr[NT], si[NT];
    const int e = blockIdx.x;
    double a = 0, c = 0;
    for (int k = threadIdx.x; k < nblk; k += NT) {
        const float2 v = part[long(k) * KK * F + e];
        a += v.x;
        c += v.y;
    }
    sr[threadIdx.x] = a;
    si[threadIdx.x] = c;
    __syncthreads();
    for (int s = NT / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            sr[threadIdx.x] += sr[threadIdx.x + s];
            si[threadIdx.x] += si[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int t = e / F, f = e % F;
        dw[t + long(KK) * f] = float2{float(sr[0]), float(si[0])};
    }
}

float2* pack_u(const cfloat* w, const ConvGeom& g, int F, int pmode)
{
    auto& c = ctx();
    const int KK = int(g.KX * g.KY);
    float2* U;
    CUDA_CHECK(cudaMallocAsync(&U, sizeof(float2) * KK * F, c.stream));
    pdl_launch(k_pack_thin, std::max(1, (KK * F + 255) / 256), 256, 0, c.stream, U, w, int(g.KX), int(g.KY), F, pmode);
    KERNEL_CHECK();
    return U;
}

template<int K>
void run_thin(cfloat* outp, const cfloat* inp, const float2* U, const ConvGeom& g, int F, bool expand, int ox, int oy,
              const ThinEpi& ep = ThinEpi{})
{
    auto& c = ctx();
    if (expand) {
        dim3 grid(unsigned((g.X + TX - 1) / TX), unsigned((g.Y + 7) / 8), unsigned(g.B));
        if (F % 2 == 0 && NT % (F / 2) == 0)
            pdl_launch(k_thin_expand<K, 2>, grid, NT, 0, c.stream, reinterpret_cast<float*>(outp), inp, U, int(g.X),
                                                           int(g.Y), F, ox, oy, ep);
        else
            pdl_launch(k_thin_expand<K, 1>, grid, NT, 0, c.stream, reinterpret_cast<float*>(outp), inp, U, int(g.X),
                                                           int(g.Y), F, ox, oy, ThinEpi{});
    } else {
        if (thin_reduce_tc(outp, reinterpret_cast<const float*>(inp), U, g.X, g.Y, g.B, F, K * K, ox, oy))
            return; // tensor-core projections + gather (conv_thin_tc.cu)
        using Cfg = ReduceCfg<K>;
        auto kern = k_thin_reduce<K>;
        allow_max_dyn_smem(reinterpret_cast<const void*>(kern));
        dim3 grid(unsigned((g.X + TX - 1) / TX), unsigned((g.Y + Cfg::TY - 1) / Cfg::TY), unsigned(g.B));
        pdl_launch(kern, grid, NT, Cfg::smem(F), c.stream, outp, reinterpret_cast<const float*>(inp), U, int(g.X), int(g.Y),
                                                  F, ox, oy);
    }
    KERNEL_CHECK();
}

template<int K>
void run_thin_wgrad(float2* part, int nblk, const cfloat* x, const cfloat* dy, const ConvGeom& g, int F, bool one_in)
{
    auto& c = ctx();
    // sred holds lanes x KK x F: lanes = NT / (F / P)
    const bool pair = F % 2 == 0 && NT % (F / 2) == 0;
    const size_t smem = sizeof(float2) * (pair ? 2 : 1) * NT * K * K;
    if (one_in) { // g = dy wide, h = x thin, window offset c0
        auto kern = pair ? k_thin_wgrad<K, true, 2> : k_thin_wgrad<K, true, 1>;
        allow_max_dyn_smem(reinterpret_cast<const void*>(kern));
        pdl_launch(kern, nblk, NT, smem, c.stream, part, reinterpret_cast<const float*>(dy), x, int(g.X), int(g.Y), int(g.B),
                                           F, int(g.px), int(g.py));
    } else { // g = dy thin, h = x wide, window offset K-1-c0
        auto kern = pair ? k_thin_wgrad<K, false, 2> : k_thin_wgrad<K, false, 1>;
        allow_max_dyn_smem(reinterpret_cast<const void*>(kern));
        pdl_launch(kern, nblk, NT, smem, c.stream, part, reinterpret_cast<const float*>(x), dy, int(g.X), int(g.Y), int(g.B),
                                           F, int(K - 1 - g.px), int(K - 1 - g.py));
    }
    KERNEL_CHECK();
}

} // namespace

bool conv_thin_supported(const ConvGeom& g)
{
    const bool one_in = g.Cin == 1, one_out = g.Cout == 1;
    const long F = one_in ? g.Cout : g.Cin;
    if (one_in == one_out || F > MAXF || 256 % F != 0 || F % RCC != 0 || g.KX != g.KY || (g.KX != 3 && g.KX != 5))
        return false;
    // the wide side must be channels-last (the thin side is layout-free)
    return one_in ? g.out_chlast : g.in_chlast;
}

// partial blocks of the expand kernel's epilogue statistics (0: none for this geometry / mode)
long conv_thin_epi_blocks(const ConvGeom& g, int mode)
{
    if (!conv_thin_supported(g))
        return 0;
    const bool one_in = g.Cin == 1;
    const bool expand = (mode == 0) == one_in;
    const long F = one_in ? g.Cout : g.Cin;
    // forward statistics from either expand; BN-backward partials only from the
    // tensor-core expand (in the issue-bound CUDA-core loop they cost more than
    // the separate reduction pass they replace: +2.4 ms vs -1.6 ms per two steps)
    if (!expand || F != 64)
        return 0;
    if (mode == 1)
        return conv_thin_tc_bnb() && g.KX == 3 ? thin_expand_tc_blocks() : 0;
    // allocation bound: the CUDA-core kernel's blocks or the tensor-core kernel's slots
    return std::max(((g.X + TX - 1) / TX) * ((g.Y + 7) / 8) * g.B, thin_expand_tc_blocks());
}

// mode: 0 fwd, 1 bwd-data
void conv_thin_run(cfloat* outp, const cfloat* inp, const cfloat* w, const ConvGeom& g, int mode)
{
    auto& c = ctx();
    const bool one_in = g.Cin == 1;
    const int F = int(one_in ? g.Cout : g.Cin);
    // expand (thin -> wide): fwd of 1->F, bwd-data of F->1; reduce otherwise
    const bool expand = (mode == 0) == one_in;
    const int pmode = mode == 0 ? (one_in ? 0 : 2) : (one_in ? 3 : 1);
    float2* U = pack_u(w, g, F, pmode);
    // window offset: forward reads p + t - c0; adjoints use flipped taps with offset K-1-c0
    const int ox = mode == 0 ? int(g.px) : int(g.KX - 1 - g.px);
    const int oy = mode == 0 ? int(g.py) : int(g.KY - 1 - g.py);
    // epilogue work for a batch-norm neighbour (expand with 64 wide channels only)
    ThinEpi ep{};
    const long eblocks = conv_thin_epi_blocks(g, mode);
    if (g.stats_blocks)
        *g.stats_blocks = 0;
    if (g.bnb_blocks)
        *g.bnb_blocks = 0;
    if (eblocks > 0 && mode == 0 && g.stats && g.stats_blocks) {
        ep.stats = g.stats;
        // blocks the CUDA-core expand writes (its grid); the tensor-core path resets this below
        *g.stats_blocks = int(((g.X + TX - 1) / TX) * ((g.Y + 7) / 8) * g.B);
    }
    // mode 1 with a BN hint: only the tensor-core expand folds the BN-backward
    // reduction (the CUDA-core loop measured slower with it)
    const bool bn_tc = eblocks > 0 && mode == 1 && g.bnb && g.bnb_part && g.bnb_blocks;
    {
        // HBM-bound: algorithmic bytes = wide side once + thin side once
        ProfScope prof(mode == 0 ? "conv_thin_fwd" : "conv_thin_bwd_data", 8.0 * double(g.X) * g.Y * g.B * (F + 1));
        int tc_blocks = 0;
        if (expand && g.KX == 3
            && thin_expand_tc(reinterpret_cast<float*>(outp), inp, U, g.X, g.Y, g.B, F, 9, ox, oy, ep.stats,
                              &tc_blocks, bn_tc ? g.bnb : nullptr, bn_tc ? g.bnb_part : nullptr,
                              bn_tc ? g.bnb_blocks : nullptr)) {
            // tensor-core im2col GEMM (conv_thin_tc.cu); its statistics partials replace the CUDA-core ones
            if (ep.stats && g.stats_blocks)
                *g.stats_blocks = tc_blocks;
            CUDA_CHECK(cudaFreeAsync(U, c.stream));
            return;
        }
        if (g.KX == 3)
            run_thin<3>(outp, inp, U, g, F, expand, ox, oy, ep);
        else
            run_thin<5>(outp, inp, U, g, F, expand, ox, oy, ep);
    }
    CUDA_CHECK(cudaFreeAsync(U, c.stream));
}

// dw[t, c, f] = sum_p dy[p, f] conj(x[p + t - c0, c]) with one thin side
void conv_thin_wgrad(cfloat* dw, const cfloat* x, const cfloat* dy, const ConvGeom& g)
{
    auto& c = ctx();
    const bool one_in = g.Cin == 1;
    const int F = int(one_in ? g.Cout : g.Cin);
    const int KK = int(g.KX * g.KY);
    const long ntiles = ((g.X + TX - 1) / TX) * ((g.Y + 7) / 8) * g.B;
    const int nblk = int(std::min<long>(ntiles, 3L * c.sm_count));
    float2* part;
    CUDA_CHECK(cudaMallocAsync(&part, sizeof(float2) * nblk * KK * F, c.stream));
    {
        ProfScope prof("conv_thin_bwd_weight", 8.0 * double(g.X) * g.Y * g.B * (F + 1));
        if (g.KX == 3)
            run_thin_wgrad<3>(part, nblk, x, dy, g, F, one_in);
        else
            run_thin_wgrad<5>(part, nblk, x, dy, g, F, one_in);
        pdl_launch(k_thin_wsum, KK * F, NT, 0, c.stream, dw, part, nblk, KK, F);
        KERNEL_CHECK();
    }
    CUDA_CHECK(cudaFreeAsync(part, c.stream));
}

} // namespace mdnn
