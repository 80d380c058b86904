// Wide -> thin 3x3 convolution (MoDL's last layer F -> 1 and the bwd-data of
// its first layer) on the tensor cores, in two passes:
//   1. k_thin_proj: the per-pixel tap projections z_t[p] = sum_c wide[p, c] U[t, c]
//      (9 complex taps) as one TF32 GEMM  Z[p][n] = wide[p][k] * Ut[n][k],
//      M = 128 pixels, N = 32 (18 used: 9 taps x re/im), K = 2F = 128 real
//      channels; the channels-last rows arrive by TMA, the packed Ut once per
//      CTA; the accumulator is double-buffered in TMEM so the Z stores of one
//      tile overlap the MMAs of the next.  Every pixel's projections are
//      computed once (the CUDA-core kernel recomputed the tile halos, 1.2x).
//   2. k_thin_gather: out[q] = sum_t z_t[q + t - o] (zero outside the image),
//      reading Z (80 B per pixel, mostly from L2).
// Same maths as k_thin_reduce (conv_thin.cu); the wide operand is read at
// TF32 by the tensor core, the packed weights are rounded RN.
#include <cudaTypedefs.h>

#include "kernels.h"
#include "profile.h"
#include "sm100.cuh"

#include <algorithm>
#include <map>
#include <mutex>

namespace mdnn {

namespace {

using namespace sm100;

constexpr int TP_ROWS = 128;  // pixels per tile (UMMA M)
constexpr int TP_N = 32;      // projection columns (18 used)
constexpr int TP_ZP = 20;     // floats per pixel in Z (18 + 2 pad: 5 float4)
constexpr int TP_K = 128;     // real channels (2F, F = 64)
constexpr int TP_CH = TP_K / 32;
constexpr int TP_ABYTES = TP_CH * TP_ROWS * 128; // one A stage: 64 KB
constexpr int TP_BBYTES = TP_CH * TP_N * 128;    // packed Ut: 16 KB
constexpr int TP_THREADS = 192;

struct TpSmem {
    static constexpr int A_OFF = 0;
    static constexpr int B_OFF = 2 * TP_ABYTES;
    static constexpr int BAR_OFF = B_OFF + TP_BBYTES;
    static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

// Ut[n][k]: row n = 2 t + comp (comp 0: Re z_t, 1: Im z_t); k < F: Re wide_c, k >= F: Im wide_c
__global__ void k_pack_thin_tc(float* __restrict__ ut, const float2* __restrict__ U, int F, int KK)
{
    MDNN_PDL_ENTRY();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < TP_N * 2 * F; i += gridDim.x * blockDim.x) {
        const int k = i % (2 * F), n = i / (2 * F);
        const int t = n >> 1, comp = n & 1;
        float v = 0.f;
        if (t < KK) {
            const bool im_in = k >= F;
            const float2 u = U[t * F + (im_in ? k - F : k)];
            // z = sum (wr + i wi)(ur + i ui): Re = wr ur - wi ui, Im = wr ui + wi ur
            v = comp == 0 ? (im_in ? -u.y : u.x) : (im_in ? u.x : u.y);
        }
        ut[size_t(n) * 2 * F + k] = to_tf32(v);
    }
}

__global__ void __launch_bounds__(TP_THREADS, 1)
    k_thin_proj(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                float* __restrict__ z, long npix)
{
    MDNN_PDL_ENTRY();
    extern __shared__ uint8_t smem_raw[];
    // aligned by an offset from the shared array (not an integer round trip), so
    // the compiler keeps the shared address space: LDS/STS, not generic LD/ST
    uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* abuf = smem + TpSmem::A_OFF;
    uint8_t* bbuf = smem + TpSmem::B_OFF;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TpSmem::BAR_OFF);
    uint64_t* a_full = bars;         // [2]
    uint64_t* a_empty = bars + 2;    // [2]
    uint64_t* b_full = bars + 4;
    uint64_t* tmem_full = bars + 5;  // [2]
    uint64_t* tmem_empty = bars + 7; // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const long ntiles = (npix + TP_ROWS - 1) / TP_ROWS;
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tm_a);
        prefetch_tmap(&tm_b);
        for (int i = 0; i < 2; i++) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 128);
        }
        mbar_init(b_full, 1);
        fence_barrier_init();
    }
    if (warp == 1)
        tmem_alloc<2 * TP_N>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            mbar_arrive_expect_tx(b_full, TP_BBYTES);
            for (int c = 0; c < TP_CH; c++)
                tma_load_2d(bbuf + c * TP_N * 128, &tm_b, b_full, c * 32, 0);
            uint32_t it = 0;
            for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
                const uint32_t st = it & 1, ph = (it >> 1) & 1;
                mbar_wait(&a_empty[st], ph ^ 1);
                mbar_arrive_expect_tx(&a_full[st], TP_ABYTES);
                for (int c = 0; c < TP_CH; c++)
                    tma_load_2d(abuf + st * TP_ABYTES + c * TP_ROWS * 128, &tm_a, &a_full[st], c * 32,
                                int(tile * TP_ROWS));
            }
        }
    } else if (warp == 1) {
        // whole warp; the elected lane issues (mma_tf32_warp)
        constexpr uint32_t idesc = idesc_tf32(TP_ROWS, TP_N);
        const uint64_t ad0 = umma_desc_sw128(smem_u32(abuf), 1024);
        const uint64_t bd0 = umma_desc_sw128(smem_u32(bbuf), 1024);
        mbar_wait(b_full, 0);
        tc_fence_after();
        uint32_t it = 0;
        for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
            const uint32_t st = it & 1, ph = (it >> 1) & 1;
            const uint32_t acc = tmem_base + st * TP_N;
            mbar_wait(&tmem_empty[st], ph ^ 1);
            mbar_wait(&a_full[st], ph);
            tc_fence_after();
            const uint64_t ad = ad0 + ((st * TP_ABYTES) >> 4);
#pragma unroll
            for (int c = 0; c < TP_CH; c++)
#pragma unroll
                for (int k = 0; k < 4; k++)
                    mma_tf32_warp(acc, ad + ((c * TP_ROWS * 128 + k * 32) >> 4), bd0 + ((c * TP_N * 128 + k * 32) >> 4),
                                  idesc, (c | k) != 0);
            mma_commit_warp(&a_empty[st]);
            mma_commit_warp(&tmem_full[st]);
        }
    } else {
        // epilogue: TMEM lane = pixel, 32 columns -> Z row (18 values + pad)
        const int lg = warp & 3;
        uint32_t it = 0;
        for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
            const uint32_t st = it & 1, ph = (it >> 1) & 1;
            mbar_wait(&tmem_full[st], ph);
            tc_fence_after();
            float v[32];
            tmem_ld32(tmem_base + st * TP_N + (uint32_t(lg * 32) << 16), v);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&tmem_empty[st]);
            const long p = tile * TP_ROWS + lg * 32 + lane;
            if (p < npix) {
                float4* zp = reinterpret_cast<float4*>(z + p * TP_ZP);
#pragma unroll
                for (int q = 0; q < TP_ZP / 4; q++)
                    zp[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<2 * TP_N>(tmem_base);
    }
}

// out[q] = sum_t z_t[q + t - o], t = (tx, ty) row-major over the 3 x 3 kernel
__global__ void __launch_bounds__(256) k_thin_gather(float2* __restrict__ out, const float* __restrict__ z, int X, int Y,
                                                     long npix, int ox, int oy)
{
    MDNN_PDL_ENTRY();
    for (long q = blockIdx.x * long(blockDim.x) + threadIdx.x; q < npix; q += long(gridDim.x) * blockDim.x) {
        const int x = int(q % X), y = int((q / X) % Y);
        const long b = q / (long(X) * Y);
        float2 acc{0.f, 0.f};
#pragma unroll
        for (int ty = 0; ty < 3; ty++) {
            const int hy = y + ty - oy;
            if (hy < 0 || hy >= Y)
                continue;
#pragma unroll
            for (int tx = 0; tx < 3; tx++) {
                const int hx = x + tx - ox;
                if (hx < 0 || hx >= X)
                    continue;
                const int t = tx + 3 * ty;
                const float2 v = *reinterpret_cast<const float2*>(z + ((b * Y + hy) * X + hx) * TP_ZP + 2 * t);
                acc.x += v.x;
                acc.y += v.y;
            }
        }
        out[q] = acc;
    }
}

// ---------------------------------------------------------------------------
// Thin -> wide (1 -> F = 64, 3x3; fwd of the first layer, bwd-data of the last)
// in channel-major form: D^T[n = output (re|im) channel, 128][p = pixel, 256]
// = Ue[n][k] x im2col[p][k], k = 2 t + (re|im) of thin[p + t - o] (18 used of
// 32).  Four builder warps write the im2col rows (128 B, SWIZZLE_128B) for a
// 256-pixel tile straight from the (L2-resident) thin image, the MMA warp
// issues 4 UMMAs of 128 x 256 x 8 per tile, and 16 epilogue warps store
// 128-B channel rows per pixel and accumulate the forward BN statistics
// (same partial layout as the channel-major conv).  B tiles and TMEM
// accumulators are double-buffered.
constexpr int TE_P = 256;                 // pixels per tile (UMMA N)
// split precision (3xTF32): K = 64 = [x_hi(18) | x_lo(18) | x_hi(18) | 0] against
// [w_hi | w_hi | w_lo | 0], i.e. w_hi x_hi + w_hi x_lo + w_lo x_hi in one GEMM --
// the first layer's output keeps fp32 accuracy (plain TF32 moved the MoDL
// loss by 1e-3); two 128-B K chunks per row, each its own swizzled tile
constexpr int TE_KCH = 2;
constexpr int TE_BCH = TE_P * 128;          // one K chunk of the im2col tile: 32 KB
constexpr int TE_BBYTES = TE_KCH * TE_BCH;  // 64 KB per buffer
constexpr int TE_ACH = 128 * 128;           // one K chunk of the packed weights: 16 KB
constexpr int TE_ABYTES = TE_KCH * TE_ACH;
constexpr int TE_BUILD = 4, TE_EPI = 16;  // warps
constexpr int TE_THREADS = 32 * (1 + TE_BUILD + TE_EPI);

constexpr int TE_STG = 16 * 32 * 4; // per epilogue warp and buffer: 16 pixels x 32 channels (2 KB)

struct TeSmem {
    static constexpr int B_OFF = 0;
    static constexpr int A_OFF = 2 * TE_BBYTES;
    static constexpr int STG_OFF = A_OFF + TE_ABYTES;        // [TE_EPI][2][16][32] floats
    static constexpr int BAR_OFF = STG_OFF + TE_EPI * 2 * TE_STG;
    // > half the SM's shared memory: one CTA per SM (it allocates all 512 TMEM columns)
    static constexpr int TOTAL = (BAR_OFF + 256 + 1024) > 120 * 1024 ? (BAR_OFF + 256 + 1024) : 120 * 1024;
};

// Ue[c][n][32] (K chunk c of row n): n < 64: Re out_f = sum_t tr ur - ti ui ; n >= 64: Im = tr ui + ti ur;
// K layout [w_hi(18) | w_hi(18) | w_lo(18) | 0]
__global__ void k_pack_thin_expand(float* __restrict__ ue, const float2* __restrict__ U, int F, int KK)
{
    MDNN_PDL_ENTRY();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 128 * 64; i += gridDim.x * blockDim.x) {
        const int kk = i % 64, n = i / 64;
        const int part = kk / 18, k = kk % 18;
        const int t = k >> 1, comp = k & 1, f = n % F;
        float v = 0.f;
        if (part < 3 && t < KK) {
            const float2 u = U[t * F + f];
            const float w = n < F ? (comp ? -u.y : u.x) : (comp ? u.x : u.y);
            const float hi = to_tf32(w);
            v = part < 2 ? hi : to_tf32(w - hi);
        }
        ue[(size_t(kk >> 5) * 128 + n) * 32 + (kk & 31)] = v;
    }
}

// byte offset of (row r, 16-B granule g) in a SWIZZLE_128B K-major tile (8-row atoms of 1024 B)
__device__ __forceinline__ int sw128_off(int r, int g) { return (r >> 3) * 1024 + (r & 7) * 128 + ((g ^ (r & 7)) << 4); }

// BN-backward reduction in the epilogue (bwd-data of the last layer: the produced
// cotangent is the last BN block's output cotangent) -- as in k_conv_tc_t
struct TeBn {
    const float* x = nullptr; // BN input, CHLAST 128 floats per pixel
    const float2* mu = nullptr;
    const float* istd = nullptr;
    const float2* gamma = nullptr;
    const float2* beta = nullptr;
    double* part = nullptr;   // [blk][128][3]
};

// EPI: 0 = store only, 1 = + forward BN statistics, 2 = + BN-backward partials
// (compile-time, as in conv_tc.cu: each form carries only its own registers)
template<int EPI>
__global__ void __launch_bounds__(TE_THREADS, 1)
    k_thin_expand_tc(const __grid_constant__ CUtensorMap tm_out, const float2* __restrict__ thin,
                     const float* __restrict__ ue, int X, int Y, long npix, int ox, int oy, double* __restrict__ stats,
                     const TeBn be)
{
    MDNN_PDL_ENTRY();
    extern __shared__ uint8_t smem_raw[];
    // aligned by an offset from the shared array (not an integer round trip), so
    // the compiler keeps the shared address space: LDS/STS, not generic LD/ST
    uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* bbuf = smem + TeSmem::B_OFF;
    uint8_t* abuf = smem + TeSmem::A_OFF;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TeSmem::BAR_OFF);
    uint64_t* b_full = bars;         // [2] builders -> MMA (128 arrivals)
    uint64_t* b_empty = bars + 2;    // [2] MMA commit -> builders
    uint64_t* tmem_full = bars + 4;  // [2]
    uint64_t* tmem_empty = bars + 6; // [2] (32 * TE_EPI arrivals)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const long ntiles = (npix + TE_P - 1) / TE_P;

    // packed weights (2 K chunks, 32 KB) into the swizzled A tiles; zero the im2col
    // granules no builder writes (chunk 1, granules 6-7: k = 56..63) once
    for (int e = threadIdx.x; e < TE_KCH * 128 * 8; e += TE_THREADS) {
        const int c = e / (128 * 8), r = (e >> 3) % 128, g = e & 7;
        *reinterpret_cast<float4*>(abuf + c * TE_ACH + sw128_off(r, g)) = reinterpret_cast<const float4*>(ue)[e];
    }
    for (int e = threadIdx.x; e < 2 * TE_P * 2; e += TE_THREADS) {
        const int bb = e / (TE_P * 2), r = (e >> 1) % TE_P, g = 6 + (e & 1);
        *reinterpret_cast<float4*>(bbuf + bb * TE_BBYTES + TE_BCH + sw128_off(r, g)) =
            make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; i++) {
            mbar_init(&b_full[i], 32 * TE_BUILD);
            mbar_init(&b_empty[i], 1);
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 32 * TE_EPI);
        }
        fence_barrier_init();
    }
    if (warp == 0)
        tmem_alloc<2 * TE_P>(tmem_slot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------- MMA warp (elected lane issues) ----------------
        constexpr uint32_t idesc = idesc_tf32(128, TE_P);
        const uint64_t ad = umma_desc_sw128(smem_u32(abuf), 1024);
        const uint64_t bd0 = umma_desc_sw128(smem_u32(bbuf), 1024);
        uint32_t it = 0;
        for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
            const uint32_t st = it & 1, ph = (it >> 1) & 1;
            mbar_wait(&tmem_empty[st], ph ^ 1);
            mbar_wait(&b_full[st], ph);
            tc_fence_after();
            const uint64_t bd = bd0 + ((st * TE_BBYTES) >> 4);
#pragma unroll
            for (int c = 0; c < TE_KCH; c++)
#pragma unroll
                for (int k = 0; k < 4; k++)
                    mma_tf32_warp(tmem_base + st * TE_P, ad + ((c * TE_ACH + k * 32) >> 4),
                                  bd + ((c * TE_BCH + k * 32) >> 4), idesc, (c | k) != 0);
            mma_commit_warp(&b_empty[st]);
            mma_commit_warp(&tmem_full[st]);
        }
    } else if (warp <= TE_BUILD) {
        // ---------------- im2col builders: rows r = bt, bt + 128 of the tile ----------------
        const int bt = threadIdx.x - 32;
        uint32_t it = 0;
        for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
            const uint32_t st = it & 1, ph = (it >> 1) & 1;
            mbar_wait(&b_empty[st], ph ^ 1);
            uint8_t* tb = bbuf + st * TE_BBYTES;
#pragma unroll
            for (int rr = 0; rr < 2; rr++) {
                const int r = bt + rr * 128;
                const long p = tile * TE_P + r;
                float v[20], lo[20];
#pragma unroll
                for (int q = 0; q < 20; q++)
                    v[q] = lo[q] = 0.f;
                if (p < npix) {
                    const int x = int(p % X), y = int((p / X) % Y);
                    const long b = p / (long(X) * Y);
#pragma unroll
                    for (int ty = 0; ty < 3; ty++)
#pragma unroll
                        for (int tx = 0; tx < 3; tx++) {
                            const int hx = x + tx - ox, hy = y + ty - oy;
                            if (hx >= 0 && hx < X && hy >= 0 && hy < Y) {
                                const float2 tv = thin[(b * Y + hy) * X + hx];
                                const int q = 2 * (tx + 3 * ty);
                                v[q] = sm100::to_tf32(tv.x);
                                v[q + 1] = sm100::to_tf32(tv.y);
                                lo[q] = sm100::to_tf32(tv.x - v[q]);
                                lo[q + 1] = sm100::to_tf32(tv.y - v[q + 1]);
                            }
                        }
                }
                // row k = [hi 0..17 | lo 18..35 | hi 36..53 | 0 54..63]
                float row[56];
#pragma unroll
                for (int q = 0; q < 18; q++) {
                    row[q] = v[q];
                    row[18 + q] = lo[q];
                    row[36 + q] = v[q];
                }
                row[54] = row[55] = 0.f;
#pragma unroll
                for (int g = 0; g < 14; g++)
                    *reinterpret_cast<float4*>(tb + (g >> 3) * TE_BCH + sw128_off(r, g & 7)) =
                        make_float4(row[4 * g], row[4 * g + 1], row[4 * g + 2], row[4 * g + 3]);
            }
            fence_proxy_async_smem();
            mbar_arrive(&b_full[st]);
        }
    } else {
        // ---------------- epilogue: TMEM lane = channel, column = pixel ----------------
        const int ew = warp - 1 - TE_BUILD, lg = warp & 3, rep = ew >> 2, n = lg * 32 + lane;
        // staged 16 x 32 blocks leave by TMA tensor stores (rows past npix are clipped):
        // the per-pixel 128-B STG stream was LSU-throttled
        float* stg = reinterpret_cast<float*>(smem + TeSmem::STG_OFF + ew * 2 * TE_STG);
        if (lane == 0)
            prefetch_tmap(&tm_out);
        int sb = 0;
        double s_acc = 0, q_acc = 0;
        const int bc = n & 63, comp = n >> 6;
        float2 bmu{0.f, 0.f}, bg{0.f, 0.f}, bb{0.f, 0.f};
        float bs = 0.f;
        if (EPI == 2) {
            bmu = be.mu[bc];
            bs = be.istd[bc];
            bg = be.gamma[bc];
            bb = be.beta[bc];
        }
        double r0 = 0, r1 = 0, r2 = 0;
        uint32_t it = 0;
        for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
            const uint32_t st = it & 1, ph = (it >> 1) & 1;
            mbar_wait(&tmem_full[st], ph);
            tc_fence_after();
            const uint32_t acc = tmem_base + st * TE_P + (uint32_t(lg * 32) << 16);
            float t0 = 0.f, t1 = 0.f, t2 = 0.f; // BN-backward sums of the tile (fp32, then double)
#pragma unroll 1
            for (int jc = rep; jc < TE_P / 16; jc += TE_EPI / 4) {
                const long p0 = tile * TE_P + jc * 16;
                const int nv = npix - p0 < 16 ? int(npix - p0) : 16;
                float v[16];
                tmem_ld16(acc + jc * 16, v);
                tmem_ld_wait();
                if (p0 >= npix)
                    continue;
                // this buffer's previous store has finished reading shared memory
                if (lane == 0)
                    bulk_wait_read<1>();
                __syncwarp();
                float* sbuf = stg + sb * (TE_STG / 4);
#pragma unroll
                for (int j = 0; j < 16; j++)
                    sbuf[j * 32 + lane] = v[j];
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&tm_out, sbuf, lg * 32, int(p0));
                    bulk_commit();
                }
                sb ^= 1;
                if (EPI == 1) {
                    // shifted by the chunk's first value, re-centred in double (see conv_tc.cu)
                    const float sh = v[0];
                    float fs = 0.f, fq = 0.f;
#pragma unroll
                    for (int j = 0; j < 16; j++) {
                        if (j < nv) {
                            const float d = v[j] - sh;
                            fs += d;
                            fq = fmaf(d, d, fq);
                        }
                    }
                    s_acc += double(nv) * sh + fs;
                    q_acc += double(sh) * (double(nv) * sh + 2.0 * fs) + fq;
                }
                if (EPI == 2) {
                    // BN input of the chunk (after the store is staged: the 672-thread CTA
                    // caps registers at 80, and holding x across the staging spilled)
                    float xr[16], xi[16];
                    const float* xp = be.x + p0 * 128 + bc;
#pragma unroll
                    for (int j = 0; j < 16; j++) {
                        xr[j] = j < nv ? __ldg(xp + j * 128) : 0.f;
                        xi[j] = j < nv ? __ldg(xp + j * 128 + 64) : 0.f;
                    }
                    float f0 = 0.f, f1 = 0.f, f2 = 0.f;
#pragma unroll
                    for (int j = 0; j < 16; j++) {
                        // yhat and z exactly as bn_z (bnblock.cu)
                        const float hr = (xr[j] - bmu.x) * bs, hi = (xi[j] - bmu.y) * bs;
                        const float zr = bg.x * hr - bg.y * hi + bb.x;
                        const float zi = bg.x * hi + bg.y * hr + bb.y;
                        const float ge = (j < nv && (comp ? zi : zr) > 0.f) ? v[j] : 0.f;
                        f0 += ge;
                        f1 = fmaf(ge, comp ? hi : hr, f1);
                        f2 = fmaf(ge, comp ? hr : -hi, f2);
                    }
                    t0 += f0;
                    t1 += f1;
                    t2 += f2;
                }
            }
            tc_fence_before();
            mbar_arrive(&tmem_empty[st]);
            if (EPI == 2) {
                r0 += t0;
                r1 += t1;
                r2 += t2;
            }
        }
        if (lane == 0)
            bulk_wait<0>(); // stores complete before the kernel's writes are consumed
        if (EPI == 2) {
            const size_t slot = size_t(blockIdx.x) * (TE_EPI / 4) + rep;
            be.part[(slot * 128 + n) * 3] = r0;
            be.part[(slot * 128 + n) * 3 + 1] = r1;
            be.part[(slot * 128 + n) * 3 + 2] = r2;
        }
        if (EPI == 1) {
            const size_t slot = size_t(blockIdx.x) * (TE_EPI / 4) + rep;
            stats[(slot * 128 + n) * 2] = s_acc;
            stats[(slot * 128 + n) * 2 + 1] = q_acc;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<2 * TE_P>(tmem_base);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 tp_encode()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess)
            throw CudaError("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

CUtensorMap tp_map(const float* base, long rows, int box_rows)
{
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(TP_K), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(TP_K) * 4};
    cuuint32_t box[2] = {32, cuuint32_t(box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = tp_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(thin) failed: " + std::to_string(int(r)));
    return m;
}

bool g_thin_tc = true;
// the tensor-core expand is correct but measured slower than the CUDA-core
// kernel at C2 (~2.9 vs 2.7 ms per two steps: its 512-B-per-pixel stores, not
// the FLOPs, bound both) -- off by default, option "conv_thin_tc_expand"
bool g_thin_tc_expand = false;
// the tensor-core expand for the last layer's bwd-data when its epilogue can
// also take the last BN block's backward reduction
bool g_thin_tc_bnb = true;

} // namespace

void conv_thin_tc_enable(bool on) { g_thin_tc = on; }
void conv_thin_tc_expand_enable(bool on) { g_thin_tc_expand = on; }
void conv_thin_tc_bnb_enable(bool on) { g_thin_tc_bnb = on; }
bool conv_thin_tc_bnb() { return g_thin_tc && g_thin_tc_bnb; }

long thin_expand_tc_blocks() { return long(ctx().sm_count) * (TE_EPI / 4); }

bool thin_expand_tc(float* out, const cfloat* thin, const float2* U, long X, long Y, long B, int F, int KK, int ox,
                    int oy, double* stats, int* stats_blocks, const BnBwdHint* bnb, double* bpart, int* bblocks)
{
    if (stats_blocks)
        *stats_blocks = 0;
    if (bblocks)
        *bblocks = 0;
    // the BN-backward-fused bwd-data (option conv_thin_tc_bnb) or everything (conv_thin_tc_expand)
    const bool bn = bnb && bpart && bblocks && g_thin_tc_bnb && bnb->C == F && bnb->npix == X * Y * B;
    if (!g_thin_tc || !(g_thin_tc_expand || bn) || F != 64 || KK != 9)
        return false;
    auto& c = ctx();
    const long npix = X * Y * B;
    float* ue;
    CUDA_CHECK(cudaMallocAsync(&ue, sizeof(float) * 128 * 64, c.stream));
    pdl_launch(k_pack_thin_expand, 32, 256, 0, c.stream, ue, U, F, KK);
    KERNEL_CHECK();
    const long ntiles = (npix + TE_P - 1) / TE_P;
    const int grid = int(std::min<long>(ntiles, c.sm_count));
    CUtensorMap tmo;
    {
        cuuint64_t dims[2] = {cuuint64_t(128), cuuint64_t(npix)};
        cuuint64_t strides[1] = {cuuint64_t(128) * 4};
        cuuint32_t box[2] = {32, 16};
        cuuint32_t es[2] = {1, 1};
        CUresult r = tp_encode()(&tmo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            throw CudaError("cuTensorMapEncodeTiled(expand out) failed: " + std::to_string(int(r)));
    }
    TeBn be{};
    if (bn)
        be = TeBn{bnb->x, bnb->mu, bnb->istd, bnb->gamma, bnb->beta, bpart};
    auto kern = bn ? k_thin_expand_tc<2> : stats ? k_thin_expand_tc<1> : k_thin_expand_tc<0>;
    {
        static std::mutex mu;
        static std::map<int, bool> done;
        const int e = bn ? 2 : stats ? 1 : 0;
        std::lock_guard<std::mutex> lk(mu);
        if (!done[c.device * 4 + e]) {
            CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TeSmem::TOTAL));
            done[c.device * 4 + e] = true;
        }
    }
    pdl_launch(kern, grid, TE_THREADS, TeSmem::TOTAL, c.stream, tmo, thin, ue, int(X), int(Y), npix, ox, oy, stats, be);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(ue, c.stream));
    if (stats && stats_blocks)
        *stats_blocks = grid * (TE_EPI / 4);
    if (bn)
        *bblocks = grid * (TE_EPI / 4);
    return true;
}

bool thin_reduce_tc(cfloat* out, const float* wide, const float2* U, long X, long Y, long B, int F, int KK, int ox,
                    int oy)
{
    if (!g_thin_tc || F != 64 || KK != 9)
        return false;
    auto& c = ctx();
    const long npix = X * Y * B;
    float *ut, *z;
    CUDA_CHECK(cudaMallocAsync(&ut, sizeof(float) * TP_N * TP_K, c.stream));
    CUDA_CHECK(cudaMallocAsync(&z, sizeof(float) * size_t(npix) * TP_ZP, c.stream));
    pdl_launch(k_pack_thin_tc, (TP_N * TP_K + 255) / 256, 256, 0, c.stream, ut, U, F, KK);
    KERNEL_CHECK();
    const CUtensorMap ta = tp_map(wide, npix, TP_ROWS), tb = tp_map(ut, TP_N, TP_N);
    static std::mutex mu;
    static std::map<int, bool> done;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!done[c.device]) {
            CUDA_CHECK(cudaFuncSetAttribute(k_thin_proj, cudaFuncAttributeMaxDynamicSharedMemorySize, TpSmem::TOTAL));
            done[c.device] = true;
        }
    }
    const long ntiles = (npix + TP_ROWS - 1) / TP_ROWS;
    pdl_launch(k_thin_proj, int(std::min<long>(ntiles, c.sm_count)), TP_THREADS, TpSmem::TOTAL, c.stream, ta, tb, z, npix);
    KERNEL_CHECK();
    pdl_launch(k_thin_gather, int(std::min<long>((npix + 255) / 256, 8L * c.sm_count)), 256, 0, c.stream, out, z, int(X), int(Y), npix, ox, oy);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(ut, c.stream));
    CUDA_CHECK(cudaFreeAsync(z, c.stream));
    return true;
}

} // namespace mdnn
