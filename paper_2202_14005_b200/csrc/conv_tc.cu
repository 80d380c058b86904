// Complex 3x3 "same" convolution as a TF32 implicit GEMM on the 5th-generation
// tensor cores (tcgen05 + TMEM + TMA), for the MoDL 64->64 layers
// (conv_tenmul, nn.hpp:305-337; SURVEY §7 hard part 3).
//
// Real formulation: activations channels-last planar (CHLAST: per pixel
// [Re c0..c(C-1) | Im c0..c(C-1)]), one real GEMM per tap
//   out[p, (Re f | Im f)] += in[p + tap, (Re c | Im c)] * [[Re u, Im u], [-Im u, Re u]]
// with u = w[t,c,f] (forward) or conj(w[flip t, f, c]) (backward-data).
//
// CTA work unit ("super-tile"): 16 x 16 output pixels of one item = 2 UMMA
// M-tiles of 8 x 16 pixels, each with its own TMEM accumulator, and the
// accumulator set double-buffered (2 x 2 x N columns) so that the epilogue of
// one super-tile overlaps the MMAs of the next (serialised, the epilogue's
// 256 KB of stores per 512 pixels cost ~30% of the MMA time).  Per 32-float
// K-chunk the CTA TMA-loads ONE zero-padded halo of 18 x 18 pixels (pitch 24,
// SWIZZLE_128B, 54 KB) and feeds all 9 taps from row-shifted shared-memory
// views of it (UMMA start address + base_offset), so activations cross
// L2->SMEM 1.7x instead of 9x; the packed weights stream per (tap, chunk)
// through a 4-stage TMA ring and are reused by the M-tiles.
// Warp roles: warp 0 TMA producer, warp 1 TMEM allocator + single-thread MMA
// issuer, warps 2-5 epilogue (TMEM -> registers -> global).  Persistent grid.
// Operands are rounded to TF32 with round-to-nearest by their producers
// (truncation would cost 7.8e-4 of the 1e-3 budget).
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

constexpr int NM = 2;                  // UMMA M-tiles (8 x 16 pixels each) per super-tile
constexpr int TILE_X = 8 * NM, TILE_Y = 16;
constexpr int HALO_P = 24;             // halo pitch (pixels per line, multiple of 8, >= TILE_X + 2)
constexpr int HALO_L = TILE_Y + 2;     // halo lines
constexpr int HALO_BYTES = HALO_L * HALO_P * 128;
constexpr int NBSTAGE = 6;
constexpr int NTHREADS = 192;

// epilogue staging per warp: 32 pixels x 16 accumulator columns, pitch 20 floats
constexpr int EPI_PITCH = 20;
constexpr int EPI_WARP_BYTES = 32 * EPI_PITCH * 4;

// ---------------------------------------------------------------------------
// Transposed form for 2*Cout = 128 (the MoDL 64 -> 64 layers): one UMMA
// computes D^T[n = output (re|im) channel, 128][p = pixel, 256] over an
// 8 x 32 pixel super-tile, with the packed weights Bt[n][k] as the A operand
// (M = 128) and the activation halo view as the B operand (N = 256, 8-pixel
// core-matrix rows strided by the halo line pitch).  Against the pixel-major
// form (M = 128 pixels, N = 128) every MMA instruction does twice the work --
// the single-thread issue loop was the limit there -- and reads 12 KB of
// operands per 2 x 128 x 128 x 8 MACs instead of 16 KB.  The accumulator is
// double-buffered (2 x 256 TMEM columns) so the epilogue of one super-tile
// overlaps the MMAs of the next; TMEM lane = output channel, so each warp
// store writes one pixel's 32 consecutive channels (128 B, coalesced).
constexpr int TT_X = 8, TT_Y = 32;             // super-tile (pixels)
constexpr int TT_P = 16;                       // halo pitch (>= TT_X + 2, multiple of 8)
constexpr int TT_L = TT_Y + 2;                 // halo lines
constexpr int TT_HALO = TT_L * TT_P * 128;     // 68 KB per 32-float chunk
constexpr int TT_WST = 4;                      // weight stages (16 KB each)
constexpr int TT_EPI_WARPS = 16;               // epilogue warps (4 per TMEM lane quarter)
constexpr int TT_THREADS = 64 + 32 * TT_EPI_WARPS;

struct TtSmem {
    static constexpr int W_BYTES = 128 * 128;
    static constexpr int HALO_OFF = 0;
    static constexpr int W_OFF = 2 * TT_HALO;
    static constexpr int BAR_OFF = W_OFF + TT_WST * W_BYTES;
    static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

// batch-norm backward reduction folded into the bwd-data epilogue: the
// produced cotangent is the BN block's output cotangent g; per real channel
// lane (Re or Im part of complex channel c) accumulate the CReLU-masked g and
// its contributions to S2 = sum gz conj(yhat) (bnblock.cu k_bwd_reduce).
struct BnEpi {
    const float* x = nullptr; // BN input (CHLAST, 2 C = 128 floats per pixel)
    const float2* mu = nullptr;
    const float* istd = nullptr;
    const float2* gamma = nullptr;
    const float2* beta = nullptr;
    double* part = nullptr; // [blk][128][3]
};

// EPI: epilogue kind, a compile-time choice so each form carries only its own
// registers (the 576-thread CTA caps them at 96): 0 = store only, 1 = store +
// forward BN statistics, 2 = store + BN-backward partials (bwd-data)
template<int CIN2, int EPI>
__global__ void __launch_bounds__(TT_THREADS, 1)
    k_conv_tc_t(const __grid_constant__ CUtensorMap tm_act, const __grid_constant__ CUtensorMap tm_w,
                float* __restrict__ out, int X, int Y, int B, int dbg, double* __restrict__ stats, const BnEpi be)
{
    MDNN_PDL_ENTRY();
    static_assert(CIN2 % 32 == 0, "K per tap must be a multiple of 32 floats");
    constexpr int N = 128, NP = TT_X * TT_Y, NCH = CIN2 / 32;
    using S = TtSmem;
    extern __shared__ uint8_t smem_raw[];
    // aligned by an offset from the shared array (not an integer round trip), so
    // the compiler keeps the shared address space: LDS/STS, not generic LD/ST
    uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* halo = smem + S::HALO_OFF;
    uint8_t* wst = smem + S::W_OFF;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
    uint64_t* halo_full = bars;        // [2]
    uint64_t* halo_empty = bars + 2;   // [2]
    uint64_t* w_full = bars + 4;       // [TT_WST]
    uint64_t* w_empty = bars + 4 + TT_WST;
    uint64_t* tmem_full = bars + 4 + 2 * TT_WST; // [2]
    uint64_t* tmem_empty = tmem_full + 2;        // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int tiles_x = (X + TT_X - 1) / TT_X, tiles_y = (Y + TT_Y - 1) / TT_Y;
    const int ntiles = tiles_x * tiles_y * B;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tm_act);
        prefetch_tmap(&tm_w);
        for (int i = 0; i < 2; i++) {
            mbar_init(&halo_full[i], 1);
            mbar_init(&halo_empty[i], 1);
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 32 * TT_EPI_WARPS);
        }
        for (int i = 0; i < TT_WST; i++) {
            mbar_init(&w_full[i], 1);
            mbar_init(&w_empty[i], 1);
        }
        fence_barrier_init();
    }
    if (warp == 1)
        tmem_alloc<2 * NP>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            uint32_t hi = 0, wi = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int tx = tile % tiles_x, ty = (tile / tiles_x) % tiles_y, b = tile / (tiles_x * tiles_y);
                const int x0 = tx * TT_X, y0 = ty * TT_Y;
                for (int c = 0; c < NCH; c++, hi++) {
                    const uint32_t hb = hi & 1, hph = (hi >> 1) & 1;
                    mbar_wait(&halo_empty[hb], hph ^ 1);
                    mbar_arrive_expect_tx(&halo_full[hb], TT_HALO);
                    tma_load_4d(halo + hb * TT_HALO, &tm_act, &halo_full[hb], c * 32, x0 - 1, y0 - 1, b);
                    for (int t = 0; t < 9; t++, wi++) {
                        const uint32_t st = wi % TT_WST, ph = (wi / TT_WST) & 1;
                        mbar_wait(&w_empty[st], ph ^ 1);
                        mbar_arrive_expect_tx(&w_full[st], S::W_BYTES);
                        tma_load_2d(wst + st * S::W_BYTES, &tm_w, &w_full[st], t * CIN2 + c * 32, 0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        {
            // ---------------- MMA issuer (whole warp, elected lane issues) ----------------
            constexpr uint32_t idesc = idesc_tf32(128, NP);
            uint32_t hi = 0, wi = 0, ti = 0;
            const uint64_t hdesc0 = umma_desc_sw128(smem_u32(halo), TT_P * 128);
            const uint64_t wdesc0 = umma_desc_sw128(smem_u32(wst), 1024);
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ti++) {
                const uint32_t ab = ti & 1, acc = tmem_base + ab * NP;
                mbar_wait(&tmem_empty[ab], ((ti >> 1) & 1) ^ 1);
                tc_fence_after();
                for (int c = 0; c < NCH; c++, hi++) {
                    const uint32_t hb = hi & 1, hph = (hi >> 1) & 1;
                    mbar_wait(&halo_full[hb], hph);
                    tc_fence_after();
                    const uint64_t hdesc = hdesc0 + (hb * TT_HALO >> 4);
#pragma unroll
                    for (int t = 0; t < 9; t++, wi++) {
                        const uint32_t st = wi % TT_WST, ph = (wi / TT_WST) & 1;
                        mbar_wait(&w_full[st], ph);
                        tc_fence_after();
                        const uint64_t wdesc = wdesc0 + (st * S::W_BYTES >> 4);
                        const int ky = t / 3, kx = t % 3;
#pragma unroll
                        for (int k = 0; k < 4; k++)
                            mma_tf32_warp(acc, wdesc + (k * 32 >> 4), hdesc + (((ky * TT_P + kx) * 128 + k * 32) >> 4), idesc,
                                     (c | t | k) != 0);
                        mma_commit_warp(&w_empty[st]);
                    }
                    mma_commit_warp(&halo_empty[hb]);
                }
                mma_commit_warp(&tmem_full[ab]);
            }
        }
    } else {
        // ---------------- epilogue: TMEM lane = channel, column = pixel ----------------
        // TT_EPI_WARPS epilogue warps: TT_EPI_WARPS / 4 per TMEM lane quarter, interleaved 32-column chunks
        const int lg = warp & 3, n = lg * 32 + lane, half = (warp - 2) >> 2;
        // per-channel sum and sum of squares of the stored values (fp32 over
        // 32 pixels, then double), for a batch-norm consumer
        double s_acc = 0, q_acc = 0;
        // batch-norm backward partials (be.part): channel c = n mod 64, component n / 64
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
        uint32_t ti = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ti++) {
            // BN-backward sums of this tile's chunks (fp32 over NP / 16 / 4 chunks of
            // 16 pixels, then double: one FP64 add per tile, not per chunk)
            float t0 = 0.f, t1 = 0.f, t2 = 0.f;
            const int tx = tile % tiles_x, ty = (tile / tiles_x) % tiles_y, b = tile / (tiles_x * tiles_y);
            const int x0 = tx * TT_X, y0 = ty * TT_Y;
            const uint32_t ab = ti & 1, acc = tmem_base + ab * NP + (uint32_t(lg * 32) << 16);
            mbar_wait(&tmem_full[ab], (ti >> 1) & 1);
            tc_fence_after();
            const bool full_x = x0 + TT_X <= X;
#pragma unroll 1
            for (int jc = half; jc < NP / 16 && dbg != 2; jc += TT_EPI_WARPS / 4) {
                const int py0 = y0 + jc * 2; // 16 columns = 2 lines x 8 pixels
                if (py0 >= Y)
                    break;
                // every pixel of the chunk in range (all but the image's last tile row / column)
                const bool full = (full_x || x0 + 8 <= X) && py0 + 2 <= Y;
                // BN-backward consumer: the BN input x of the chunk's pixels, issued
                // before the TMEM load so their latency overlaps it and the stores
                float xr[16], xi[16];
                if (EPI == 2) {
                    const float* xp = be.x + ((long(b) * Y + py0) * X + x0) * N + bc;
#pragma unroll
                    for (int j = 0; j < 16; j++) { // 32 loads in flight
                        const int l = j >> 3, xo = j & 7;
                        const bool ok = full || ((full_x || x0 + xo < X) && py0 + l < Y);
                        const long off = (long(l) * X + xo) * N;
                        xr[j] = ok ? __ldg(xp + off) : 0.f;
                        xi[j] = ok ? __ldg(xp + off + 64) : 0.f;
                    }
                }
                float v[16];
                tmem_ld16(acc + jc * 16, v);
                tmem_ld_wait();
                float* o = out + ((long(b) * Y + py0) * X + x0) * N + n;
                if (dbg != 1) {
#pragma unroll
                    for (int j = 0; j < 16; j++) {
                        const int l = j >> 3, xo = j & 7;
                        if (full || ((full_x || x0 + xo < X) && py0 + l < Y))
                            o[(long(l) * X + xo) * N] = v[j];
                    }
                }
                if (EPI == 1) {
                    // fp32 sums shifted by the chunk's first value (always in range), so the
                    // sum of squares carries the spread, not the mean; re-centred in double
                    const float sh = v[0];
                    float fs = 0.f, fq = 0.f;
                    int nv = 0;
#pragma unroll
                    for (int j = 0; j < 16; j++) {
                        const int l = j >> 3, xo = j & 7;
                        if (full || ((full_x || x0 + xo < X) && py0 + l < Y)) {
                            const float d = v[j] - sh;
                            fs += d;
                            fq = fmaf(d, d, fq);
                            nv++;
                        }
                    }
                    s_acc += double(nv) * sh + fs;
                    q_acc += double(sh) * (double(nv) * sh + 2.0 * fs) + fq;
                }
                if (EPI == 2) {
                    float f0 = 0.f, f1 = 0.f, f2 = 0.f;
#pragma unroll
                    for (int j = 0; j < 16; j++) {
                        const int l = j >> 3, xo = j & 7;
                        const bool ok = full || ((full_x || x0 + xo < X) && py0 + l < Y);
                        // yhat and z exactly as bn_z (bnblock.cu)
                        const float hr = (xr[j] - bmu.x) * bs, hi = (xi[j] - bmu.y) * bs;
                        const float zr = bg.x * hr - bg.y * hi + bb.x;
                        const float zi = bg.x * hi + bg.y * hr + bb.y;
                        const float ge = (ok && (comp ? zi : zr) > 0.f) ? v[j] : 0.f;
                        f0 += ge;
                        // Re lane: (g_r hr, -g_r hi); Im lane: (g_i hi, g_i hr)
                        f1 = fmaf(ge, comp ? hi : hr, f1);
                        f2 = fmaf(ge, comp ? hr : -hi, f2);
                    }
                    t0 += f0;
                    t1 += f1;
                    t2 += f2;
                }
            }
            tc_fence_before();
            mbar_arrive(&tmem_empty[ab]);
            if (EPI == 2) {
                r0 += t0;
                r1 += t1;
                r2 += t2;
            }
        }
        // one partial block per (CTA, epilogue half)
        const size_t slot = size_t(blockIdx.x) * (TT_EPI_WARPS / 4) + half;
        if (EPI == 1) {
            stats[(slot * N + n) * 2] = s_acc;
            stats[(slot * N + n) * 2 + 1] = q_acc;
        }
        if (EPI == 2) {
            be.part[(slot * N + n) * 3] = r0;
            be.part[(slot * N + n) * 3 + 1] = r1;
            be.part[(slot * N + n) * 3 + 2] = r2;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<2 * NP>(tmem_base);
    }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cluster of 2, tcgen05 cta_group::2): the pair runs one
// M = 256 UMMA per (M-tile, tap, k-step) whose rows 0-127 come from the leader
// CTA's halo view and rows 128-255 from the peer's (two neighbouring
// super-tiles), and whose B operand (packed weights) is split by N: each CTA
// TMA-loads and holds only its N/2 rows of every weight stage.  Per CTA this
// halves the weight traffic from L2 and the weight reads from shared memory
// (the 1-CTA kernel's two limits: ~40 B/clk of L2->SMEM and ~120 B/clk of
// SMEM operand reads per SM at the TF32 rate).  The leader's single thread
// issues all MMAs; the TMA loads of both CTAs complete on the leader's
// full-barriers (.cta_group::2), and the leader's commits arrive on the
// empty / accumulator-full barriers of both CTAs (multicast).  Both epilogues
// release the accumulator buffer on the leader's barrier (8 warp arrivals).
template<int N>
struct TcPairSmem {
    static constexpr int B_BYTES = (N / 2) * 128; // this CTA's half of a weight stage
    static constexpr int HALO_OFF = 0;
    static constexpr int B_OFF = 2 * HALO_BYTES;
    static constexpr int EPI_OFF = B_OFF + NBSTAGE * B_BYTES;
    static constexpr int BAR_OFF = EPI_OFF + 4 * EPI_WARP_BYTES;
    static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

template<int CIN2, int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    k_conv_tc_pair(const __grid_constant__ CUtensorMap tm_act, const __grid_constant__ CUtensorMap tm_w,
                   float* __restrict__ out, int X, int Y, int B, int dbg)
{
    MDNN_PDL_ENTRY();
    static_assert(CIN2 % 32 == 0, "K per tap must be a multiple of 32 floats");
    static_assert(N % 32 == 0 && N >= 32 && 2 * NM * N <= 512, "N must fit 2 x NM accumulators in TMEM");
    constexpr int NCH = CIN2 / 32;
    constexpr int ACC = 2 * NM * N;
    constexpr int TMEM_COLS = ACC <= 32 ? 32 : (ACC <= 64 ? 64 : (ACC <= 128 ? 128 : (ACC <= 256 ? 256 : 512)));
    using S = TcPairSmem<N>;

    extern __shared__ uint8_t smem_raw[];
    // aligned by an offset from the shared array (not an integer round trip), so
    // the compiler keeps the shared address space: LDS/STS, not generic LD/ST
    uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* halo = smem + S::HALO_OFF;
    uint8_t* bst = smem + S::B_OFF;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
    uint64_t* halo_full = bars;            // [2]   (leader's used)
    uint64_t* halo_empty = bars + 2;       // [2]
    uint64_t* b_full = bars + 4;           // [NBSTAGE] (leader's used)
    uint64_t* b_empty = bars + 4 + NBSTAGE;
    uint64_t* tmem_full = bars + 4 + 2 * NBSTAGE; // [2]
    uint64_t* tmem_empty = tmem_full + 2;         // [2] (leader's used)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int tiles_x = (X + TILE_X - 1) / TILE_X, tiles_y = (Y + TILE_Y - 1) / TILE_Y;
    const int ntiles = tiles_x * tiles_y * B;
    const int npairs = (ntiles + 1) / 2, ncl = gridDim.x / 2, cid = blockIdx.x / 2;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tm_act);
        prefetch_tmap(&tm_w);
        for (int i = 0; i < 2; i++) {
            mbar_init(&halo_full[i], 1);
            mbar_init(&halo_empty[i], 1);
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 8);
        }
        for (int i = 0; i < NBSTAGE; i++) {
            mbar_init(&b_full[i], 1);
            mbar_init(&b_empty[i], 1);
        }
        fence_barrier_init();
    }
    if (warp == 1)
        tmem_alloc_pair<TMEM_COLS>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer (both CTAs) ----------------
            uint32_t hi = 0, bi = 0;
            for (int q = cid; q < npairs; q += ncl) {
                const int tile = 2 * q + int(rank); // past the end: OOB coordinates, zero-filled
                const int tx = tile % tiles_x, ty = (tile / tiles_x) % tiles_y, b = tile / (tiles_x * tiles_y);
                const int x0 = tx * TILE_X, y0 = ty * TILE_Y;
                for (int c = 0; c < NCH; c++, hi++) {
                    const uint32_t hb = hi & 1, hph = (hi >> 1) & 1;
                    mbar_wait(&halo_empty[hb], hph ^ 1);
                    if (leader)
                        mbar_arrive_expect_tx(&halo_full[hb], 2 * HALO_BYTES);
                    tma_load_4d_pair(halo + hb * HALO_BYTES, &tm_act, mapa_shared(&halo_full[hb], 0), c * 32, x0 - 1,
                                     y0 - 1, b);
                    for (int t = 0; t < 9; t++, bi++) {
                        const uint32_t st = bi % NBSTAGE, bph = (bi / NBSTAGE) & 1;
                        mbar_wait(&b_empty[st], bph ^ 1);
                        if (leader)
                            mbar_arrive_expect_tx(&b_full[st], 2 * S::B_BYTES);
                        tma_load_2d_pair(bst + st * S::B_BYTES, &tm_w, mapa_shared(&b_full[st], 0),
                                         t * CIN2 + c * 32, int(rank) * (N / 2));
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            // ---------------- MMA issuer (leader CTA, single thread) ----------------
            constexpr uint32_t idesc = idesc_tf32(256, N);
            uint32_t hi = 0, bi = 0, ti = 0;
            const uint32_t halo_addr = smem_u32(halo), b_addr = smem_u32(bst);
            for (int q = cid; q < npairs; q += ncl, ti++) {
                const uint32_t ab = ti & 1, acc = tmem_base + ab * NM * N;
                mbar_wait(&tmem_empty[ab], ((ti >> 1) & 1) ^ 1);
                tc_fence_after();
                for (int c = 0; c < NCH; c++, hi++) {
                    const uint32_t hb = hi & 1, hph = (hi >> 1) & 1;
                    mbar_wait(&halo_full[hb], hph);
                    tc_fence_after();
                    const uint32_t hbase = halo_addr + hb * HALO_BYTES;
                    for (int t = 0; t < 9; t++, bi++) {
                        const uint32_t st = bi % NBSTAGE, bph = (bi / NBSTAGE) & 1;
                        mbar_wait(&b_full[st], bph);
                        tc_fence_after();
                        const int ky = t / 3, kx = t % 3;
                        const uint32_t bbase = b_addr + st * S::B_BYTES;
#pragma unroll
                        for (int xt = 0; xt < NM; xt++) {
                            const uint32_t row0 = ky * HALO_P + xt * 8 + kx;
#pragma unroll
                            for (int k = 0; k < 4; k++) {
                                const uint64_t ad = umma_desc_sw128(hbase + row0 * 128 + k * 32, HALO_P * 128);
                                const uint64_t bd = umma_desc_sw128(bbase + k * 32, 1024);
                                mma_tf32_pair(acc + xt * N, ad, bd, idesc, (c | t | k) != 0);
                            }
                        }
                        mma_commit_pair(&b_empty[st], 0x3);
                    }
                    mma_commit_pair(&halo_empty[hb], 0x3);
                }
                mma_commit_pair(&tmem_full[ab], 0x3);
            }
        }
    } else {
        // ---------------- epilogue (both CTAs): own TMEM lanes = own super-tile ----------------
        const int lg = warp & 3;
        float* estage = reinterpret_cast<float*>(smem + S::EPI_OFF + lg * EPI_WARP_BYTES);
        uint32_t ti = 0;
        for (int q = cid; q < npairs; q += ncl, ti++) {
            const int tile = 2 * q + int(rank);
            const int tx = tile % tiles_x, ty = (tile / tiles_x) % tiles_y, b = tile / (tiles_x * tiles_y);
            const int x0 = tx * TILE_X, y0 = ty * TILE_Y;
            const uint32_t ab = ti & 1, acc = tmem_base + ab * NM * N;
            mbar_wait(&tmem_full[ab], (ti >> 1) & 1);
            tc_fence_after();
            const bool store = tile < ntiles && dbg != 2;
            const int qd = lane & 3, pl = lane >> 2;
#pragma unroll 1
            for (int xt = 0; xt < NM && store; xt++) {
#pragma unroll 1
                for (int nc = 0; nc < N / 16; nc++) {
                    float v[16];
                    tmem_ld16(acc + (uint32_t(lg * 32) << 16) + xt * N + nc * 16, v);
                    tmem_ld_wait();
                    float4* st4 = reinterpret_cast<float4*>(estage + lane * EPI_PITCH);
#pragma unroll
                    for (int q4 = 0; q4 < 4; q4++)
                        st4[q4] = make_float4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]);
                    __syncwarp();
#pragma unroll
                    for (int it = 0; it < 4; it++) {
                        const int rr = it * 8 + pl;
                        const int px = x0 + xt * 8 + pl, py = y0 + lg * 4 + it;
                        const float4 val = reinterpret_cast<const float4*>(estage + rr * EPI_PITCH)[qd];
                        if (px < X && py < Y && dbg != 1)
                            reinterpret_cast<float4*>(out + ((long(b) * Y + py) * X + px) * N + nc * 16)[qd] = val;
                    }
                    __syncwarp();
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0)
                mbar_arrive_cluster(mapa_shared(&tmem_empty[ab], 0));
        }
    }
    tc_fence_before();
    cluster_sync(); // the peer's smem and TMEM stay live until the leader's last MMAs are done
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair<TMEM_COLS>(tmem_base);
    }
}

// ---------------------------------------------------------------------------
// Backward-weight: per tap t, D_t[m = x channel (re|im)][n = dy channel (re|im)]
//   = sum_p x[p + t - c0][m] * dy[p][n]
// as a K = pixels GEMM with both operands MN-major straight from CHLAST rows.
// A CTA owns one kernel row ky (3 accumulators, kx = 0..2, 3 x N TMEM
// columns) and a contiguous range of 64-pixel dy row segments; per segment
// it TMA-loads the dy segment and the 66-pixel x halo row once and feeds the
// 3 taps from row-shifted views.  Partials per CTA are reduced in a fixed
// order (deterministic) and folded into complex dW:
//   Re dW = D[cr][fr] + D[ci][fi],  Im dW = D[cr][fi] - D[ci][fr].
constexpr int WG_SEG = 64;                    // dy pixels per segment (8 K-steps)
constexpr int WG_XROWS = 72;                  // x halo rows per channel block (66 used, 1024-B aligned)
constexpr int WG_XBLK = WG_XROWS * 128;       // 9216 B
constexpr int WG_DBLK = WG_SEG * 128;         // 8192 B
constexpr int WG_STAGES = 3;

template<int N>
struct WgSmem {
    static constexpr int STAGE = 4 * WG_XBLK + (N / 32) * WG_DBLK;
    static constexpr int BAR_OFF = WG_STAGES * STAGE;
    static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

template<int N>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_conv_tc_wgrad(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_dy,
                    float* __restrict__ part, int X, int Y, int B, int nsplit)
{
    MDNN_PDL_ENTRY();
    using S = WgSmem<N>;
    constexpr int TMEM_COLS = 3 * N <= 128 ? 128 : (3 * N <= 256 ? 256 : 512);
    constexpr int NDB = N / 32;
    extern __shared__ uint8_t smem_raw[];
    // aligned by an offset from the shared array (not an integer round trip), so
    // the compiler keeps the shared address space: LDS/STS, not generic LD/ST
    uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
    uint64_t* full = bars;
    uint64_t* empty = bars + WG_STAGES;
    uint64_t* tmem_full = bars + 2 * WG_STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int ky = blockIdx.x % 3, split = blockIdx.x / 3;
    const int segx = (X + WG_SEG - 1) / WG_SEG;
    const long nseg = long(segx) * Y * B;
    const long s_begin = nseg * split / nsplit, s_end = nseg * (split + 1) / nsplit;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tm_x);
        prefetch_tmap(&tm_dy);
        for (int i = 0; i < WG_STAGES; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tmem_full, 1);
        fence_barrier_init();
    }
    if (warp == 1)
        tmem_alloc<TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            uint32_t it = 0;
            for (long s = s_begin; s < s_end; s++, it++) {
                const int sx = int(s % segx), y = int((s / segx) % Y), b = int(s / (long(segx) * Y));
                const int x0 = sx * WG_SEG;
                const uint32_t st = it % WG_STAGES, ph = (it / WG_STAGES) & 1;
                mbar_wait(&empty[st], ph ^ 1);
                mbar_arrive_expect_tx(&full[st], 4 * (WG_SEG + 2) * 128 + NDB * WG_SEG * 128);
                uint8_t* base = smem + st * S::STAGE;
                for (int j = 0; j < 4; j++)
                    tma_load_4d(base + j * WG_XBLK, &tm_x, &full[st], j * 32, x0 - 1, y + ky - 1, b);
                for (int j = 0; j < NDB; j++)
                    tma_load_4d(base + 4 * WG_XBLK + j * WG_DBLK, &tm_dy, &full[st], j * 32, x0, y, b);
            }
        }
    } else if (warp == 1) {
        { // whole warp, elected lane issues (mma_tf32_warp)
            // a_major = b_major = MN (bits 15, 16)
            // a_major = b_major = MN (bits 15, 16); operands SWIZZLE_128B_BASE32B
            constexpr uint32_t idesc = idesc_tf32(128, N) | (1u << 15) | (1u << 16);
            uint32_t it = 0;
            const uint32_t sbase = smem_u32(smem);
            // descriptors of stage 0; every other view is a constant start-address offset
            const uint64_t xd0 = umma_desc_mn_sw128_32b(sbase, 512, WG_XBLK);
            const uint64_t dd0 = umma_desc_mn_sw128_32b(sbase + 4 * WG_XBLK, 512, WG_DBLK);
            const int nseg_cta = int(s_end - s_begin);
            uint32_t st = 0, ph = 0; // ring position kept incrementally (no division by the stage count)
            for (int si = 0; si < nseg_cta; si++, it++) {
                if (si > 0 && ++st == WG_STAGES) {
                    st = 0;
                    ph ^= 1;
                }
                mbar_wait(&full[st], ph);
                tc_fence_after();
                // start-address field (bits 0-13) + offset: no carry for smem < 256 KB
                const uint64_t so = (st * S::STAGE) >> 4;
                const uint64_t xd = xd0 + so, dd = dd0 + so;
#pragma unroll
                for (int ks = 0; ks < WG_SEG / 8; ks++) {
                    const uint64_t bd = dd + ((ks * 8 * 128) >> 4);
#pragma unroll
                    for (int kx = 0; kx < 3; kx++)
                        mma_tf32_warp(tmem_base + kx * N, xd + (((kx + ks * 8) * 128) >> 4), bd, idesc,
                                      (si != 0 || ks != 0) ? 1u : 0u);
                }
                mma_commit_warp(&empty[st]);
            }
            mma_commit_warp(tmem_full);
        }
    } else {
        const int lg = warp & 3;
        const int m = lg * 32 + lane; // x channel (re|im)
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const bool any = s_end > s_begin;
        for (int kx = 0; kx < 3; kx++) {
            float* dst = part + ((size_t(split) * 9 + ky * 3 + kx) * 128 + m) * N;
#pragma unroll 1
            for (int nc = 0; nc < N / 32; nc++) {
                float v[32];
                tmem_ld32(tmem_base + (uint32_t(lg * 32) << 16) + kx * N + nc * 32, v);
                tmem_ld_wait();
                float4* d4 = reinterpret_cast<float4*>(dst + nc * 32);
#pragma unroll
                for (int q = 0; q < 8; q++)
                    d4[q] = any ? make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3])
                                : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem_base);
    }
}

// dw[t, c, f] from the per-split real blocks (fp64 sums in a fixed order: split group g
// sums splits g, g + 4, ...; the four groups are then added in order g = 0..3).
// Block = 64 outputs (f fastest: coalesced partial rows) x 4 split groups.
__global__ void __launch_bounds__(256) k_wgrad_fold(cfloat* __restrict__ dw, const float* __restrict__ part, int Cin,
                                                    int Cout, int N, int nsplit)
{
    MDNN_PDL_ENTRY();
    __shared__ double2 red[4][64];
    const int n_out = 9 * Cin * Cout;
    const int o = threadIdx.x & 63, g = threadIdx.x >> 6;
    const int i = blockIdx.x * 64 + o;
    double re = 0, im = 0;
    int f = 0, c = 0, t = 0;
    if (i < n_out) {
        f = i % Cout;
        c = (i / Cout) % Cin;
        t = i / (Cout * Cin);
        const size_t sstride = size_t(9) * 128 * N;
        const float* D = part + size_t(t) * 128 * N + size_t(g) * sstride;
#pragma unroll 4
        for (int s = g; s < nsplit; s += 4, D += 4 * sstride) {
            const float a0 = D[c * N + f], a1 = D[(Cin + c) * N + Cout + f];
            const float b0 = D[c * N + Cout + f], b1 = D[(Cin + c) * N + f];
            re += double(a0) + double(a1);
            im += double(b0) - double(b1);
        }
    }
    red[g][o] = double2{re, im};
    __syncthreads();
    if (g == 0 && i < n_out) {
        double2 r = red[0][o];
        for (int k = 1; k < 4; k++) {
            r.x += red[k][o].x;
            r.y += red[k][o].y;
        }
        dw[t + 9 * (c + Cin * f)] = float2{float(r.x), float(r.y)};
    }
}

// packed real-block weights Bt[n][k], k = t*CIN2 + (in re | in im), n = (out re | out im);
// mode 0 (fwd): u = w[t, c=in, f=out]; mode 1 (bwd-data): u = conj(w[flip t, c=out, f=in])
__global__ void k_pack_weights(float* __restrict__ bt, const cfloat* __restrict__ w, int KX, int KY, int Cin,
                               int Cout, int mode)
{
    MDNN_PDL_ENTRY();
    const int taps = KX * KY;
    const int nin = mode == 0 ? Cin : Cout, nout = mode == 0 ? Cout : Cin;
    const int K = taps * 2 * nin, N = 2 * nout;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < K * N; idx += gridDim.x * blockDim.x) {
        const int k = idx % K, n = idx / K;
        const int t = k / (2 * nin), kin = k % (2 * nin);
        const int ci = kin % nin, in_im = kin / nin;
        const int co = n % nout, out_im = n / nout;
        float2 u;
        if (mode == 0) {
            u = w[t + taps * (ci + Cin * co)];
        } else {
            const int tx = t % KX, tyy = t / KX;
            const int tf = (KX - 1 - tx) + KX * (KY - 1 - tyy);
            float2 ww = w[tf + taps * (co + Cin * ci)];
            u = float2{ww.x, -ww.y};
        }
        // [[Re u, Im u], [-Im u, Re u]]
        float v = !in_im ? (!out_im ? u.x : u.y) : (!out_im ? -u.y : u.x);
        bt[size_t(n) * K + k] = to_tf32(v);
    }
}

// CANON [X*Y][C][B] complex -> CHLAST floats with RN tf32 rounding (operand staging)
__global__ void k_to_chlast_tf32(float* __restrict__ out, const cfloat* __restrict__ in, long inner, long C,
                                 long outer)
{
    MDNN_PDL_ENTRY();
    __shared__ cfloat tile[32][33];
    const long pix0 = long(blockIdx.x) * 32, c0 = long(blockIdx.y) * 32, o = blockIdx.z;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        long c = c0 + k, p = pix0 + threadIdx.x;
        tile[k][threadIdx.x] = (c < C && p < inner) ? in[(o * C + c) * inner + p] : cfloat{0, 0};
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        long p = pix0 + k, c = c0 + threadIdx.x;
        if (p < inner && c < C) {
            float* dst = out + (o * inner + p) * 2 * C;
            cfloat v = tile[threadIdx.x][k];
            dst[c] = to_tf32(v.x);
            dst[C + c] = to_tf32(v.y);
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn()
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

CUtensorMap make_act_map(const float* base, int C2, int X, int Y, int B, int box_x = HALO_P, int box_y = HALO_L,
                         CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B)
{
    CUtensorMap m;
    cuuint64_t dims[4] = {cuuint64_t(C2), cuuint64_t(X), cuuint64_t(Y), cuuint64_t(B)};
    cuuint64_t strides[3] = {cuuint64_t(C2) * 4, cuuint64_t(C2) * 4 * X, cuuint64_t(C2) * 4 * X * Y};
    cuuint32_t box[4] = {32, cuuint32_t(box_x), cuuint32_t(box_y), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(activation) failed: " + std::to_string(int(r)));
    return m;
}

CUtensorMap make_w_map(const float* base, int K, int N, int box_n = 0)
{
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(N)};
    cuuint64_t strides[1] = {cuuint64_t(K) * 4};
    cuuint32_t box[2] = {32, cuuint32_t(box_n ? box_n : N)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(weights) failed: " + std::to_string(int(r)));
    return m;
}

int g_tc_dbg = 0; // diagnostics: 1 = epilogue without global stores, 2 = no epilogue

// 2 Cout = 128: channel-major kernel (k_conv_tc_t); 2 Cout = 64: CTA-pair
// pixel-major kernel (k_conv_tc_pair)
template<int CIN2, int N>
void launch_tc(const float* act, const float* wpk, float* out, int X, int Y, int B, double* stats = nullptr,
               int* stats_blocks = nullptr, const BnEpi& be = BnEpi{}, int* be_blocks = nullptr)
{
    if (stats_blocks)
        *stats_blocks = 0;
    if (be_blocks)
        *be_blocks = 0;
    auto& c = ctx();
    static std::mutex mu;
    CUtensorMap tw = make_w_map(wpk, 9 * CIN2, N);
    if constexpr (N == 128) {
        // transposed form: D^T[channel][pixel], N = 256 pixels per MMA
        CUtensorMap tat = make_act_map(act, CIN2, X, Y, B, TT_P, TT_L);
        const int epi = be.part ? 2 : stats ? 1 : 0;
        auto kt = epi == 2 ? k_conv_tc_t<CIN2, 2> : epi == 1 ? k_conv_tc_t<CIN2, 1> : k_conv_tc_t<CIN2, 0>;
        const int smem_t = TtSmem::TOTAL;
        {
            std::lock_guard<std::mutex> lk(mu);
            static std::map<int, bool> done_t;
            if (!done_t[c.device * 4 + epi]) {
                CUDA_CHECK(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_t));
                done_t[c.device * 4 + epi] = true;
            }
        }
        const int nt = ((X + TT_X - 1) / TT_X) * ((Y + TT_Y - 1) / TT_Y) * B;
        const int grid = std::min(nt, c.sm_count);
        pdl_launch(kt, grid, TT_THREADS, smem_t, c.stream, tat, tw, out, X, Y, B, g_tc_dbg, stats, be);
        KERNEL_CHECK();
        if (stats && stats_blocks)
            *stats_blocks = grid * (TT_EPI_WARPS / 4);
        if (be.part && be_blocks)
            *be_blocks = grid * (TT_EPI_WARPS / 4);
    } else {
        // CTA pairs: half of every weight stage per CTA, multicast commits
        CUtensorMap ta = make_act_map(act, CIN2, X, Y, B);
        const int ntiles = ((X + TILE_X - 1) / TILE_X) * ((Y + TILE_Y - 1) / TILE_Y) * B;
        CUtensorMap twp = make_w_map(wpk, 9 * CIN2, N, N / 2);
        auto kp = k_conv_tc_pair<CIN2, N>;
        const int smem_p = TcPairSmem<N>::TOTAL;
        {
            std::lock_guard<std::mutex> lk(mu);
            static std::map<int, bool> done_p;
            if (!done_p[c.device]) {
                CUDA_CHECK(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_p));
                done_p[c.device] = true;
            }
        }
        const int npairs = (ntiles + 1) / 2;
        const int grid = 2 * std::min(npairs, c.sm_count / 2);
        pdl_launch(kp, grid, NTHREADS, smem_p, c.stream, ta, twp, out, X, Y, B, g_tc_dbg);
        KERNEL_CHECK();
    }
}

template<int N>
void launch_tc_wgrad(const float* x, const float* dy, cfloat* dw, int X, int Y, int B, int Cin, int Cout)
{
    auto& c = ctx();
    CUtensorMap tx = make_act_map(x, 128, X, Y, B, WG_SEG + 2, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    CUtensorMap td = make_act_map(dy, N, X, Y, B, WG_SEG, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    auto kern = k_conv_tc_wgrad<N>;
    const int smem = WgSmem<N>::TOTAL;
    static std::mutex mu;
    static std::map<int, bool> done;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!done[c.device]) {
            CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            done[c.device] = true;
        }
    }
    const long nseg = long((X + WG_SEG - 1) / WG_SEG) * Y * B;
    const int nsplit = int(std::max(1L, std::min<long>(c.sm_count / 3, nseg)));
    float* part;
    CUDA_CHECK(cudaMallocAsync(&part, sizeof(float) * size_t(nsplit) * 9 * 128 * N, c.stream));
    pdl_launch(kern, 3 * nsplit, NTHREADS, smem, c.stream, tx, td, part, X, Y, B, nsplit);
    KERNEL_CHECK();
    pdl_launch(k_wgrad_fold, (9 * Cin * Cout + 63) / 64, 256, 0, c.stream, dw, part, Cin, Cout, N, nsplit);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(part, c.stream));
}

bool g_tc_enabled = true;

} // namespace

bool conv_tc_wgrad_supported(long cin, long cout, long kx, long ky)
{
    return g_tc_enabled && kx == 3 && ky == 3 && cin == 64 && (cout == 32 || cout == 64);
}

// dw = conv_bwd_weight(x, dy) on the tensor cores (x: Cin channels, dy: Cout channels)
namespace {

__global__ void k_round_tf32(float* __restrict__ out, const float* __restrict__ in, long n)
{
    MDNN_PDL_ENTRY();
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        out[i] = to_tf32(in[i]);
}

// TF32-rounded CHLAST view of a C-channel operand: the array itself when it
// already is one, else a staged copy (*tmp, freed by the caller)
const float* stage_operand(const cfloat* p, long C, const ConvGeom& g, bool chlast, bool tf32, float** tmp)
{
    *tmp = nullptr;
    if (chlast && tf32)
        return reinterpret_cast<const float*>(p);
    auto& c = ctx();
    const long inner = g.X * g.Y, n = 2 * C * inner * g.B;
    CUDA_CHECK(cudaMallocAsync(tmp, sizeof(float) * n, c.stream));
    if (chlast) {
        pdl_launch(k_round_tf32, int(std::min<long>(c.sm_count * 8, (n + 255) / 256)), 256, 0, c.stream, *tmp, reinterpret_cast<const float*>(p), n);
    } else {
        pdl_launch(k_to_chlast_tf32, dim3(unsigned((inner + 31) / 32), unsigned((C + 31) / 32), unsigned(g.B)), dim3(32, 8), 0,
                           c.stream, *tmp, p, inner, C, g.B);
    }
    KERNEL_CHECK();
    return *tmp;
}

} // namespace

void conv_tc_wgrad(cfloat* dw, const cfloat* x, const cfloat* dy, const ConvGeom& g)
{
    auto& c = ctx();
    float *xt, *dt;
    const float* xs = stage_operand(x, g.Cin, g, g.in_chlast, g.in_tf32, &xt);
    const float* ds = stage_operand(dy, g.Cout, g, g.out_chlast, g.out_tf32, &dt);
    {
        const double flops = 8.0 * double(g.X) * g.Y * g.B * g.Cin * g.Cout * 9;
        ProfScope prof("conv_tc_bwd_weight", flops);
        if (g.Cout == 64)
            launch_tc_wgrad<128>(xs, ds, dw, int(g.X), int(g.Y), int(g.B), int(g.Cin), int(g.Cout));
        else
            launch_tc_wgrad<64>(xs, ds, dw, int(g.X), int(g.Y), int(g.B), int(g.Cin), int(g.Cout));
    }
    if (xt)
        CUDA_CHECK(cudaFreeAsync(xt, c.stream));
    if (dt)
        CUDA_CHECK(cudaFreeAsync(dt, c.stream));
}

void conv_tc_enable(bool on) { g_tc_enabled = on; }
void conv_tc_debug(int mode) { g_tc_dbg = mode; }
int conv_tc_stat_slots() { return TT_EPI_WARPS / 4; }
namespace {
bool g_bn_fuse = true;
}
void conv_bn_fuse_enable(bool on) { g_bn_fuse = on; }
bool conv_bn_fuse() { return g_bn_fuse; }

namespace {
bool g_force_chlast = false;
}
void conv_force_chlast(bool on) { g_force_chlast = on; }
bool conv_chlast_forced() { return g_force_chlast; }

// 3x3, 2*Cin in {64, 128} floats per pixel, 2*Cout in {64, 128}
bool conv_tc_supported(long cin, long cout, long kx, long ky)
{
    if (!g_tc_enabled || kx != 3 || ky != 3)
        return false;
    return (cin == 32 || cin == 64) && (cout == 32 || cout == 64);
}

// mode 0: y = conv(x, w) (x: Cin channels); mode 1: dx = conv^H(dy, w) (dy: Cout channels)
void conv_tc_run(cfloat* outp, const cfloat* inp, const cfloat* w, const ConvGeom& g, int mode)
{
    auto& c = ctx();
    const long nin = mode == 0 ? g.Cin : g.Cout, nout = mode == 0 ? g.Cout : g.Cin;
    const bool in_chl = mode == 0 ? g.in_chlast : g.out_chlast, in_rnd = mode == 0 ? g.in_tf32 : g.out_tf32;
    const bool out_chl = mode == 0 ? g.out_chlast : g.in_chlast;
    const long inner = g.X * g.Y;
    // operand staging only when the producer did not already deliver CHLAST + RN tf32
    float* act_tmp;
    const float* act = stage_operand(inp, nin, g, in_chl, in_rnd, &act_tmp);
    float* res = out_chl ? reinterpret_cast<float*>(outp) : nullptr;
    float* wpk;
    const long K = 9 * 2 * nin, N = 2 * nout;
    if (!out_chl)
        CUDA_CHECK(cudaMallocAsync(&res, sizeof(float) * 2 * nout * inner * g.B, c.stream));
    CUDA_CHECK(cudaMallocAsync(&wpk, sizeof(float) * K * N, c.stream));
    pdl_launch(k_pack_weights, int(std::min<long>(1024, (K * N + 255) / 256)), 256, 0, c.stream, wpk, w, int(g.KX), int(g.KY), int(g.Cin), int(g.Cout), mode);
    KERNEL_CHECK();
    {
        const double flops = 8.0 * double(g.X) * g.Y * g.B * g.Cin * g.Cout * 9;
        ProfScope prof(mode == 0 ? "conv_tc_fwd" : "conv_tc_bwd_data", flops);
        const int X = int(g.X), Y = int(g.Y), B = int(g.B);
        // epilogue channel statistics for a batch-norm consumer (forward, CHLAST output)
        double* st = (mode == 0 && out_chl) ? g.stats : nullptr;
        int* stb = st ? g.stats_blocks : nullptr;
        if (g.stats_blocks)
            *g.stats_blocks = 0;
        // batch-norm backward partials for the BN block consuming dx (bwd-data, CHLAST)
        BnEpi be{};
        int* beb = nullptr;
        if (g.bnb_blocks)
            *g.bnb_blocks = 0;
        if (mode == 1 && out_chl && g.bnb && g.bnb_part && g.bnb->C == 64 && g.bnb->npix == inner * g.B) {
            be = BnEpi{g.bnb->x, g.bnb->mu, g.bnb->istd, g.bnb->gamma, g.bnb->beta, g.bnb_part};
            beb = g.bnb_blocks;
        }
        if (nin == 64 && nout == 64)
            launch_tc<128, 128>(act, wpk, res, X, Y, B, st, stb, be, beb);
        else if (nin == 64 && nout == 32)
            launch_tc<128, 64>(act, wpk, res, X, Y, B);
        else if (nin == 32 && nout == 64)
            launch_tc<64, 128>(act, wpk, res, X, Y, B, st, stb, be, beb);
        else
            launch_tc<64, 64>(act, wpk, res, X, Y, B);
    }
    if (!out_chl) { // CHLAST -> CANON for a reference-layout consumer
        Dims d(max_rank, 1);
        d[0] = g.X;
        d[1] = g.Y;
        d[2] = nout;
        d[15] = g.B;
        DArray src = DArray::view(reinterpret_cast<cfloat*>(res), d);
        src.layout = Layout::CHLAST;
        DArray dst = DArray::view(outp, d);
        launch_layout_convert(src, dst);
        CUDA_CHECK(cudaFreeAsync(res, c.stream));
    }
    if (act_tmp)
        CUDA_CHECK(cudaFreeAsync(act_tmp, c.stream));
    CUDA_CHECK(cudaFreeAsync(wpk, c.stream));
}

} // namespace mdnn
