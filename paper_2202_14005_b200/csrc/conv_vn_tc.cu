// VarNet 11 x 11 convolutions of real operands on the tensor cores (tcgen05,
// kind::tf32, fp32 accumulate).  The layers (recon.hpp:522-609 via
// nn.hpp:305-337) are K: 2 -> F (forward of K, adjoint of K^T) and
// K^T: F -> 2 (forward of K^T, adjoint of K), F = 24, on CANON complex arrays
// whose imaginary parts are known zero (DArray::known_real).
//
// Both kernels are row GEMMs whose accumulators live in per-output-row TMEM
// "slots": an UMMA over one input row r writes the contributions of r to every
// output row o = r - ky + 5 (ky = 0..10) of the current chunk at once -- the N
// dimension runs over (output row, ...) and the ky of each slot is folded into
// the B operand -- so the MMA's N is 24..256 instead of F, and the A operand
// (one input row) is read once per K-step for all 11 kernel rows.
//
//  * k_vn_expand (2 -> F), y[p, f] = sum_{k, c} x[p + k - 5, c] w[k, c, f]:
//    A = the im2col of one input row read through overlapping no-swizzle
//    core matrices: a row holds (c0, c1) per pixel (8 B), UMMA row m = output
//    pixel 2m (+ parity), K = (kx, c) = 24 (kx 11 = zero weight); rows are one
//    pixel pair (16 B) apart and the K core matrices overlap (lbo = 16 B).
//    Odd-start windows are 16-B aligned in a second copy of the row shifted by
//    one pixel, so a 256-pixel tile is two M = 128 MMAs (even / odd outputs).
//    N = (output row j, f) with slot width F8 = F rounded to 8; B rows are
//    ordered by descending ky so consecutive slots meet consecutive B rows.
//  * k_vn_reduce (F -> 2), dx[q, c] = sum_{k, f} dy[q - k + 5, f] w[k, c, f]:
//    projection + gather.  A = one dy row (M = 128 input pixels, K = F), N =
//    (output row j, kx, c) with 24-column slots: the MMA accumulates over ky
//    (rows) in TMEM; the epilogue gathers the kx shift across lanes through
//    shared memory (out[q] = sum_kx P[q - kx + 5][kx]); tiles overlap by 10
//    pixels so every output's 11 inputs are in one tile.
//
// Warp roles (both kernels): warp 9 TMA-loads raw input rows (complex, zero
// filled outside the image) into a ring, warps 0-3 convert them into the UMMA
// operand layout (real parts, TF32-RN) in a second ring, warp 4 allocates TMEM
// and issues the MMAs, warps 5-8 drain a finished chunk (double-buffered TMEM:
// the epilogue of chunk i overlaps the MMAs of chunk i + 1) and re-zero its
// slots.
#include <cudaTypedefs.h>

#include "kernels.h"
#include "profile.h"
#include "sm100.cuh"

#include <algorithm>
#include <string>

namespace mdnn {

namespace {

using namespace sm100;

constexpr int VK = 11, VP = 5;          // kernel extent, corner offset
constexpr int V_THREADS = 320;          // 4 converter + 1 MMA + 4 epilogue + 1 TMA warps
// k_vn_reduce: 4 more converter warps (10-13): its per-row conversion (F channels of 128
// pixels -> the K-major A operand) was the critical path
constexpr int VR_THREADS = V_THREADS + 128, VR_CONV = 256;
constexpr int V_SMEM_MIN = 120 * 1024;  // one CTA per SM: the kernels own all 512 TMEM columns

// ---- expand (2 -> F) --------------------------------------------------------------
constexpr int VE_RC = 5;                // output rows per chunk
constexpr int VE_TILE = 256;            // output pixels per tile (128 even + 128 odd)
constexpr int VE_ROWPX = 272;           // pixels per staged row copy (>= 256 + 12)
constexpr int VE_COPY = VE_ROWPX * 8;   // bytes per copy
constexpr int VE_NS = 8;                // operand ring slots (input rows)
constexpr int VE_NR = 4;                // raw ring slots
constexpr int VE_BOXPX = 96;            // pixels per TMA box (192 floats)
constexpr int VE_RAW = 3 * 2 * VE_BOXPX * 8; // 3 boxes x 2 channels x 96 complex: pixels x0 - 6 .. x0 + 281
// (TMA box starts must be 16-B aligned in the innermost dimension: even pixels)

struct VeSmem {
    int nb;         // B rows: 12 ky blocks of F8
    int wb_bytes;   // B operand
    int ring_off;
    int raw_off;
    int bar_off;
    int total;
    __host__ __device__ explicit VeSmem(int f8)
    {
        nb = 12 * f8;
        wb_bytes = 6 * nb * 16;
        ring_off = (wb_bytes + 1023) & ~1023;
        raw_off = ring_off + VE_NS * 2 * VE_COPY;
        bar_off = raw_off + VE_NR * VE_RAW;
        total = bar_off + 256 + 1024 > V_SMEM_MIN ? bar_off + 256 + 1024 : V_SMEM_MIN;
    }
};

__global__ void __launch_bounds__(V_THREADS, 1)
    k_vn_expand(const __grid_constant__ CUtensorMap tm_x, float2* __restrict__ y, const float2* __restrict__ w, int X,
                int Y, int B, int F, int F8, const unsigned* __restrict__ imag)
{
    MDNN_PDL_ENTRY();
    if (*imag) // complex operands: the CUDA-core complex kernel of this launch pair runs instead
        return;
    const VeSmem L(F8);
    extern __shared__ uint8_t smem_raw[];
    // aligned by an offset from the shared array (not an integer round trip), so
    // the compiler keeps the shared address space: LDS/STS, not generic LD/ST
    uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
    float* wb = reinterpret_cast<float*>(smem);
    uint8_t* ring = smem + L.ring_off;
    const float* raw = reinterpret_cast<const float*>(smem + L.raw_off);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* full = bars;                 // [VE_NS] 128 converter arrivals
    uint64_t* empty = bars + VE_NS;        // [VE_NS] MMA commit
    uint64_t* tfull = bars + 2 * VE_NS;    // [2] MMA commit
    uint64_t* tempty = tfull + 2;          // [2] 4 epilogue warps
    uint64_t* wb_full = tempty + 2;        // 128 converter arrivals
    uint64_t* rfull = wb_full + 1;         // [VE_NR] TMA transaction bytes
    uint64_t* rempty = rfull + VE_NR;      // [VE_NR] 128 converter arrivals
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rempty + VE_NR);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nxt = (X + VE_TILE - 1) / VE_TILE, nch = (Y + VE_RC - 1) / VE_RC;
    const long units = long(nxt) * nch * B;
    const long u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
    const int NB = L.nb;

    if (threadIdx.x == 0) {
        for (int i = 0; i < VE_NS; i++) {
            mbar_init(&full[i], 128);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        mbar_init(wb_full, 128);
        for (int i = 0; i < VE_NR; i++) {
            mbar_init(&rfull[i], 1);
            mbar_init(&rempty[i], 128);
        }
        fence_barrier_init();
    }
    if (warp == 4)
        tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 9) {
        // ---- raw input rows by TMA: 3 boxes of 96 pixels x 2 channels from pixel x0 - 6, zero filled outside
        if (lane == 0) {
            prefetch_tmap(&tm_x);
            uint32_t it = 0;
            for (long u = u0; u < u1; u++) {
                const int ch = int(u % nch), xt = int((u / nch) % nxt), b = int(u / (long(nch) * nxt));
                const int o0 = ch * VE_RC, x0 = xt * VE_TILE;
                for (int i = 0; i < VE_RC + 2 * VP; i++, it++) {
                    const uint32_t rs = it % VE_NR, ph = (it / VE_NR) & 1;
                    mbar_wait(&rempty[rs], ph ^ 1);
                    mbar_arrive_expect_tx(&rfull[rs], VE_RAW);
                    for (int j = 0; j < 3; j++)
                        tma_load_3d(smem + L.raw_off + rs * VE_RAW + j * (VE_RAW / 3), &tm_x, &rfull[rs],
                                    2 * (x0 - 6 + j * VE_BOXPX), o0 - VP + i, 2 * b);
                }
            }
        }
    } else if (warp < 4) {
        // ---- converters: B operand once, then raw rows -> two im2col copies
        const int t = threadIdx.x;
        for (int e = t; e < 6 * NB * 4; e += 128) {
            const int kk = e & 3, n = (e >> 2) % NB, kg = (e >> 2) / NB;
            const int k = kg * 4 + kk, kx = k >> 1, c = k & 1, kyr = n / F8, f = n - kyr * F8;
            float v = 0.f;
            if (kx < VK && kyr < VK && f < F)
                v = w[kx + VK * ((VK - 1 - kyr) + VK * (c + 2 * f))].x;
            wb[(kg * NB + n) * 4 + kk] = to_tf32(v);
        }
        fence_proxy_async_smem();
        mbar_arrive(wb_full);
        uint32_t it = 0;
        for (long u = u0; u < u1; u++) {
            for (int i = 0; i < VE_RC + 2 * VP; i++, it++) {
                const uint32_t st = it % VE_NS, ph = (it / VE_NS) & 1;
                const uint32_t rs = it % VE_NR, rph = (it / VE_NR) & 1;
                mbar_wait(&rfull[rs], rph);
                mbar_wait(&empty[st], ph ^ 1);
                const float* rw = raw + rs * (VE_RAW / 4);
                float2* P = reinterpret_cast<float2*>(ring + st * 2 * VE_COPY); // pixel x0 - 4 + k
                float2* Q = P + VE_ROWPX;                                       // pixel x0 - 5 + k
                for (int k = t + 1; k <= VE_ROWPX + 1; k += 128) {              // raw pixel x0 - 6 + k
                    const float* bx = rw + (k / VE_BOXPX) * (4 * VE_BOXPX) + 2 * (k % VE_BOXPX);
                    const float2 v{to_tf32(bx[0]), to_tf32(bx[2 * VE_BOXPX])};
                    if (k <= VE_ROWPX)
                        Q[k - 1] = v;
                    if (k >= 2)
                        P[k - 2] = v;
                }
                fence_proxy_async_smem();
                mbar_arrive(&full[st]);
                mbar_arrive(&rempty[rs]);
            }
        }
    } else if (warp == 4) {
        // ---- MMA issue (whole warp, elected lane issues)
        mbar_wait(wb_full, 0);
        tc_fence_after();
        const uint32_t wb_s = smem_u32(wb), ring_s = smem_u32(ring);
        uint32_t it = 0, cit = 0;
        for (long u = u0; u < u1; u++, cit++) {
            const uint32_t buf = cit & 1;
            mbar_wait(&tempty[buf], (cit >> 1) & 1); // zeroed by the epilogue
            tc_fence_after();
            for (int i = 0; i < VE_RC + 2 * VP; i++, it++) {
                const uint32_t st = it % VE_NS, ph = (it / VE_NS) & 1;
                mbar_wait(&full[st], ph);
                tc_fence_after();
                const int jlo = max(0, i - 2 * VP), jhi = min(VE_RC - 1, i);
                const int n = ((jhi - jlo + 1) * F8 + 15) & ~15;
                const uint32_t idesc = idesc_tf32(128, n);
                const int kyr0 = 2 * VP - i + jlo;
#pragma unroll
                for (int par = 0; par < 2; par++) {
                    // even outputs read the copy starting one pixel earlier (Q)
                    const uint32_t a0 = ring_s + st * 2 * VE_COPY + (par == 0 ? VE_COPY : 0);
                    const uint32_t d = tmem_base + buf * 256 + par * 128 + jlo * F8;
#pragma unroll
                    for (int s = 0; s < 3; s++) {
                        const uint64_t ad = umma_desc_kn(a0 + 32 * s, 16, 128);
                        const uint64_t bd = umma_desc_kn(wb_s + (2 * s * NB + kyr0 * F8) * 16, NB * 16, 128);
                        mma_tf32_warp(d, ad, bd, idesc, 1u);
                    }
                }
                mma_commit_warp(&empty[st]);
            }
            mma_commit_warp(&tfull[buf]);
        }
    } else {
        // ---- epilogue: slots -> y (both parities of a pixel pair in one 16-B store), re-zero
        const int lq = warp & 3, m = lq * 32 + lane;
        const uint32_t lrow = uint32_t(lq * 32) << 16;
        for (int c = 0; c < 512; c += 32)
            tmem_st32_zero(tmem_base + lrow + c);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&tempty[0]);
            mbar_arrive(&tempty[1]);
        }
        uint32_t cit = 0;
        for (long u = u0; u < u1; u++, cit++) {
            const int ch = int(u % nch), xt = int((u / nch) % nxt), b = int(u / (long(nch) * nxt));
            const int o0 = ch * VE_RC, xx = xt * VE_TILE + 2 * m;
            const uint32_t buf = cit & 1;
            mbar_wait(&tfull[buf], (cit >> 1) & 1);
            tc_fence_after();
            for (int j = 0; j < VE_RC; j++) {
                float v0[32], v1[32];
                tmem_ld32(tmem_base + lrow + buf * 256 + j * F8, v0);
                tmem_ld32(tmem_base + lrow + buf * 256 + 128 + j * F8, v1);
                tmem_ld_wait();
                const int o = o0 + j;
                if (o < Y && xx < X) {
                    float4* dst = reinterpret_cast<float4*>(y + xx + long(X) * (o + long(Y) * F * b));
                    const long fs = long(X) * Y / 2; // float4 stride between channels
#pragma unroll
                    for (int f = 0; f < 32; f++)
                        if (f < F)
                            dst[f * fs] = make_float4(v0[f], 0.f, v1[f], 0.f);
                }
            }
            for (int c = 0; c < 256; c += 32)
                tmem_st32_zero(tmem_base + lrow + buf * 256 + c);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0)
                mbar_arrive(&tempty[buf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

// ---- reduce (F -> 2) --------------------------------------------------------------
constexpr int VR_RC = 10;               // output rows per chunk
constexpr int VR_OUT = 116;             // output pixels per tile: input pixels x0 - 6 .. x0 + 121 (the
                                        // TMA box start must be 16-B aligned: an even pixel)
constexpr int VR_NS = 4;                // operand ring slots
constexpr int VR_NR = 3;                // raw ring slots (F x 128 complex each)
constexpr int VR_SLOT = 24;             // TMEM columns per output row: (kx 0..11, c)
constexpr int VR_EP = 25;               // gather buffer pitch (floats, odd: conflict-free)

struct VrSmem {
    int a_bytes, raw_bytes, wb_off, ring_off, raw_off, e_off, bar_off, total;
    __host__ __device__ VrSmem(int f, int f8)
    {
        a_bytes = (f8 / 4) * 128 * 16;
        raw_bytes = f * 128 * 8;
        wb_off = 0;
        ring_off = ((f8 / 4) * 288 * 16 + 1023) & ~1023;
        raw_off = ring_off + VR_NS * a_bytes;
        e_off = raw_off + VR_NR * raw_bytes;
        bar_off = e_off + 2 * 128 * VR_EP * 4;
        total = bar_off + 256 + 1024 > V_SMEM_MIN ? bar_off + 256 + 1024 : V_SMEM_MIN;
    }
};

__global__ void __launch_bounds__(VR_THREADS, 1)
    k_vn_reduce(const __grid_constant__ CUtensorMap tm_dy, float2* __restrict__ dx, const float2* __restrict__ w, int X,
                int Y, int B, int F, int F8, const unsigned* __restrict__ imag)
{
    MDNN_PDL_ENTRY();
    if (*imag)
        return;
    const VrSmem L(F, F8);
    constexpr int NB = 12 * VR_SLOT; // B rows: (ky 0..11, kx 0..11, c)
    extern __shared__ uint8_t smem_raw[];
    // aligned by an offset from the shared array (not an integer round trip), so
    // the compiler keeps the shared address space: LDS/STS, not generic LD/ST
    uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
    float* wb = reinterpret_cast<float*>(smem + L.wb_off);
    uint8_t* ring = smem + L.ring_off;
    const float* raw = reinterpret_cast<const float*>(smem + L.raw_off);
    float* E = reinterpret_cast<float*>(smem + L.e_off);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* full = bars;
    uint64_t* empty = bars + VR_NS;
    uint64_t* tfull = bars + 2 * VR_NS;
    uint64_t* tempty = tfull + 2;
    uint64_t* wb_full = tempty + 2;
    uint64_t* rfull = wb_full + 1;
    uint64_t* rempty = rfull + VR_NR;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rempty + VR_NR);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nxt = (X + VR_OUT - 1) / VR_OUT, nch = (Y + VR_RC - 1) / VR_RC;
    const long units = long(nxt) * nch * B;
    const long u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
    const int KG = F8 / 4;

    if (threadIdx.x == 0) {
        for (int i = 0; i < VR_NS; i++) {
            mbar_init(&full[i], VR_CONV);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        mbar_init(wb_full, VR_CONV);
        for (int i = 0; i < VR_NR; i++) {
            mbar_init(&rfull[i], 1);
            mbar_init(&rempty[i], VR_CONV);
        }
        fence_barrier_init();
    }
    if (warp == 4)
        tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 9) {
        // ---- raw dy rows by TMA: 128 complex x F channels, zero filled outside the image
        if (lane == 0) {
            prefetch_tmap(&tm_dy);
            uint32_t it = 0;
            for (long u = u0; u < u1; u++) {
                const int ch = int(u % nch), xt = int((u / nch) % nxt), b = int(u / (long(nch) * nxt));
                const int o0 = ch * VR_RC;
                for (int i = 0; i < VR_RC + 2 * VP; i++, it++) {
                    const uint32_t rs = it % VR_NR, ph = (it / VR_NR) & 1;
                    mbar_wait(&rempty[rs], ph ^ 1);
                    mbar_arrive_expect_tx(&rfull[rs], L.raw_bytes);
                    tma_load_3d(smem + L.raw_off + rs * L.raw_bytes, &tm_dy, &rfull[rs], 2 * (xt * VR_OUT - VP - 1),
                                o0 - VP + i, F * b);
                }
            }
        }
    } else if (warp < 4 || warp >= 10) {
        // converter ct: pixel t = ct % 128, channel groups [kg0, kg1) of half ct / 128
        const int ct = warp < 4 ? int(threadIdx.x) : int(threadIdx.x) - V_THREADS + 128;
        const int t = ct & 127, half = ct >> 7;
        const int kgh = (KG + 1) / 2, kg0 = half * kgh, kg1 = min(KG, kg0 + kgh);
        for (int e = ct; e < KG * NB * 4; e += VR_CONV) {
            const int kk = e & 3, n = (e >> 2) % NB, kg = (e >> 2) / NB;
            const int f = kg * 4 + kk, ky = n / VR_SLOT, rem = n - ky * VR_SLOT, kx = rem >> 1, c = rem & 1;
            float v = 0.f;
            if (kx < VK && ky < VK && f < F)
                v = w[kx + VK * (ky + VK * (c + 2 * f))].x;
            wb[(kg * NB + n) * 4 + kk] = to_tf32(v);
        }
        fence_proxy_async_smem();
        mbar_arrive(wb_full);
        uint32_t it = 0;
        for (long u = u0; u < u1; u++) {
            for (int i = 0; i < VR_RC + 2 * VP; i++, it++) {
                const uint32_t st = it % VR_NS, ph = (it / VR_NS) & 1;
                const uint32_t rs = it % VR_NR, rph = (it / VR_NR) & 1;
                mbar_wait(&rfull[rs], rph);
                mbar_wait(&empty[st], ph ^ 1);
                const float* rw = raw + rs * (L.raw_bytes / 4) + 2 * t; // real part of pixel t, channel 0
                float4* A = reinterpret_cast<float4*>(ring + st * L.a_bytes);
                for (int kg = kg0; kg < kg1; kg++) {
                    float q[4];
#pragma unroll
                    for (int kk = 0; kk < 4; kk++) {
                        const int f = kg * 4 + kk;
                        q[kk] = f < F ? to_tf32(rw[f * 256]) : 0.f;
                    }
                    A[kg * 128 + t] = make_float4(q[0], q[1], q[2], q[3]);
                }
                fence_proxy_async_smem();
                mbar_arrive(&full[st]);
                mbar_arrive(&rempty[rs]);
            }
        }
    } else if (warp == 4) {
        mbar_wait(wb_full, 0);
        tc_fence_after();
        const uint32_t wb_s = smem_u32(wb), ring_s = smem_u32(ring);
        uint32_t it = 0, cit = 0;
        for (long u = u0; u < u1; u++, cit++) {
            const uint32_t buf = cit & 1;
            mbar_wait(&tempty[buf], (cit >> 1) & 1);
            tc_fence_after();
            for (int i = 0; i < VR_RC + 2 * VP; i++, it++) {
                const uint32_t st = it % VR_NS, ph = (it / VR_NS) & 1;
                mbar_wait(&full[st], ph);
                tc_fence_after();
                const int jlo = max(0, i - 2 * VP), jhi = min(VR_RC - 1, i);
                const int n = ((jhi - jlo + 1) * VR_SLOT + 15) & ~15;
                const uint32_t idesc = idesc_tf32(128, n);
                const int ky0 = jlo - i + 2 * VP;
                const uint32_t d = tmem_base + buf * 256 + jlo * VR_SLOT;
                for (int s = 0; s < KG / 2; s++) {
                    const uint64_t ad = umma_desc_kn(ring_s + st * L.a_bytes + 2 * s * 2048, 2048, 128);
                    const uint64_t bd = umma_desc_kn(wb_s + (2 * s * NB + ky0 * VR_SLOT) * 16, NB * 16, 128);
                    mma_tf32_warp(d, ad, bd, idesc, 1u);
                }
                mma_commit_warp(&empty[st]);
            }
            mma_commit_warp(&tfull[buf]);
        }
    } else {
        // ---- epilogue: per output row, P[m][(kx, c)] -> E (smem) -> kx gather across pixels
        const int lq = warp & 3, m = lq * 32 + lane, et = threadIdx.x - 160; // warps 5-8: et 0..127
        const uint32_t lrow = uint32_t(lq * 32) << 16;
        for (int c = 0; c < 512; c += 32)
            tmem_st32_zero(tmem_base + lrow + c);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&tempty[0]);
            mbar_arrive(&tempty[1]);
        }
        uint32_t cit = 0;
        for (long u = u0; u < u1; u++, cit++) {
            const int ch = int(u % nch), xt = int((u / nch) % nxt), b = int(u / (long(nch) * nxt));
            const int o0 = ch * VR_RC, xq = xt * VR_OUT + et;
            const uint32_t buf = cit & 1;
            mbar_wait(&tfull[buf], (cit >> 1) & 1);
            tc_fence_after();
            for (int j = 0; j < VR_RC; j++) {
                float v[32];
                tmem_ld32(tmem_base + lrow + buf * 256 + j * VR_SLOT, v);
                tmem_ld_wait();
                float* e = E + (j & 1) * 128 * VR_EP;
#pragma unroll
                for (int k = 0; k < 2 * VK; k++)
                    e[m * VR_EP + k] = v[k];
                asm volatile("bar.sync 1, 128;" ::: "memory");
                const int o = o0 + j;
                if (et < VR_OUT && xq < X && o < Y) {
                    float a0 = 0.f, a1 = 0.f;
#pragma unroll
                    for (int kx = 0; kx < VK; kx++) {
                        const float* s = e + (et + 2 * VP + 1 - kx) * VR_EP + 2 * kx; // input pixel q - kx + 5
                        a0 += s[0];
                        a1 += s[1];
                    }
                    float2* dst = dx + xq + long(X) * (o + long(Y) * 2 * b);
                    dst[0] = float2{a0, 0.f};
                    dst[long(X) * Y] = float2{a1, 0.f};
                }
            }
            for (int c = 0; c < 256; c += 32)
                tmem_st32_zero(tmem_base + lrow + buf * 256 + c);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0)
                mbar_arrive(&tempty[buf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

// ---- weight gradient ---------------------------------------------------------------
// dw[kx, ky, c, f] = sum_p x[p + (kx - 5, ky - 5), c] dy[p, f] as a K = pixels
// GEMM per dy row o: D_g[m = (ky, s, c), f] for kx = 4 g + s (g = 0..2, three
// M = 128 accumulators, 32 TMEM columns each).  A is a window of the 11 x rows
// o - 5 .. o + 5 staged as [pixel quad][row slot][s][c][4 px] with the four
// one-pixel phases s pre-shifted: the kx = 4 g shift is a whole quad (+LBO)
// and consecutive row slots are consecutive 8-row groups (SBO = 128 B), so
// every MMA's M rows are the 11 kernel rows (+5 unused slots) of one g.  The
// window is a ring of 16 rows stored twice (slots j and j + 16) so the 16
// slots an MMA reads are always contiguous.  B = the dy row as [quad][f][4].
constexpr int VW_PC = 64;               // dy pixels per column chunk
constexpr int VW_PQ = 19;               // staged x pixel quads: p0 - 5 + 4 pq + s + i
constexpr int VW_SL = 16;               // window rows (ring)
constexpr int VW_XRAW = 2 * 160 * 4;    // raw x row: 2 planes x 80 complex from pixel p0 - 6
constexpr int VW_NXR = 16;              // raw x ring
constexpr int VW_NB = 3;                // B ring
constexpr int VW_BB = (VW_PC / 4) * 32 * 16; // B slot: 16 quads x 32 f rows x 16 B
constexpr int VW_MD = 8;                // dy-row completion ring

struct VwSmem {
    int xb_off, b_off, xr_off, dr_off, bar_off, total, dr_bytes;
    __host__ __device__ explicit VwSmem(int f)
    {
        dr_bytes = f * VW_PC * 8;
        xb_off = 0;
        b_off = VW_PQ * 2 * VW_SL * 128;
        xr_off = b_off + VW_NB * VW_BB;
        dr_off = xr_off + VW_NXR * VW_XRAW;
        bar_off = dr_off + 2 * dr_bytes;
        total = bar_off + 512 + 1024 > V_SMEM_MIN ? bar_off + 512 + 1024 : V_SMEM_MIN;
    }
};

__global__ void __launch_bounds__(VR_THREADS, 1)
    k_vn_wgrad(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_dy,
               float2* __restrict__ part, int X, int Y, int B, int F, const unsigned* __restrict__ imag)
{
    MDNN_PDL_ENTRY();
    if (*imag)
        return;
    const VwSmem L(F);
    extern __shared__ uint8_t smem_raw[];
    // aligned by an offset from the shared array (not an integer round trip), so
    // the compiler keeps the shared address space: LDS/STS, not generic LD/ST
    uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
    float* xb = reinterpret_cast<float*>(smem + L.xb_off);
    uint8_t* bring = smem + L.b_off;
    const float* xr = reinterpret_cast<const float*>(smem + L.xr_off);
    const float* dr = reinterpret_cast<const float*>(smem + L.dr_off);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* bfull = bars;                  // [VW_NB] 128 converter arrivals
    uint64_t* bempty = bfull + VW_NB;        // [VW_NB] MMA commit
    uint64_t* mdone = bempty + VW_NB;        // [VW_MD] MMA commit per dy row
    uint64_t* xfull = mdone + VW_MD;         // [VW_NXR] TMA
    uint64_t* xempty = xfull + VW_NXR;       // [VW_NXR] 128 converter arrivals
    uint64_t* dfull = xempty + VW_NXR;       // [2] TMA
    uint64_t* dempty = dfull + 2;            // [2] 128 converter arrivals
    uint64_t* tfull = dempty + 2;            // MMA commit after the last row
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nxc = (X + VW_PC - 1) / VW_PC;
    const long items = long(nxc) * Y * B;
    const long i0 = items * blockIdx.x / gridDim.x, i1 = items * (blockIdx.x + 1) / gridDim.x;

    if (threadIdx.x == 0) {
        for (int i = 0; i < VW_NB; i++) {
            mbar_init(&bfull[i], VR_CONV);
            mbar_init(&bempty[i], 1);
        }
        for (int i = 0; i < VW_MD; i++)
            mbar_init(&mdone[i], 1);
        for (int i = 0; i < VW_NXR; i++) {
            mbar_init(&xfull[i], 1);
            mbar_init(&xempty[i], VR_CONV);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&dfull[i], 1);
            mbar_init(&dempty[i], VR_CONV);
        }
        mbar_init(tfull, 1);
        fence_barrier_init();
    }
    if (warp == 4)
        tmem_alloc<128>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 9) {
        if (lane == 0) {
            prefetch_tmap(&tm_x);
            prefetch_tmap(&tm_dy);
            uint32_t xit = 0;
            auto load_x = [&](int r, int p0, int b) {
                const uint32_t s = xit % VW_NXR, ph = (xit / VW_NXR) & 1;
                mbar_wait(&xempty[s], ph ^ 1);
                mbar_arrive_expect_tx(&xfull[s], VW_XRAW);
                tma_load_3d(smem + L.xr_off + s * VW_XRAW, &tm_x, &xfull[s], 2 * (p0 - 6), r, 2 * b);
                xit++;
            };
            uint32_t it = 0;
            for (long w = i0; w < i1; w++, it++) {
                const int o = int(w % Y), xc = int((w / Y) % nxc), b = int(w / (long(Y) * nxc));
                const int p0 = xc * VW_PC;
                if (w == i0 || o == 0)
                    for (int r = o - VP; r < o + VP; r++)
                        load_x(r, p0, b);
                load_x(o + VP, p0, b);
                const uint32_t s = it & 1, ph = (it >> 1) & 1;
                mbar_wait(&dempty[s], ph ^ 1);
                mbar_arrive_expect_tx(&dfull[s], L.dr_bytes);
                tma_load_3d(smem + L.dr_off + s * L.dr_bytes, &tm_dy, &dfull[s], 2 * p0, o, F * b);
            }
        }
    } else if (warp < 4 || warp >= 10) {
        // ---- converters (8 warps: 0-3 and 10-13)
        const int t = warp < 4 ? int(threadIdx.x) : int(threadIdx.x) - V_THREADS + 128;
        for (int e = t; e < VW_NB * (VW_PC / 4) * (32 - F) * 4; e += VR_CONV) { // unused f rows stay zero
            const int per = (32 - F) * 4, sl = e / ((VW_PC / 4) * per), rem = e % ((VW_PC / 4) * per);
            const int pq = rem / per, fi = rem % per;
            reinterpret_cast<float*>(bring + sl * VW_BB)[(pq * 32 + F + fi / 4) * 4 + (fi & 3)] = 0.f;
        }
        uint32_t xit = 0;
        auto stage_x = [&](int r) { // raw x row -> window slot r mod 16 (both copies)
            const uint32_t s = xit % VW_NXR, ph = (xit / VW_NXR) & 1;
            mbar_wait(&xfull[s], ph);
            const float* raw = xr + s * (VW_XRAW / 4);
            const int j = r & (VW_SL - 1);
            for (int e = t; e < VW_PQ * 32; e += VR_CONV) {
                const int pq = e >> 5, q = e & 31, ss = q >> 3, c = (q >> 2) & 1, i = q & 3;
                const float v = to_tf32(raw[c * 160 + 2 * (1 + 4 * pq + ss + i)]);
                xb[(pq * 2 * VW_SL + j) * 32 + q] = v;
                xb[(pq * 2 * VW_SL + j + VW_SL) * 32 + q] = v;
            }
            mbar_arrive(&xempty[s]);
            xit++;
        };
        uint32_t it = 0, seg_it = 0;
        for (long w = i0; w < i1; w++, it++) {
            const int o = int(w % Y);
            if (w == i0 || o == 0) {
                if (it > 0) // window slots of the previous column: every MMA issued so far done
                    mbar_wait(&mdone[(it - 1) % VW_MD], ((it - 1) / VW_MD) & 1);
                seg_it = it;
                for (int r = o - VP; r < o + VP; r++)
                    stage_x(r);
            } else if (it >= seg_it + 6) {
                // slot of row o + 5 last held row o - 11, read by dy rows up to o - 6
                mbar_wait(&mdone[(it - 6) % VW_MD], ((it - 6) / VW_MD) & 1);
            }
            stage_x(o + VP);
            const uint32_t ds = it & 1, dph = (it >> 1) & 1;
            const uint32_t bs = it % VW_NB, bph = (it / VW_NB) & 1;
            mbar_wait(&dfull[ds], dph);
            mbar_wait(&bempty[bs], bph ^ 1);
            const float* raw = dr + ds * (L.dr_bytes / 4);
            float4* bo = reinterpret_cast<float4*>(bring + bs * VW_BB);
            // lanes = 8 channels x 4 pixel quads: the raw rows (pitch 2 VW_PC floats, a
            // multiple of the bank count) put every channel of one quad in the same bank,
            // so 8 channels per quad bound the read conflicts at 8-way (24-way with all
            // channels of a quad in one warp), and the B-slot writes stay conflict-free
            const int fgroups = (F + 7) >> 3;
            for (int e = t; e < (VW_PC / 4) * 8 * fgroups; e += VR_CONV) {
                const int ln = e & 31, k = e >> 5;
                const int f = 8 * (k % fgroups) + (ln & 7), pq = 4 * (k / fgroups) + (ln >> 3);
                if (f < F) {
                    const float* src = raw + f * 2 * VW_PC + 8 * pq;
                    bo[pq * 32 + f] = make_float4(to_tf32(src[0]), to_tf32(src[2]), to_tf32(src[4]), to_tf32(src[6]));
                }
            }
            mbar_arrive(&dempty[ds]);
            fence_proxy_async_smem();
            mbar_arrive(&bfull[bs]);
        }
    } else if (warp == 4) {
        constexpr uint32_t idesc = idesc_tf32(128, 32);
        const uint32_t xb_s = smem_u32(xb), b_s = smem_u32(bring);
        uint32_t it = 0;
        bool started = false;
        for (long w = i0; w < i1; w++, it++) {
            const int o = int(w % Y);
            const uint32_t bs = it % VW_NB, bph = (it / VW_NB) & 1;
            mbar_wait(&bfull[bs], bph);
            tc_fence_after();
            const int ws = (o - VP) & (VW_SL - 1);
#pragma unroll
            for (int g = 0; g < 3; g++)
#pragma unroll
                for (int ks = 0; ks < VW_PC / 8; ks++) {
                    const uint64_t ad = umma_desc_kn(xb_s + ((2 * ks + g) * 2 * VW_SL + ws) * 128, 2 * VW_SL * 128, 128);
                    const uint64_t bd = umma_desc_kn(b_s + bs * VW_BB + 2 * ks * 512, 512, 128);
                    mma_tf32_warp(tmem_base + g * 32, ad, bd, idesc, (started || ks > 0) ? 1u : 0u);
                }
            started = true;
            mma_commit_warp(&bempty[bs]);
            mma_commit_warp(&mdone[it % VW_MD]);
        }
        mma_commit_warp(tfull);
    } else if (warp >= 5) {
        const int lq = warp & 3, m = lq * 32 + lane;
        const int ky = m >> 3, s = (m >> 1) & 3, c = m & 1;
        const bool any = i1 > i0;
        if (any) {
            mbar_wait(tfull, 0);
            tc_fence_after();
        }
        const long n = 121L * 2 * F;
        float2* dst = part + size_t(blockIdx.x) * n;
        for (int g = 0; g < 3; g++) {
            float v[32];
            if (any) {
                tmem_ld32(tmem_base + (uint32_t(lq * 32) << 16) + g * 32, v);
                tmem_ld_wait();
            }
            const int kx = 4 * g + s;
            if (kx < VK && ky < VK)
#pragma unroll
                for (int f = 0; f < 32; f++)
                    if (f < F)
                        dst[kx + VK * (ky + VK * (c + 2 * f))] = float2{any ? v[f] : 0.f, 0.f};
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        tmem_dealloc<128>(tmem_base);
    }
}

// dw[i] = sum_s part[s][i] (fixed order, double accumulation: deterministic)
__global__ void __launch_bounds__(256) k_vn_fold(float2* __restrict__ dw, const float2* __restrict__ part, long n,
                                                 int nsplit, const unsigned* __restrict__ imag)
{
    MDNN_PDL_ENTRY();
    if (*imag)
        return;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        double a = 0;
        for (int s = 0; s < nsplit; s++)
            a += part[size_t(s) * n + i].x;
        dw[i] = float2{float(a), 0.f};
    }
}

bool g_vn_tc = true;

PFN_cuTensorMapEncodeTiled_v12000 vn_encode()
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

// complex CANON array [X][Y][planes] as fp32 [2X][Y][planes]; box (bx floats, 1 row, bp planes)
CUtensorMap vn_map(const cfloat* base, int X, int Y, long planes, int bx, int bp)
{
    CUtensorMap m;
    cuuint64_t dims[3] = {cuuint64_t(2 * X), cuuint64_t(Y), cuuint64_t(planes)};
    cuuint64_t strides[2] = {cuuint64_t(2 * X) * 4, cuuint64_t(2 * X) * Y * 4};
    cuuint32_t box[3] = {cuuint32_t(bx), 1, cuuint32_t(bp)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = vn_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<cfloat*>(base), dims, strides, box,
                             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(varnet row) failed: " + std::to_string(int(r)));
    return m;
}

// real flops of one 11 x 11 pass: 2 per real MAC
double vn_flops(const ConvGeom& g) { return 2.0 * double(g.X) * g.Y * g.B * g.Cin * g.Cout * g.KX * g.KY; }
// algorithmic HBM bytes (complex CANON arrays, 8 B per element): the thin side
// (2 channels) makes these layers memory-bound (~55 flop/B against a TF32 ridge
// of ~110), so the roofline row is bytes; the flops row is kept (tag suffix _tf)
double vn_bytes(const ConvGeom& g) { return 8.0 * double(g.X) * g.Y * g.B * (g.Cin + g.Cout); }

} // namespace

void conv_vn_tc_enable(bool on) { g_vn_tc = on; }

bool conv_vn_tc_supported(const ConvGeom& g)
{
    return g_vn_tc && g.KX == VK && g.KY == VK && g.Cin == 2 && g.Cout >= 1 && g.Cout <= 24 && !g.in_chlast
           && !g.out_chlast && !(g.X & 1) && g.X * g.Y * g.B * g.Cout < (1L << 31);
}

void conv_vn_tc_wgrad(cfloat* dw, const cfloat* x, const cfloat* dy, const ConvGeom& g, const unsigned* imag)
{
    auto& c = ctx();
    const int F = int(g.Cout), X = int(g.X), Y = int(g.Y), B = int(g.B);
    const VwSmem L(F);
    const long items = long((X + VW_PC - 1) / VW_PC) * Y * B;
    const int grid = int(std::min<long>(items, c.sm_count));
    const long n = 121L * 2 * F;
    CUDA_CHECK(cudaFuncSetAttribute(k_vn_wgrad, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total));
    const CUtensorMap tx = vn_map(x, X, Y, 2L * B, 160, 2);
    const CUtensorMap td = vn_map(dy, X, Y, long(F) * B, 2 * VW_PC, F);
    float2* part;
    CUDA_CHECK(cudaMallocAsync(&part, sizeof(float2) * n * grid, c.stream));
    {
        ProfScope prof("conv_vn_bwd_weight", vn_bytes(g));
        ProfScope prof_tf("conv_vn_bwd_weight_tf", vn_flops(g));
        pdl_launch(k_vn_wgrad, grid, VR_THREADS, L.total, c.stream, tx, td, part, X, Y, B, F, imag);
        KERNEL_CHECK();
    }
    pdl_launch(k_vn_fold, int((n + 255) / 256), 256, 0, c.stream, dw, part, n, grid, imag);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(part, c.stream));
}

void conv_vn_tc_run(cfloat* out, const cfloat* in, const cfloat* w, const ConvGeom& g, int mode, const unsigned* imag)
{
    auto& c = ctx();
    const int F = int(g.Cout), F8 = (F + 7) & ~7;
    const int X = int(g.X), Y = int(g.Y), B = int(g.B);
    if (mode == 0) {
        const VeSmem L(F8);
        const long units = long((X + VE_TILE - 1) / VE_TILE) * ((Y + VE_RC - 1) / VE_RC) * B;
        const int grid = int(std::min<long>(units, c.sm_count));
        CUDA_CHECK(cudaFuncSetAttribute(k_vn_expand, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total));
        const CUtensorMap tm = vn_map(in, X, Y, 2L * B, 2 * VE_BOXPX, 2);
        ProfScope prof("conv_vn_fwd", vn_bytes(g));
        ProfScope prof_tf("conv_vn_fwd_tf", vn_flops(g));
        pdl_launch(k_vn_expand, grid, V_THREADS, L.total, c.stream, tm, out, w, X, Y, B, F, F8, imag);
    } else {
        const VrSmem L(F, F8);
        const long units = long((X + VR_OUT - 1) / VR_OUT) * ((Y + VR_RC - 1) / VR_RC) * B;
        const int grid = int(std::min<long>(units, c.sm_count));
        CUDA_CHECK(cudaFuncSetAttribute(k_vn_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total));
        const CUtensorMap tm = vn_map(in, X, Y, long(F) * B, 256, F);
        ProfScope prof("conv_vn_bwd_data", vn_bytes(g));
        ProfScope prof_tf("conv_vn_bwd_data_tf", vn_flops(g));
        pdl_launch(k_vn_reduce, grid, VR_THREADS, L.total, c.stream, tm, out, w, X, Y, B, F, F8, imag);
    }
    KERNEL_CHECK();
}

} // namespace mdnn
