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
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
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

} // namespace

void conv_thin_tc_enable(bool on) { g_thin_tc = on; }

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
    k_pack_thin_tc<<<(TP_N * TP_K + 255) / 256, 256, 0, c.stream>>>(ut, U, F, KK);
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
    k_thin_proj<<<int(std::min<long>(ntiles, c.sm_count)), TP_THREADS, TpSmem::TOTAL, c.stream>>>(ta, tb, z, npix);
    KERNEL_CHECK();
    k_thin_gather<<<int(std::min<long>((npix + 255) / 256, 8L * c.sm_count)), 256, 0, c.stream>>>(
        out, z, int(X), int(Y), npix, ox, oy);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(ut, c.stream));
    CUDA_CHECK(cudaFreeAsync(z, c.stream));
    return true;
}

} // namespace mdnn
