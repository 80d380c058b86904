// Complex 3x3 "same" convolution as a TF32 implicit GEMM on the 5th-generation
// tensor cores (tcgen05 + TMEM + TMA), for the MoDL 64->64 layers
// (conv_tenmul, nn.hpp:305-337; SURVEY §7 hard part 3).
//
// Real formulation: activations channels-last planar (CHLAST: per pixel
// [Re c0..c(C-1) | Im c0..c(C-1)]), one real GEMM per tap
//   out[p, (Re f | Im f)] += in[p + tap, (Re c | Im c)] * [[Re u, Im u], [-Im u, Re u]]
// with u = w[t,c,f] (forward) or conj(w[flip t, f, c]) (backward-data).
//
// CTA work unit ("super-tile"): 32 x 16 output pixels of one item = 4 UMMA
// M-tiles of 8 x 16 pixels, each with its own TMEM accumulator (4 x N
// columns).  Per 32-float K-chunk the CTA TMA-loads ONE zero-padded halo of
// 34 x 18 pixels (pitch 40, SWIZZLE_128B, 92 KB) and feeds all 9 taps from
// row-shifted shared-memory views of it (UMMA start address + base_offset), so
// activations cross L2->SMEM 1.4x instead of 9x; the packed weights stream
// per (tap, chunk) through a 2-stage TMA ring and are reused by the 4 M-tiles.
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

constexpr int TILE_X = 32, TILE_Y = 16;
constexpr int HALO_P = 40;             // halo pitch (pixels per line, multiple of 8, >= TILE_X + 2)
constexpr int HALO_L = TILE_Y + 2;     // halo lines
constexpr int HALO_BYTES = HALO_L * HALO_P * 128;
constexpr int NBSTAGE = 2;
constexpr int NTHREADS = 192;

template<int N>
struct TcSmem {
    static constexpr int B_BYTES = N * 128;
    static constexpr int HALO_OFF = 0;
    static constexpr int B_OFF = 2 * HALO_BYTES;
    static constexpr int BAR_OFF = B_OFF + NBSTAGE * B_BYTES;
    static constexpr int TOTAL = BAR_OFF + 256 + 1024; // + barriers + alignment slack
};

template<int CIN2, int N>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_conv_tc(const __grid_constant__ CUtensorMap tm_act, const __grid_constant__ CUtensorMap tm_w,
              float* __restrict__ out, int X, int Y, int B)
{
    static_assert(CIN2 % 32 == 0, "K per tap must be a multiple of 32 floats");
    static_assert(N % 16 == 0 && N >= 16 && 4 * N <= 512, "N must fit 4 accumulators in TMEM");
    constexpr int NCH = CIN2 / 32;
    constexpr int TMEM_COLS = 4 * N <= 32 ? 32 : (4 * N <= 64 ? 64 : (4 * N <= 128 ? 128 : (4 * N <= 256 ? 256 : 512)));
    using S = TcSmem<N>;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* halo = smem + S::HALO_OFF;
    uint8_t* bst = smem + S::B_OFF;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
    uint64_t* halo_full = bars;            // [2]
    uint64_t* halo_empty = bars + 2;       // [2]
    uint64_t* b_full = bars + 4;           // [NBSTAGE]
    uint64_t* b_empty = bars + 4 + NBSTAGE;
    uint64_t* tmem_full = bars + 4 + 2 * NBSTAGE;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int tiles_x = (X + TILE_X - 1) / TILE_X, tiles_y = (Y + TILE_Y - 1) / TILE_Y;
    const int ntiles = tiles_x * tiles_y * B;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tm_act);
        prefetch_tmap(&tm_w);
        for (int i = 0; i < 2; i++) {
            mbar_init(&halo_full[i], 1);
            mbar_init(&halo_empty[i], 1);
        }
        for (int i = 0; i < NBSTAGE; i++) {
            mbar_init(&b_full[i], 1);
            mbar_init(&b_empty[i], 1);
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, 128);
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
            // ---------------- TMA producer ----------------
            uint32_t hi = 0, bi = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int tx = tile % tiles_x, ty = (tile / tiles_x) % tiles_y, b = tile / (tiles_x * tiles_y);
                const int x0 = tx * TILE_X, y0 = ty * TILE_Y;
                for (int c = 0; c < NCH; c++, hi++) {
                    const uint32_t hb = hi & 1, hph = (hi >> 1) & 1;
                    mbar_wait(&halo_empty[hb], hph ^ 1);
                    mbar_arrive_expect_tx(&halo_full[hb], HALO_BYTES);
                    tma_load_4d(halo + hb * HALO_BYTES, &tm_act, &halo_full[hb], c * 32, x0 - 1, y0 - 1, b);
                    for (int t = 0; t < 9; t++, bi++) {
                        const uint32_t st = bi % NBSTAGE, bph = (bi / NBSTAGE) & 1;
                        mbar_wait(&b_empty[st], bph ^ 1);
                        mbar_arrive_expect_tx(&b_full[st], S::B_BYTES);
                        tma_load_2d(bst + st * S::B_BYTES, &tm_w, &b_full[st], t * CIN2 + c * 32, 0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer (single thread) ----------------
            constexpr uint32_t idesc = idesc_tf32(128, N);
            uint32_t hi = 0, bi = 0, ti = 0;
            const uint32_t halo_addr = smem_u32(halo), b_addr = smem_u32(bst);
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ti++) {
                mbar_wait(tmem_empty, (ti & 1) ^ 1);
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
                        for (int xt = 0; xt < 4; xt++) {
                            const uint32_t row0 = ky * HALO_P + xt * 8 + kx;
#pragma unroll
                            for (int k = 0; k < 4; k++) {
                                const uint64_t ad = umma_desc_sw128(hbase + row0 * 128 + k * 32, HALO_P * 128);
                                const uint64_t bd = umma_desc_sw128(bbase + k * 32, 1024);
                                mma_tf32(tmem_base + xt * N, ad, bd, idesc, (c | t | k) != 0);
                            }
                        }
                        mma_commit(&b_empty[st]);
                    }
                    mma_commit(&halo_empty[hb]);
                }
                mma_commit(tmem_full);
            }
        }
    } else {
        // ---------------- epilogue: TMEM -> registers -> global ----------------
        const int lg = warp & 3; // TMEM lane group this warp may access
        const int r = lg * 32 + lane;
        const int gy = r / 8, gx = r % 8;
        uint32_t ti = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ti++) {
            const int tx = tile % tiles_x, ty = (tile / tiles_x) % tiles_y, b = tile / (tiles_x * tiles_y);
            const int x0 = tx * TILE_X, y0 = ty * TILE_Y;
            mbar_wait(tmem_full, ti & 1);
            tc_fence_after();
            const int py = y0 + gy;
#pragma unroll 1
            for (int xt = 0; xt < 4; xt++) {
                const int px = x0 + xt * 8 + gx;
                const bool ok = px < X && py < Y;
                float* dst = out + ((long(b) * Y + py) * X + px) * N;
#pragma unroll 1
                for (int nc = 0; nc < N / 32; nc++) {
                    float v[32];
                    tmem_ld32(tmem_base + (uint32_t(lg * 32) << 16) + xt * N + nc * 32, v);
                    tmem_ld_wait();
                    if (ok) {
                        float4* d4 = reinterpret_cast<float4*>(dst + nc * 32);
#pragma unroll
                        for (int q = 0; q < 8; q++)
                            d4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(tmem_empty);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem_base);
    }
}

// packed real-block weights Bt[n][k], k = t*CIN2 + (in re | in im), n = (out re | out im);
// mode 0 (fwd): u = w[t, c=in, f=out]; mode 1 (bwd-data): u = conj(w[flip t, c=out, f=in])
__global__ void k_pack_weights(float* __restrict__ bt, const cfloat* __restrict__ w, int KX, int KY, int Cin,
                               int Cout, int mode)
{
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

CUtensorMap make_act_map(const float* base, int C2, int X, int Y, int B)
{
    CUtensorMap m;
    cuuint64_t dims[4] = {cuuint64_t(C2), cuuint64_t(X), cuuint64_t(Y), cuuint64_t(B)};
    cuuint64_t strides[3] = {cuuint64_t(C2) * 4, cuuint64_t(C2) * 4 * X, cuuint64_t(C2) * 4 * X * Y};
    cuuint32_t box[4] = {32, HALO_P, HALO_L, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(activation) failed: " + std::to_string(int(r)));
    return m;
}

CUtensorMap make_w_map(const float* base, int K, int N)
{
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(N)};
    cuuint64_t strides[1] = {cuuint64_t(K) * 4};
    cuuint32_t box[2] = {32, cuuint32_t(N)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(weights) failed: " + std::to_string(int(r)));
    return m;
}

template<int CIN2, int N>
void launch_tc(const float* act, const float* wpk, float* out, int X, int Y, int B)
{
    auto& c = ctx();
    CUtensorMap ta = make_act_map(act, CIN2, X, Y, B);
    CUtensorMap tw = make_w_map(wpk, 9 * CIN2, N);
    auto kern = k_conv_tc<CIN2, N>;
    const int smem = TcSmem<N>::TOTAL;
    static std::mutex mu;
    static std::map<int, bool> done;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!done[c.device]) {
            CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            done[c.device] = true;
        }
    }
    const int ntiles = ((X + TILE_X - 1) / TILE_X) * ((Y + TILE_Y - 1) / TILE_Y) * B;
    const int grid = std::min(ntiles, c.sm_count);
    kern<<<grid, NTHREADS, smem, c.stream>>>(ta, tw, out, X, Y, B);
    KERNEL_CHECK();
}

bool g_tc_enabled = true;

} // namespace

void conv_tc_enable(bool on) { g_tc_enabled = on; }

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
    const long inner = g.X * g.Y;
    // operand staging: CHLAST + RN tf32
    float* act;
    float* res;
    float* wpk;
    const long K = 9 * 2 * nin, N = 2 * nout;
    CUDA_CHECK(cudaMallocAsync(&act, sizeof(float) * 2 * nin * inner * g.B, c.stream));
    CUDA_CHECK(cudaMallocAsync(&res, sizeof(float) * 2 * nout * inner * g.B, c.stream));
    CUDA_CHECK(cudaMallocAsync(&wpk, sizeof(float) * K * N, c.stream));
    dim3 cb(32, 8);
    k_to_chlast_tf32<<<dim3(unsigned((inner + 31) / 32), unsigned((nin + 31) / 32), unsigned(g.B)), cb, 0,
                       c.stream>>>(act, inp, inner, nin, g.B);
    KERNEL_CHECK();
    k_pack_weights<<<int(std::min<long>(1024, (K * N + 255) / 256)), 256, 0, c.stream>>>(
        wpk, w, int(g.KX), int(g.KY), int(g.Cin), int(g.Cout), mode);
    KERNEL_CHECK();
    {
        const double flops = 8.0 * double(g.X) * g.Y * g.B * g.Cin * g.Cout * 9;
        ProfScope prof(mode == 0 ? "conv_tc_fwd" : "conv_tc_bwd_data", flops);
        const int X = int(g.X), Y = int(g.Y), B = int(g.B);
        if (nin == 64 && nout == 64)
            launch_tc<128, 128>(act, wpk, res, X, Y, B);
        else if (nin == 64 && nout == 32)
            launch_tc<128, 64>(act, wpk, res, X, Y, B);
        else if (nin == 32 && nout == 64)
            launch_tc<64, 128>(act, wpk, res, X, Y, B);
        else
            launch_tc<64, 64>(act, wpk, res, X, Y, B);
    }
    // CHLAST -> CANON
    DArray tmp_in, tmp_out;
    Dims d(max_rank, 1);
    d[0] = g.X;
    d[1] = g.Y;
    d[2] = nout;
    d[15] = g.B;
    DArray src = DArray::view(reinterpret_cast<cfloat*>(res), d);
    src.layout = Layout::CHLAST;
    DArray dst = DArray::view(outp, d);
    launch_layout_convert(src, dst);
    CUDA_CHECK(cudaFreeAsync(act, c.stream));
    CUDA_CHECK(cudaFreeAsync(res, c.stream));
    CUDA_CHECK(cudaFreeAsync(wpk, c.stream));
}

} // namespace mdnn
