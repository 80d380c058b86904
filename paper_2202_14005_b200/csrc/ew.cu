// Elementwise, broadcast, reduction and generic contraction kernels.
// Memory-bound helpers: grid-stride loops sized to a multiple of the SM count,
// float4 (two complex) vector accesses where the data is contiguous, and
// deterministic fixed-order two-stage reductions accumulated in double
// (mirrors md_zdot's double accumulation, mdarray.hpp:679-708).
#include "kernels.h"

#include <algorithm>
#include <numeric>

namespace mdnn {

namespace {

constexpr int kThreads = 256;

int grid_for(long n, int per_thread = 1)
{
    long blocks = (n + long(kThreads) * per_thread - 1) / (long(kThreads) * per_thread);
    long cap = long(ctx().sm_count) * 8;
    return int(std::max(1L, std::min(blocks, cap)));
}

struct Md3 {
    int rank;
    long dims[max_rank];
    long s0[max_rank], s1[max_rank], s2[max_rank];
};

Md3 make_md3(const Dims& d, const Dims& a, const Dims& b, const Dims& c)
{
    Md3 m{};
    m.rank = int(d.size());
    for (int i = 0; i < m.rank; i++) {
        m.dims[i] = d[i];
        m.s0[i] = a.empty() ? 0 : a[i];
        m.s1[i] = b.empty() ? 0 : b[i];
        m.s2[i] = c.empty() ? 0 : c[i];
    }
    return m;
}

__device__ __forceinline__ cfloat cmul(cfloat a, cfloat b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ cfloat cmulc(cfloat a, cfloat b) { return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y}; }

__global__ void k_strided_copy(Md3 m, long n, cfloat* dst, const cfloat* src)
{
    MDNN_PDL_ENTRY();
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        long r = i, od = 0, os = 0;
        for (int d = 0; d < m.rank; d++) {
            long q = r % m.dims[d];
            r /= m.dims[d];
            od += q * m.s0[d];
            os += q * m.s1[d];
        }
        dst[od] = src[os];
    }
}

__global__ void k_bcast_binary(Md3 m, long n, cfloat* out, const cfloat* a, const cfloat* b, int op)
{
    MDNN_PDL_ENTRY();
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        long r = i, oa = 0, ob = 0;
        for (int d = 0; d < m.rank; d++) {
            long q = r % m.dims[d];
            r /= m.dims[d];
            oa += q * m.s1[d];
            ob += q * m.s2[d];
        }
        cfloat x = a[oa], y = b[ob];
        out[i] = op == 0 ? cfloat{x.x + y.x, x.y + y.y} : (op == 1 ? cmul(x, y) : cmulc(x, y));
    }
}

// ---- vectorised elementwise kernels (two complex per float4) ----------------
template<class F>
__global__ void k_map1(cfloat* __restrict__ out, const cfloat* __restrict__ in, long n, F f)
{
    MDNN_PDL_ENTRY();
    long n2 = n / 2;
    const float4* in4 = reinterpret_cast<const float4*>(in);
    float4* out4 = reinterpret_cast<float4*>(out);
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n2; i += long(gridDim.x) * blockDim.x) {
        float4 v = in4[i];
        cfloat a = f(cfloat{v.x, v.y}), b = f(cfloat{v.z, v.w});
        out4[i] = make_float4(a.x, a.y, b.x, b.y);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0)
        out[n - 1] = f(in[n - 1]);
}

template<class F>
__global__ void k_map2(cfloat* __restrict__ out, const cfloat* __restrict__ a, const cfloat* __restrict__ b, long n,
                       F f)
{
    MDNN_PDL_ENTRY();
    long n2 = n / 2;
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* b4 = reinterpret_cast<const float4*>(b);
    float4* o4 = reinterpret_cast<float4*>(out);
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n2; i += long(gridDim.x) * blockDim.x) {
        float4 u = a4[i], v = b4[i];
        cfloat r0 = f(cfloat{u.x, u.y}, cfloat{v.x, v.y}), r1 = f(cfloat{u.z, u.w}, cfloat{v.z, v.w});
        o4[i] = make_float4(r0.x, r0.y, r1.x, r1.y);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0)
        out[n - 1] = f(a[n - 1], b[n - 1]);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template<class F>
void map1(cfloat* out, const cfloat* in, long n, F f)
{
    if (n <= 0)
        return;
    if (!aligned16(out) || !aligned16(in))
        throw Error("map1: misaligned buffers");
    pdl_launch(k_map1<F>, grid_for(n / 2 + 1), kThreads, 0, ctx().stream, out, in, n, f);
    KERNEL_CHECK();
}

template<class F>
void map2(cfloat* out, const cfloat* a, const cfloat* b, long n, F f)
{
    if (n <= 0)
        return;
    pdl_launch(k_map2<F>, grid_for(n / 2 + 1), kThreads, 0, ctx().stream, out, a, b, n, f);
    KERNEL_CHECK();
}

// ---- deterministic ISO reduction ------------------------------------------------
constexpr int kRedChunk = 16384; // elements of (inner x outer) per block

__device__ __forceinline__ double2 warp_sum2(double2 v)
{
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    return v;
}

__device__ double2 block_sum2(double2 v)
{
    __shared__ double2 red[32];
    v = warp_sum2(v);
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0)
        red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = (l < int(blockDim.x >> 5)) ? red[l] : double2{0, 0};
        v = warp_sum2(v);
    }
    __syncthreads();
    return v;
}

__global__ void k_iso_partial(double2* part, const cfloat* a, const cfloat* b, long inner, long nstat, long outer,
                              int mode, int nchunk, long chunk)
{
    MDNN_PDL_ENTRY();
    const long stat = blockIdx.y;
    const long total = inner * outer;
    const long begin = long(blockIdx.x) * chunk;
    const long end = min(total, begin + chunk);
    double2 acc{0, 0};
    // element j of this statistic sits at i + inner (stat + nstat o), (i, o) = (j mod inner, j / inner):
    // one division per thread, then walked incrementally (nstat == 1: idx = j)
    long j = begin + threadIdx.x;
    long i = j % inner, o = j / inner;
    const long di = long(blockDim.x) % inner, dO = long(blockDim.x) / inner;
    for (; j < end; j += blockDim.x) {
        const long idx = nstat == 1 ? j : i + inner * (stat + nstat * o);
        i += di;
        o += dO;
        if (i >= inner) {
            i -= inner;
            o++;
        }
        cfloat x = a[idx];
        if (mode == 0) {
            acc.x += x.x;
            acc.y += x.y;
        } else if (mode == 1) {
            cfloat y = b[idx];
            acc.x += double(x.x) * y.x + double(x.y) * y.y;
            acc.y += double(x.y) * y.x - double(x.x) * y.y;
        } else {
            acc.x += double(x.x) * x.x + double(x.y) * x.y;
        }
    }
    acc = block_sum2(acc);
    if (threadIdx.x == 0)
        part[stat * nchunk + blockIdx.x] = acc;
}

__global__ void k_iso_final(cfloat* out, double2* out_d, const double2* part, long nstat, int nchunk, float scale)
{
    MDNN_PDL_ENTRY();
    for (long s = blockIdx.x * long(blockDim.x) + threadIdx.x; s < nstat; s += long(gridDim.x) * blockDim.x) {
        double2 acc{0, 0};
        for (int c = 0; c < nchunk; c++) {
            acc.x += part[s * nchunk + c].x;
            acc.y += part[s * nchunk + c].y;
        }
        if (out)
            out[s] = cfloat{float(acc.x * scale), float(acc.y * scale)};
        if (out_d)
            out_d[s] = acc;
    }
}

// one block per statistic: strided chunk sums, then a fixed-order block tree
// (many chunks, few statistics: the serial loop above is latency-bound)
__global__ void k_iso_final_block(cfloat* out, double2* out_d, const double2* part, int nchunk, float scale)
{
    MDNN_PDL_ENTRY();
    const long s = blockIdx.x;
    double2 acc{0, 0};
    for (int c = threadIdx.x; c < nchunk; c += blockDim.x) {
        acc.x += part[s * nchunk + c].x;
        acc.y += part[s * nchunk + c].y;
    }
    acc = block_sum2(acc);
    if (threadIdx.x == 0) {
        if (out)
            out[s] = cfloat{float(acc.x * scale), float(acc.y * scale)};
        if (out_d)
            out_d[s] = acc;
    }
}

void iso_reduce_impl(cfloat* out, double2* out_d, const cfloat* a, const cfloat* b, long inner, long nstat,
                     long outer, int mode, float scale)
{
    auto& c = ctx();
    long total = inner * outer;
    // chunk: kRedChunk elements, smaller for large single statistics so that the
    // grid fills the GPU (about 4 blocks per SM); fixed for given sizes -> deterministic
    long chunk = kRedChunk;
    if (total * nstat > long(kRedChunk) * 4 * c.sm_count)
        chunk = kRedChunk;
    else
        chunk = std::max(2048L, (total * nstat + 4L * c.sm_count - 1) / (4L * c.sm_count) / std::max(1L, nstat));
    chunk = std::min<long>(chunk, kRedChunk);
    int nchunk = int(std::max(1L, (total + chunk - 1) / chunk));
    double2* part;
    CUDA_CHECK(cudaMallocAsync(&part, sizeof(double2) * nchunk * nstat, c.stream));
    dim3 grid(nchunk, unsigned(nstat));
    pdl_launch(k_iso_partial, grid, kThreads, 0, c.stream, part, a, b, inner, nstat, outer, mode, nchunk, chunk);
    KERNEL_CHECK();
    if (nchunk >= 64 && nstat <= 4096)
        pdl_launch(k_iso_final_block, unsigned(nstat), 256, 0, c.stream, out, out_d, part, nchunk, scale);
    else
        pdl_launch(k_iso_final, int(std::min(1024L, (nstat + 127) / 128)), 128, 0, c.stream, out, out_d, part, nstat, nchunk,
                                                                                     scale);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(part, c.stream));
}

// ---- generic TenMul ---------------------------------------------------------------
struct FmacPlan {
    int nout, nred;
    long odims[max_rank], oso[max_rank], os1[max_rank], os2[max_rank];
    long rdims[max_rank], rs1[max_rank], rs2[max_rank];
};

__global__ void k_fmac_gather(FmacPlan p, long nout_total, long nred_total, cfloat* out, const cfloat* a,
                              const cfloat* b, bool conj2)
{
    MDNN_PDL_ENTRY();
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < nout_total; i += long(gridDim.x) * blockDim.x) {
        long r = i, oo = 0, o1 = 0, o2 = 0;
        for (int d = 0; d < p.nout; d++) {
            long q = r % p.odims[d];
            r /= p.odims[d];
            oo += q * p.oso[d];
            o1 += q * p.os1[d];
            o2 += q * p.os2[d];
        }
        float accr = 0.f, acci = 0.f;
        for (long j = 0; j < nred_total; j++) {
            long rr = j, x1 = o1, x2 = o2;
            for (int d = 0; d < p.nred; d++) {
                long q = rr % p.rdims[d];
                rr /= p.rdims[d];
                x1 += q * p.rs1[d];
                x2 += q * p.rs2[d];
            }
            cfloat u = a[x1], v = b[x2];
            if (conj2)
                v.y = -v.y;
            accr += u.x * v.x - u.y * v.y;
            acci += u.x * v.y + u.y * v.x;
        }
        out[oo].x += accr;
        out[oo].y += acci;
    }
}

// layout conversion: CANON [inner][C][outer] <-> CHLAST per pixel [re C][im C]
__global__ void k_canon_to_chlast(float* __restrict__ out, const cfloat* __restrict__ in, long inner, long C,
                                  long outer)
{
    MDNN_PDL_ENTRY();
    __shared__ cfloat tile[32][33];
    long pix0 = long(blockIdx.x) * 32; // pixel within item
    long c0 = long(blockIdx.y) * 32;
    long o = blockIdx.z;
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
            dst[c] = v.x;
            dst[C + c] = v.y;
        }
    }
}

__global__ void k_chlast_to_canon(cfloat* __restrict__ out, const float* __restrict__ in, long inner, long C,
                                  long outer)
{
    MDNN_PDL_ENTRY();
    __shared__ cfloat tile[32][33];
    long pix0 = long(blockIdx.x) * 32;
    long c0 = long(blockIdx.y) * 32;
    long o = blockIdx.z;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        long p = pix0 + k, c = c0 + threadIdx.x;
        if (p < inner && c < C) {
            const float* src = in + (o * inner + p) * 2 * C;
            tile[threadIdx.x][k] = cfloat{src[c], src[C + c]};
        }
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        long c = c0 + k, p = pix0 + threadIdx.x;
        if (c < C && p < inner)
            out[(o * C + c) * inner + p] = tile[k][threadIdx.x];
    }
}

__global__ void k_check_finite(const float* a, long n, unsigned* flags)
{
    MDNN_PDL_ENTRY();
    bool bad = false;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        bad |= !isfinite(a[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0)
        atomicOr(flags, unsigned(ERRF_NONFINITE_GRAD));
}

__global__ void k_check_binary(const cfloat* a, long n, unsigned* flags)
{
    MDNN_PDL_ENTRY();
    bool bad = false;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        const cfloat v = a[i];
        bad |= v.y != 0.f || (v.x != 0.f && v.x != 1.f);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0)
        atomicOr(flags, unsigned(ERRF_PATTERN));
}

__global__ void k_split(cfloat* out, const cfloat* in, long inner, long outer)
{
    MDNN_PDL_ENTRY();
    long n = inner * outer;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        long p = i % inner, o = i / inner;
        cfloat v = in[i];
        out[p + inner * (2 * o)] = cfloat{v.x, 0.f};
        out[p + inner * (2 * o + 1)] = cfloat{v.y, 0.f};
    }
}

__global__ void k_join(cfloat* out, const cfloat* in, long inner, long outer)
{
    MDNN_PDL_ENTRY();
    long n = inner * outer;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        long p = i % inner, o = i / inner;
        out[i] = cfloat{in[p + inner * (2 * o)].x, in[p + inner * (2 * o + 1)].x};
    }
}

} // namespace

void launch_strided_copy(const Dims& dims, cfloat* dst, const Dims& sd, const cfloat* src, const Dims& ss)
{
    long n = md_size(dims);
    if (n == 0)
        return;
    auto m = make_md3(dims, sd, ss, {});
    pdl_launch(k_strided_copy, grid_for(n), kThreads, 0, ctx().stream, m, n, dst, src);
    KERNEL_CHECK();
}

void launch_layout_convert(const DArray& in, const DArray& out)
{
    const Dims& d = in.dims;
    long inner = d[0] * d[1], C = d[2], outer = 1;
    for (size_t i = 3; i < d.size(); i++)
        outer *= d[i];
    dim3 grid(unsigned((inner + 31) / 32), unsigned((C + 31) / 32), unsigned(outer));
    dim3 block(32, 8);
    if (in.layout == Layout::CANON && out.layout == Layout::CHLAST)
        pdl_launch(k_canon_to_chlast, grid, block, 0, ctx().stream, out.fdata(), in.data(), inner, C, outer);
    else if (in.layout == Layout::CHLAST && out.layout == Layout::CANON)
        pdl_launch(k_chlast_to_canon, grid, block, 0, ctx().stream, out.data(), in.fdata(), inner, C, outer);
    else
        throw Error("layout_convert: unsupported pair");
    KERNEL_CHECK();
}

void launch_add(cfloat* out, const cfloat* a, const cfloat* b, float s, long n)
{
    map2(out, a, b, n, [s] __device__(cfloat x, cfloat y) { return cfloat{x.x + s * y.x, x.y + s * y.y}; });
}

void launch_axpy(cfloat* y, cfloat al, const cfloat* x, long n)
{
    map2(y, y, x, n, [al] __device__(cfloat u, cfloat v) {
        return cfloat{u.x + (al.x * v.x - al.y * v.y), u.y + (al.x * v.y + al.y * v.x)};
    });
}

void launch_scale(cfloat* out, const cfloat* in, cfloat s, long n)
{
    map1(out, in, n, [s] __device__(cfloat v) { return cfloat{s.x * v.x - s.y * v.y, s.x * v.y + s.y * v.x}; });
}

namespace {
__global__ void k_scale_dev(cfloat* out, const cfloat* in, const cfloat* sp, bool cj, long n)
{
    MDNN_PDL_ENTRY();
    cfloat s = *sp;
    if (cj)
        s.y = -s.y;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        cfloat v = in[i];
        out[i] = cfloat{s.x * v.x - s.y * v.y, s.x * v.y + s.y * v.x};
    }
}
} // namespace

namespace {
__global__ void k_scale_dev_real(cfloat* out, const cfloat* in, const cfloat* sp, float factor, long n)
{
    MDNN_PDL_ENTRY();
    const float s = factor * sp[0].x;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        cfloat v = in[i];
        out[i] = cfloat{s * v.x, s * v.y};
    }
}
__global__ void k_real_scalar(cfloat* out, const cfloat* in, float factor) {
    MDNN_PDL_ENTRY(); out[0] = cfloat{factor * in[0].x, 0.f}; }
} // namespace

void launch_scale_dev_real(cfloat* out, const cfloat* in, const cfloat* s, float factor, long n)
{
    pdl_launch(k_scale_dev_real, grid_for(n), kThreads, 0, ctx().stream, out, in, s, factor, n);
    KERNEL_CHECK();
}

void launch_real_scalar(cfloat* out, const cfloat* in, float factor)
{
    pdl_launch(k_real_scalar, 1, 1, 0, ctx().stream, out, in, factor);
    KERNEL_CHECK();
}

void launch_scale_dev(cfloat* out, const cfloat* in, const cfloat* s, bool conj_s, long n)
{
    pdl_launch(k_scale_dev, grid_for(n), kThreads, 0, ctx().stream, out, in, s, conj_s, n);
    KERNEL_CHECK();
}

void launch_conj(cfloat* out, const cfloat* in, long n)
{
    map1(out, in, n, [] __device__(cfloat v) { return cfloat{v.x, -v.y}; });
}
void launch_real(cfloat* out, const cfloat* in, long n)
{
    map1(out, in, n, [] __device__(cfloat v) { return cfloat{v.x, 0.f}; });
}
void launch_neg(cfloat* out, const cfloat* in, long n)
{
    map1(out, in, n, [] __device__(cfloat v) { return cfloat{-v.x, -v.y}; });
}
void launch_crelu(cfloat* out, const cfloat* in, long n)
{
    map1(out, in, n, [] __device__(cfloat v) { return cfloat{v.x > 0.f ? v.x : 0.f, v.y > 0.f ? v.y : 0.f}; });
}
void launch_crelu_mask(cfloat* out, const cfloat* d, const cfloat* x, long n)
{
    map2(out, d, x, n, [] __device__(cfloat dv, cfloat xv) {
        return cfloat{xv.x > 0.f ? dv.x : 0.f, xv.y > 0.f ? dv.y : 0.f};
    });
}
void launch_exp_real(cfloat* out, const cfloat* in, long n)
{
    map1(out, in, n, [] __device__(cfloat v) { return cfloat{expf(v.x), 0.f}; });
}
void launch_mul_real_real(cfloat* out, const cfloat* y, const cfloat* d, long n)
{
    map2(out, y, d, n, [] __device__(cfloat a, cfloat b) { return cfloat{a.x * b.x, 0.f}; });
}

void launch_real_chan_split(cfloat* out, const cfloat* in, long inner, long outer)
{
    pdl_launch(k_split, grid_for(inner * outer), kThreads, 0, ctx().stream, out, in, inner, outer);
    KERNEL_CHECK();
}
void launch_real_chan_join(cfloat* out, const cfloat* in, long inner, long outer)
{
    pdl_launch(k_join, grid_for(inner * outer), kThreads, 0, ctx().stream, out, in, inner, outer);
    KERNEL_CHECK();
}

void launch_bcast_binary(const Dims& dims, cfloat* out, const cfloat* a, const Dims& sa, const cfloat* b,
                         const Dims& sb, int op)
{
    long n = md_size(dims);
    auto m = make_md3(dims, {}, sa, sb);
    pdl_launch(k_bcast_binary, grid_for(n), kThreads, 0, ctx().stream, m, n, out, a, b, op);
    KERNEL_CHECK();
}

void launch_iso_reduce(cfloat* out, const cfloat* a, const cfloat* b, long inner, long nstat, long outer, int mode,
                       float scale)
{
    iso_reduce_impl(out, nullptr, a, b, inner, nstat, outer, mode, scale);
}

void launch_zdot(double* out2, const cfloat* a, const cfloat* b, long n)
{
    iso_reduce_impl(nullptr, reinterpret_cast<double2*>(out2), a, b, n, 1, 1, a == b ? 2 : 1, 1.f);
}

double host_znorm(const cfloat* a, long n)
{
    double* d;
    auto& c = ctx();
    CUDA_CHECK(cudaMallocAsync(&d, 2 * sizeof(double), c.stream));
    iso_reduce_impl(nullptr, reinterpret_cast<double2*>(d), a, a, n, 1, 1, 2, 1.f);
    double h[2];
    CUDA_CHECK(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    CUDA_CHECK(cudaFreeAsync(d, c.stream));
    return std::sqrt(h[0]);
}

// Generic md_fmac2 (ops.hpp:79-111 via mdarray.hpp md_zfmac2 / md_zfmacc2).
// Output dims whose strides overlap (an adjoint through a strided window view,
// e.g. a convolution written as TenMul) cannot run as one gather: the greedy
// injective chain of output dims (ascending stride) stays in the kernel and
// every index of the remaining "serial" dims is its own launch, in a fixed
// order -- no atomics, bitwise run-to-run deterministic (SURVEY §7 hard part 5,
// reference guarantee mdarray.hpp:322-342).
void launch_fmac_generic(const Dims& iter, cfloat* out, const Dims& so, const cfloat* in1, const Dims& s1,
                         const cfloat* in2, const Dims& s2, bool conj2)
{
    struct Dim {
        long n, so, s1, s2;
    };
    std::vector<Dim> odim, rdim;
    for (size_t d = 0; d < iter.size(); d++) {
        if (iter[d] == 1)
            continue;
        (so[d] != 0 ? odim : rdim).push_back({iter[d], so[d], s1[d], s2[d]});
    }
    std::stable_sort(odim.begin(), odim.end(), [](const Dim& a, const Dim& b) { return std::labs(a.so) < std::labs(b.so); });
    std::vector<Dim> inj, serial;
    long span = 1;
    for (const Dim& d : odim) {
        if (std::labs(d.so) >= span) {
            inj.push_back(d);
            span = std::labs(d.so) * d.n;
        } else {
            serial.push_back(d);
        }
    }
    FmacPlan p{};
    for (const Dim& d : inj) {
        p.odims[p.nout] = d.n;
        p.oso[p.nout] = d.so;
        p.os1[p.nout] = d.s1;
        p.os2[p.nout] = d.s2;
        p.nout++;
    }
    for (const Dim& d : rdim) {
        p.rdims[p.nred] = d.n;
        p.rs1[p.nred] = d.s1;
        p.rs2[p.nred] = d.s2;
        p.nred++;
    }
    long nout = 1, nred = 1, nser = 1;
    for (int i = 0; i < p.nout; i++)
        nout *= p.odims[i];
    for (int i = 0; i < p.nred; i++)
        nred *= p.rdims[i];
    for (const Dim& d : serial)
        nser *= d.n;
    for (long k = 0; k < nser; k++) {
        long r = k, oo = 0, o1 = 0, o2 = 0;
        for (const Dim& d : serial) {
            const long q = r % d.n;
            r /= d.n;
            oo += q * d.so;
            o1 += q * d.s1;
            o2 += q * d.s2;
        }
        pdl_launch(k_fmac_gather, grid_for(nout), kThreads, 0, ctx().stream, p, nout, nred, out + oo, in1 + o1, in2 + o2,
                                                                     conj2);
        KERNEL_CHECK();
    }
}

void launch_copy(cfloat* dst, const cfloat* src, long n)
{
    CUDA_CHECK(cudaMemcpyAsync(dst, src, n * sizeof(cfloat), cudaMemcpyDeviceToDevice, ctx().stream));
}

void launch_check_finite(const cfloat* a, long n)
{
    pdl_launch(k_check_finite, grid_for(2 * n), kThreads, 0, ctx().stream, reinterpret_cast<const float*>(a), 2 * n,
                                                                   ctx().d_errflags);
    KERNEL_CHECK();
}

void launch_check_binary(const cfloat* a, long n)
{
    pdl_launch(k_check_binary, int(std::min<long>(grid_for(n), 64)), kThreads, 0, ctx().stream, a, n, ctx().d_errflags);
    KERNEL_CHECK();
}

} // namespace mdnn
