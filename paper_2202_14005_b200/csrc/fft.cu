// Batched strided 1-D FFT along one dimension of a column-major array, and the
// multi-dimensional unitary DFT built from it (fft.hpp:180-226).
//
// A CTA transforms W lines at once.  Lines along a strided dim (d > 0) are
// batched over W consecutive inner indices so every global access is a
// coalesced row of W complex values; lines along dim 0 are batched over W
// consecutive outer indices (contiguous rows).  Data is staged once into
// shared memory, all radix stages run there (fft.cuh), and the result is
// scaled by 1/sqrt(n) on the way out: one HBM read + one write per element.
#include "fft.cuh"
#include "kernels.h"
#include "profile.h"

#include <cmath>
#include <map>
#include <mutex>

namespace mdnn {

namespace {

bool radix_ok(int r)
{
    switch (r) {
    case 2: case 3: case 4: case 5: case 7: case 8: case 11: case 13: case 16: case 17: case 19: case 23:
    case 29: case 31:
        return true;
    default:
        return false;
    }
}

std::vector<int> factor(long n)
{
    std::vector<int> r;
    long m = n;
    int e2 = 0;
    while (m % 2 == 0) {
        m /= 2;
        e2++;
    }
    while (e2 >= 4) {
        r.push_back(16);
        e2 -= 4;
    }
    if (e2 == 3)
        r.push_back(8);
    else if (e2 == 2)
        r.push_back(4);
    else if (e2 == 1)
        r.push_back(2);
    for (long p = 3; m > 1; p += 2) {
        while (m % p == 0) {
            r.push_back(int(p));
            m /= p;
        }
        if (p * p > m && m > 1) {
            r.push_back(int(m));
            m = 1;
        }
    }
    return r;
}

std::mutex g_plan_mu;
std::map<std::pair<int, int>, std::unique_ptr<fftd::Plan>> g_plans; // (device, n)

} // namespace

bool fft_supported(long n)
{
    if (n < 1 || n > 16384)
        return false;
    auto r = factor(n);
    if (int(r.size()) > fftd::kMaxStages)
        return false;
    for (int x : r)
        if (!radix_ok(x))
            return false;
    return true;
}

const fftd::Plan& fft_plan(int n)
{
    auto& c = ctx();
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto key = std::make_pair(c.device, n);
    auto it = g_plans.find(key);
    if (it != g_plans.end())
        return *it->second;
    if (!fft_supported(n))
        throw ConfigError("dft: length " + std::to_string(n) + " has a prime factor > 31 (unsupported on device)");
    auto p = std::make_unique<fftd::Plan>();
    p->n = n;
    auto rad = factor(n);
    p->nstages = int(rad.size());
    int ns = 1;
    std::vector<std::vector<float2>> tabs;
    for (int s = 0; s < p->nstages; s++) {
        int R = rad[s];
        p->radix[s] = R;
        p->ns[s] = ns;
        std::vector<float2> t(size_t(ns) * (R - 1));
        for (int k = 0; k < ns; k++)
            for (int q = 1; q < R; q++) {
                long m = (long(q) * k) % (long(ns) * R);
                double ang = -2.0 * M_PI * double(m) / double(long(ns) * R);
                t[size_t(k) * (R - 1) + q - 1] = float2{float(std::cos(ang)), float(std::sin(ang))};
            }
        float2* d = nullptr;
        if (!t.empty()) {
            CUDA_CHECK(cudaMalloc(&d, t.size() * sizeof(float2)));
            CUDA_CHECK(cudaMemcpy(d, t.data(), t.size() * sizeof(float2), cudaMemcpyHostToDevice));
        }
        p->tw[s] = d;
        ns *= R;
    }
    return *g_plans.emplace(key, std::move(p)).first->second;
}

namespace {

// mode 0: lines batched over inner index (sd > 1); mode 1: over outer index (sd == 1)
__global__ void __launch_bounds__(256) k_fft_lines(cfloat* __restrict__ out, const cfloat* __restrict__ in,
                                                   fftd::Plan plan, long sd, long outer, int W, int LD, int mode,
                                                   bool inverse, float scale)
{
    MDNN_PDL_ENTRY();
    extern __shared__ float2 smem[];
    const int n = plan.n;
    float2* a = smem;
    float2* b = smem + size_t(n) * LD;
    long i0, o0;
    if (mode == 0) {
        long nib = (sd + W - 1) / W;
        i0 = (blockIdx.x % nib) * W;
        o0 = blockIdx.x / nib;
    } else {
        i0 = 0;
        o0 = long(blockIdx.x) * W;
    }
    const float cj = inverse ? -1.f : 1.f;
    // load (conj for inverse: IDFT(x) = conj(DFT(conj x))); UL elements' loads in
    // flight per thread (one at a time left the kernel latency-bound: ncu long
    // scoreboard 47%, 2 CTAs per SM)
    auto locate = [&](int e, int& sidx, long& addr, bool& ok) {
        int w, k;
        if (mode == 0) {
            w = e % W;
            k = e / W;
            ok = i0 + w < sd;
            addr = o0 * sd * n + long(k) * sd + i0 + w;
        } else {
            k = e % n;
            w = e / n;
            ok = o0 + w < outer;
            addr = (o0 + w) * long(n) + k;
        }
        sidx = k * LD + w;
    };
    constexpr int UL = 8;
    for (int e0 = threadIdx.x; e0 < n * W; e0 += UL * blockDim.x) {
        float2 v[UL];
        int sidx[UL];
#pragma unroll
        for (int u = 0; u < UL; u++) {
            const int e = e0 + u * blockDim.x;
            long addr = 0;
            bool ok = false;
            sidx[u] = -1;
            if (e < n * W)
                locate(e, sidx[u], addr, ok);
            v[u] = ok ? in[addr] : float2{0.f, 0.f};
        }
#pragma unroll
        for (int u = 0; u < UL; u++)
            if (sidx[u] >= 0)
                a[sidx[u]] = float2{v[u].x, cj * v[u].y};
    }
    __syncthreads();
    float2* r = fftd::fft_smem(a, b, plan, LD);
    for (int e = threadIdx.x; e < n * W; e += blockDim.x) {
        int w, k;
        long addr;
        bool ok;
        if (mode == 0) {
            w = e % W;
            k = e / W;
            ok = i0 + w < sd;
            addr = o0 * sd * n + long(k) * sd + i0 + w;
        } else {
            k = e % n;
            w = e / n;
            ok = o0 + w < outer;
            addr = (o0 + w) * long(n) + k;
        }
        if (ok) {
            float2 v = r[k * LD + w];
            out[addr] = float2{scale * v.x, cj * scale * v.y};
        }
    }
}

} // namespace

void launch_fft_dim(cfloat* out, const cfloat* in, const Dims& dims, int dim, bool inverse)
{
    const long n = dims[dim];
    if (n == 1) {
        if (out != in)
            launch_copy(out, in, md_size(dims));
        return;
    }
    const auto& plan = fft_plan(int(n));
    long sd = 1, outer = 1;
    for (int d = 0; d < dim; d++)
        sd *= dims[d];
    for (size_t d = dim + 1; d < dims.size(); d++)
        outer *= dims[d];
    int mode = sd > 1 ? 0 : 1;
    int W = 16;
    while (W > 1 && long(n) * (W + 1) > 6144)
        W /= 2;
    if (mode == 0)
        W = int(std::min<long>(W, sd));
    int LD = mode == 1 && W > 1 ? W + 1 : W;
    size_t smem = size_t(2) * n * LD * sizeof(float2);
    auto& c = ctx();
    if (smem > c.smem_optin)
        throw ConfigError("dft: line length " + std::to_string(n) + " exceeds shared memory");
    allow_max_dyn_smem(reinterpret_cast<const void*>(k_fft_lines));
    long blocks = mode == 0 ? ((sd + W - 1) / W) * outer : (outer + W - 1) / W;
    float scale = float(1.0 / std::sqrt(double(n)));
    ProfScope prof("fft", 16.0 * double(n) * double(sd) * double(outer));
    pdl_launch(k_fft_lines, unsigned(blocks), 256, smem, c.stream, out, in, plan, sd, outer, W, LD, mode, inverse, scale);
    KERNEL_CHECK();
}

void fft_flags(cfloat* out, const cfloat* in, const Dims& dims, unsigned long flags, bool inverse)
{
    for (size_t d = dims.size(); d < 64; d++)
        if (flags & (1UL << d))
            throw ConfigError("dft: flag selects nonexistent dimension " + std::to_string(d));
    const cfloat* src = in;
    bool any = false;
    for (int d = 0; d < int(dims.size()); d++) {
        if (!(flags & (1UL << d)) || dims[d] == 1)
            continue;
        launch_fft_dim(out, src, dims, d, inverse); // in-place safe: CTA stages its lines in smem
        src = out;
        any = true;
    }
    if (!any && out != in)
        launch_copy(out, in, md_size(dims));
}

} // namespace mdnn
