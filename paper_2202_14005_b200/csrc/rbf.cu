// Gaussian radial-basis activation of the Variational Network (RbfNode,
// ops.hpp:1308-1427):  phi(z)_k = sum_j w[f,j] exp(-(z_k - mu_j)^2 / (2 sigma^2))
// acting on Re z, with z viewed as [inner][filter][outer] and w as [nf, nw].
// Weight gradients reduce per (filter, basis) with fixed-order partials.
#include "kernels.h"
#include "profile.h"

#include <algorithm>
#include <cmath>
#include <type_traits>

namespace mdnn {

namespace {

bool g_rbf_window = true;
int g_rbf_cut = 55;  // windowed RBF: centres within cut / 10 sigma (+ 1 sigma margin) of z
int g_rbf_pair = 8; // k_rbf_map mode flag: paired-fp32 K = 9 window (0: rbf_visit_k)

constexpr int kT = 256;
constexpr int kMaxW = 64;

// Evenly spaced centres (g.win = 2K + 1 > 0): visits (j, e_j, d_j = z - mu_j) for the
// centres within K of the one nearest z, by the Gaussian recurrence
//   e_{j+1} = e_j U_j, U_{j+1} = U_j q ;  e_{j-1} = e_j D_j, D_{j-1} = D_j q,
//   U_j = exp(dmu (2 d_j - dmu) / 2s^2), D_j = exp(-dmu (2 d_j + dmu) / 2s^2),
// 3 MUFU per element instead of one per centre.  Rounding grows ~k^2 / 2 ulp over k
// steps, where the basis value is already below exp(-k^2 / 2) of the peak.
template<int KT, class F>
__device__ __forceinline__ void rbf_visit_k(float zk, const float* smu, const RbfGeom& g, float k2, F&& f)
{
    const int K = KT > 0 ? KT : (g.win >> 1);
    const float t = rintf((zk - g.mu0) * g.inv_dmu);
    const int jc = int(fminf(fmaxf(t, 0.f), float(g.nw - 1))); // NaN z: fmax(NaN, 0) = 0
    const float dc = zk - smu[jc];
    const float ec = exp2f(-(dc * dc) * k2);
    f(jc, ec, dc);
    const float dm = g.dmu;
    float U = exp2f(k2 * dm * (2.f * dc - dm)), D = exp2f(-k2 * dm * (2.f * dc + dm));
    float eu = ec, ed = ec;
    const bool inner = jc >= K && jc + K < g.nw; // no edge: every visited centre exists
#pragma unroll
    for (int k = 1; k <= (KT > 0 ? KT : 64); k++) {
        if (KT == 0 && k > K)
            break;
        eu *= U;
        U *= g.q;
        ed *= D;
        D *= g.q;
        if (inner || jc + k < g.nw)
            f(jc + k, eu, fmaf(-float(k), dm, dc));
        if (inner || jc - k >= 0)
            f(jc - k, ed, fmaf(float(k), dm, dc));
    }
}

template<class F>
__device__ __forceinline__ void rbf_visit(float zk, const float* smu, const RbfGeom& g, float k2, F&& f)
{
    if (g.win == 19) // VarNet: 31 centres at sigma = spacing, 8.5 sigma cut
        rbf_visit_k<9>(zk, smu, g, k2, f);
    else if (g.win == 13) // VarNet, 5.5 sigma cut (default)
        rbf_visit_k<6>(zk, smu, g, k2, f);
    else
        rbf_visit_k<0>(zk, smu, g, k2, f);
}

int grid_for(long n)
{
    long blocks = (n + kT - 1) / kT;
    return int(std::max(1L, std::min(blocks, long(ctx().sm_count) * 8)));
}

// exp(-(z - mu)^2 / (2 sigma^2)) as exp2(-(z - mu)^2 * k2), k2 = log2(e) / (2 sigma^2):
// no division, one MUFU.EX2 (the per-basis division + expf dominated the kernel)
__device__ __forceinline__ float gauss2(float z, float mu, float k2)
{
    const float d = z - mu;
    return exp2f(-(d * d) * k2);
}

// K-windowed phi(z) (mode 0) or sum_j w_j phi_j'(z) (mode 1) for evenly spaced
// centres, in paired fp32: the up / down recurrences of rbf_visit_k advance as one
// FMUL2 each step (bitwise the same basis values), their weighted sums as FFMA2 /
// FADD2 pairs.  Mode 1 uses sum_j w_j e_j (-d_j) = dm B - dc A with
// A = sum_j w_j e_j, B = sum_j w_j e_j (j - jc)  (d_j = dc - (j - jc) dm).
template<int K, bool INNER, int MODE>
__device__ __forceinline__ float rbf_map_win(const float* wf, int jc, float dc, float ec, float U, float D,
                                             const RbfGeom& g, float inv_s2)
{
    float2 st = make_float2(U, D), e2 = make_float2(ec, ec);
    const float2 q2 = make_float2(g.q, g.q);
    float2 a2 = make_float2(0.f, 0.f), b2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 1; k <= K; k++) {
        e2 = __fmul2_rn(e2, st);
        st = __fmul2_rn(st, q2);
        float2 es = e2, w2;
        if (INNER) {
            w2 = make_float2(wf[jc + k], wf[jc - k]);
        } else { // edge: centres outside [0, nw) contribute nothing (their recurrence may overflow)
            const bool up = jc + k < g.nw, dn = jc - k >= 0;
            es = make_float2(up ? e2.x : 0.f, dn ? e2.y : 0.f);
            w2 = make_float2(up ? wf[jc + k] : 0.f, dn ? wf[jc - k] : 0.f);
        }
        if constexpr (MODE == 0) {
            a2 = __ffma2_rn(w2, es, a2);
        } else {
            const float2 p2 = __fmul2_rn(w2, es);
            a2 = __fadd2_rn(a2, p2);
            b2 = __ffma2_rn(p2, make_float2(float(k), -float(k)), b2);
        }
    }
    const float a = fmaf(wf[jc], ec, a2.x + a2.y);
    if constexpr (MODE == 0)
        return a;
    return (g.dmu * (b2.x + b2.y) - dc * a) * inv_s2;
}

template<int K, int MODE>
__device__ __forceinline__ float rbf_map_w(float zk, const float* wf, const float* smu, const RbfGeom& g, float k2,
                                           float inv_s2)
{
    const float t = rintf((zk - g.mu0) * g.inv_dmu);
    const int jc = int(fminf(fmaxf(t, 0.f), float(g.nw - 1))); // NaN z: fmax(NaN, 0) = 0
    const float dc = zk - smu[jc];
    const float ec = exp2f(-(dc * dc) * k2);
    const float dm = g.dmu;
    const float U = exp2f(k2 * dm * (2.f * dc - dm)), D = exp2f(-k2 * dm * (2.f * dc + dm));
    if (jc >= K && jc + K < g.nw)
        return rbf_map_win<K, true, MODE>(wf, jc, dc, ec, U, D, g, inv_s2);
    return rbf_map_win<K, false, MODE>(wf, jc, dc, ec, U, D, g, inv_s2);
}

// mode 0: y = phi(z); 1: dz = Re(g) * phi'(z) (adjoint, also tangent with g = dx);
// 2: y = sum_j Re(dw) e_j (tangent wrt w).  The filter's weights and the centres
// are staged in shared memory; the element loop walks (inner, filter, outer)
// incrementally (no 64-bit division per element).
__global__ void k_rbf_map(cfloat* __restrict__ out, const cfloat* __restrict__ z, const cfloat* __restrict__ w,
                          const cfloat* __restrict__ gin, const float* __restrict__ mu, RbfGeom g, int mode)
{
    MDNN_PDL_ENTRY();
    const bool paired = mode & 8; // rbf_map_w (option rbf_pair) for the K = 9 window
    mode &= 7;
    __shared__ float smu[kMaxW];
    extern __shared__ float sw[]; // [nf][nw] real parts
    for (int j = threadIdx.x; j < g.nw; j += blockDim.x)
        smu[j] = mu[j];
    for (long e = threadIdx.x; e < g.nf * g.nw; e += blockDim.x) {
        const long f = e / g.nw, j = e % g.nw;
        sw[e] = w[f + j * g.nf].x;
    }
    __syncthreads();
    const long n = g.inner * g.nf * g.outer;
    const float s2 = g.sigma * g.sigma;
    const float inv_s2 = 1.f / s2;
    const float k2 = 1.4426950408889634f / (2.f * s2);
    const long stride = long(gridDim.x) * blockDim.x;
    long i = blockIdx.x * long(blockDim.x) + threadIdx.x;
    long f = (i / g.inner) % g.nf;
    long rem = i % g.inner;
    const long df = (stride / g.inner) % g.nf, drem = stride % g.inner;
    // advance (rem, f) by stride elements
    auto step = [&](long& r_, long& f_) {
        r_ += drem;
        f_ += df;
        if (r_ >= g.inner) {
            r_ -= g.inner;
            f_++;
        }
        if (f_ >= g.nf)
            f_ -= g.nf;
    };
    if (paired && (g.win == 19 || g.win == 13) && mode != 2) {
        // UE elements per thread per round, their loads issued together (one
        // element in flight per thread left the kernel latency-bound); the mode is
        // a template argument (a runtime mode predicated both forms' instructions)
        auto run = [&](auto MODE_) {
            constexpr int M = decltype(MODE_)::value;
            constexpr int UE = 4;
            for (; i < n; i += UE * stride) {
                float zk[UE], gk[UE];
                long fe[UE];
#pragma unroll
                for (int u = 0; u < UE; u++) {
                    const long ie = i + u * stride;
                    zk[u] = ie < n ? z[ie].x : 0.f;
                    gk[u] = (M == 1 && ie < n) ? gin[ie].x : 0.f;
                    fe[u] = f;
                    step(rem, f);
                }
#pragma unroll
                for (int u = 0; u < UE; u++) {
                    const long ie = i + u * stride;
                    if (ie < n) {
                        float acc = g.win == 13 ? rbf_map_w<6, M>(zk[u], sw + fe[u] * g.nw, smu, g, k2, inv_s2)
                                                : rbf_map_w<9, M>(zk[u], sw + fe[u] * g.nw, smu, g, k2, inv_s2);
                        if (M == 1)
                            acc *= gk[u];
                        out[ie] = float2{acc, 0.f};
                    }
                }
            }
        };
        if (mode == 0)
            run(std::integral_constant<int, 0>{});
        else
            run(std::integral_constant<int, 1>{});
        return;
    }
    for (; i < n; i += stride) {
        const float zk = z[i].x;
        const float* wf = sw + f * g.nw;
        float acc = 0.f;
        if (g.win) {
            if (mode == 1)
                rbf_visit(zk, smu, g, k2, [&](int j, float e, float d) { acc = fmaf(wf[j] * e, -d * inv_s2, acc); });
            else
                rbf_visit(zk, smu, g, k2, [&](int j, float e, float) { acc = fmaf(wf[j], e, acc); });
        } else {
            for (int j = 0; j < g.nw; j++) {
                const float e = gauss2(zk, smu[j], k2);
                if (mode == 1)
                    acc = fmaf(wf[j] * e, -(zk - smu[j]) * inv_s2, acc);
                else
                    acc = fmaf(wf[j], e, acc);
            }
        }
        if (mode == 1)
            acc *= gin[i].x;
        out[i] = float2{acc, 0.f};
        step(rem, f);
    }
}

// partial[(f * nw + j) * nchunk + chunk] = sum over the chunk of e_j(z) Re(g)
constexpr int kChunk = 8192;
// dz != nullptr: also the adjoint wrt z of the same elements (the basis values
// e_j are shared: one pass instead of k_rbf_map mode 1 + this kernel)
__global__ void k_rbf_wgrad(double* __restrict__ part, const cfloat* __restrict__ dy, const cfloat* __restrict__ z,
                            const float* __restrict__ mu, RbfGeom g, int nchunk, cfloat* __restrict__ dz,
                            const cfloat* __restrict__ w)
{
    MDNN_PDL_ENTRY();
    __shared__ float smu[kMaxW];
    __shared__ float swf[kMaxW];
    __shared__ double red[kMaxW][8];
    const long f = blockIdx.y;
    for (int j = threadIdx.x; j < g.nw; j += blockDim.x) {
        smu[j] = mu[j];
        swf[j] = dz ? w[f + j * g.nf].x : 0.f;
    }
    __syncthreads();
    const float inv_s2 = 1.f / (g.sigma * g.sigma);
    const long total = g.inner * g.outer;
    const long begin = long(blockIdx.x) * kChunk, end = min(total, begin + kChunk);
    // fp32 running sums per thread (kChunk / blockDim = 32 terms each), folded in
    // double.  Windowed centres: the sums live in shared memory [j][thread]
    // (the window start varies per element; bank = thread, conflict-free)
    extern __shared__ float sacc[];
    float acc[kMaxW];
    for (int j = 0; j < g.nw; j++) {
        acc[j] = 0.f;
        if (g.win)
            sacc[j * blockDim.x + threadIdx.x] = 0.f;
    }
    const float k2 = 1.4426950408889634f / (2.f * g.sigma * g.sigma);
    // element t = ii + inner * o walked incrementally (no 64-bit division per element)
    long ii = (begin + threadIdx.x) % g.inner, o = (begin + threadIdx.x) / g.inner;
    const long dii = long(blockDim.x) % g.inner, dob = long(blockDim.x) / g.inner;
    for (long t = begin + threadIdx.x; t < end; t += blockDim.x) {
        const long idx = ii + g.inner * (f + g.nf * o);
        ii += dii;
        o += dob;
        if (ii >= g.inner) {
            ii -= g.inner;
            o++;
        }
        const float zk = z[idx].x, gv = dy[idx].x;
        if (g.win) {
            float d = 0.f;
            float* ab = sacc + threadIdx.x;
            if (dz) {
                rbf_visit(zk, smu, g, k2, [&](int j, float e, float dj) {
                    ab[j * blockDim.x] = fmaf(e, gv, ab[j * blockDim.x]);
                    d = fmaf(swf[j] * e, -dj * inv_s2, d);
                });
                dz[idx] = float2{d * gv, 0.f};
            } else {
                rbf_visit(zk, smu, g, k2, [&](int j, float e, float) { ab[j * blockDim.x] = fmaf(e, gv, ab[j * blockDim.x]); });
            }
        } else if (dz) {
            float d = 0.f;
            for (int j = 0; j < g.nw; j++) {
                const float e = gauss2(zk, smu[j], k2);
                acc[j] = fmaf(e, gv, acc[j]);
                d = fmaf(swf[j] * e, -(zk - smu[j]) * inv_s2, d);
            }
            dz[idx] = float2{d * gv, 0.f};
        } else {
            for (int j = 0; j < g.nw; j++)
                acc[j] = fmaf(gauss2(zk, smu[j], k2), gv, acc[j]);
        }
    }
    if (g.win) {
        for (int j = 0; j < g.nw; j++)
            acc[j] = sacc[j * blockDim.x + threadIdx.x];
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = 0; j < g.nw; j++) {
        double v = double(acc[j]);
        for (int o2 = 16; o2 > 0; o2 >>= 1)
            v += __shfl_xor_sync(0xffffffffu, v, o2);
        if (lane == 0)
            red[j][warp] = v;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < g.nw; j += blockDim.x) {
        double s = 0;
        for (int w = 0; w < int(blockDim.x >> 5); w++)
            s += red[j][w];
        part[(f * g.nw + j) * nchunk + blockIdx.x] = s;
    }
}

// Windowed form with a compile-time half width K (VarNet: K = 9 of 31 centres):
// the per-thread sums live in shared memory rows padded by K on both sides
// ([nw + 2K][thread]), so the 2K + 1 read-modify-writes of an element need no
// bounds checks, and they are issued as independent loads, FMAs and stores
// (distinct rows) instead of one serialised load-add-store per centre.
template<int K, bool DZ>
__global__ void __launch_bounds__(kT) k_rbf_wgrad_w(double* __restrict__ part, const cfloat* __restrict__ dy,
                                                   const cfloat* __restrict__ z, const float* __restrict__ mu,
                                                   RbfGeom g, int nchunk, cfloat* __restrict__ dz,
                                                   const cfloat* __restrict__ w)
{
    MDNN_PDL_ENTRY();
    constexpr int NW2 = 2 * K + 1;
    __shared__ float smu[kMaxW];
    __shared__ float swf[kMaxW + 2 * K]; // weights, zero outside [0, nw)
    __shared__ double red[kMaxW][kT / 32];
    extern __shared__ float sacc[];    // [nw + 2K][kT]
    const long f = blockIdx.y;
    for (int j = threadIdx.x; j < g.nw; j += blockDim.x)
        smu[j] = mu[j];
    for (int j = threadIdx.x; j < g.nw + 2 * K; j += blockDim.x)
        swf[j] = (DZ && j >= K && j < g.nw + K) ? w[f + (j - K) * g.nf].x : 0.f;
    for (int j = 0; j < g.nw + 2 * K; j++)
        sacc[j * kT + threadIdx.x] = 0.f;
    __syncthreads();
    const float inv_s2 = 1.f / (g.sigma * g.sigma);
    const float k2 = 1.4426950408889634f / (2.f * g.sigma * g.sigma);
    const float dm = g.dmu;
    const long total = g.inner * g.outer;
    const long begin = long(blockIdx.x) * kChunk, end = min(total, begin + kChunk);
    long ii = (begin + threadIdx.x) % g.inner, o = (begin + threadIdx.x) / g.inner;
    const long dii = long(kT) % g.inner, dob = long(kT) / g.inner;
    // the next element's z and dy are loaded while this one is processed
    auto next_idx = [&]() {
        const long v = ii + g.inner * (f + g.nf * o);
        ii += dii;
        o += dob;
        if (ii >= g.inner) {
            ii -= g.inner;
            o++;
        }
        return v;
    };
    long idx_n = 0;
    float z_n = 0.f, g_n = 0.f;
    if (begin + threadIdx.x < end) {
        idx_n = next_idx();
        z_n = z[idx_n].x;
        g_n = dy[idx_n].x;
    }
    for (long t = begin + threadIdx.x; t < end; t += kT) {
        const long idx = idx_n;
        const float zk = z_n, gv = g_n;
        if (t + kT < end) {
            idx_n = next_idx();
            z_n = z[idx_n].x;
            g_n = dy[idx_n].x;
        }
        // basis values around the nearest centre jc (rbf_visit_k), position k <-> j = jc - K + k;
        // positions outside [0, nw) are zeroed (their recurrence values may overflow)
        const float tt = rintf((zk - g.mu0) * g.inv_dmu);
        const int jc = int(fminf(fmaxf(tt, 0.f), float(g.nw - 1)));
        const float dc = zk - smu[jc];
        float ew[NW2];
        ew[K] = exp2f(-(dc * dc) * k2);
        // up / down recurrences as one FMUL2 per step (bitwise rbf_visit_k's values)
        float2 st = make_float2(exp2f(k2 * dm * (2.f * dc - dm)), exp2f(-k2 * dm * (2.f * dc + dm)));
        float2 e2 = make_float2(ew[K], ew[K]);
        const float2 q2 = make_float2(g.q, g.q);
#pragma unroll
        for (int k = 1; k <= K; k++) {
            e2 = __fmul2_rn(e2, st);
            st = __fmul2_rn(st, q2);
            ew[K + k] = e2.x;
            ew[K - k] = e2.y;
        }
        if (jc < K || jc + K >= g.nw) {
#pragma unroll
            for (int k = 1; k <= K; k++) {
                ew[K + k] = jc + k < g.nw ? ew[K + k] : 0.f;
                ew[K - k] = jc - k >= 0 ? ew[K - k] : 0.f;
            }
        }
        float* ab = sacc + jc * kT + threadIdx.x; // padded row jc - K + k + K = jc + k
        float cur[NW2];
#pragma unroll
        for (int k = 0; k < NW2; k++)
            cur[k] = ab[k * kT];
        const float2 g2 = make_float2(gv, gv);
#pragma unroll
        for (int k = 0; k + 1 < NW2; k += 2) {
            const float2 r2 = __ffma2_rn(make_float2(ew[k], ew[k + 1]), g2, make_float2(cur[k], cur[k + 1]));
            ab[k * kT] = r2.x;
            ab[(k + 1) * kT] = r2.y;
        }
        ab[(NW2 - 1) * kT] = fmaf(ew[NW2 - 1], gv, cur[NW2 - 1]);
        if constexpr (DZ) {
            // sum_k w e_k (-(dc - (k - K) dm)) / s^2 = (dm B - dc A) / s^2,
            // (A, B) = sum_k w e_k (1, k - K) as one FFMA2 per centre
            float2 ab2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < NW2; k++) {
                const float pk = swf[jc + k] * ew[k];
                ab2 = __ffma2_rn(make_float2(pk, pk), make_float2(1.f, float(k - K)), ab2);
            }
            const float d = (dm * ab2.y - dc * ab2.x) * inv_s2;
            dz[idx] = float2{d * gv, 0.f};
        }
    }
    __syncthreads(); // (own column only, but keep the reduction below ordered)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = 0; j < g.nw; j++) {
        double v = double(sacc[(j + K) * kT + threadIdx.x]);
        for (int o2 = 16; o2 > 0; o2 >>= 1)
            v += __shfl_xor_sync(0xffffffffu, v, o2);
        if (lane == 0)
            red[j][warp] = v;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < g.nw; j += blockDim.x) {
        double s = 0;
        for (int ww = 0; ww < kT / 32; ww++)
            s += red[j][ww];
        part[(f * g.nw + j) * nchunk + blockIdx.x] = s;
    }
}

__global__ void k_rbf_wfinal(cfloat* dw, const double* part, RbfGeom g, int nchunk)
{
    MDNN_PDL_ENTRY();
    const long n = g.nf * g.nw;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        const long f = i / g.nw, j = i % g.nw;
        double s = 0;
        for (int c = 0; c < nchunk; c++)
            s += part[i * nchunk + c];
        dw[f + j * g.nf] = float2{float(s), 0.f};
    }
}

} // namespace

void rbf_window_enable(bool on) { g_rbf_window = on; }
void rbf_pair_enable(bool on) { g_rbf_pair = on ? 8 : 0; }
void rbf_cut_set(int tenths_sigma) { g_rbf_cut = tenths_sigma < 10 ? 10 : tenths_sigma; }

void rbf_set_window(RbfGeom& g, const std::vector<float>& mu)
{
    g.win = 0;
    const int n = int(mu.size());
    if (!g_rbf_window || n < 3)
        return;
    const double dmu = (double(mu[n - 1]) - mu[0]) / (n - 1);
    for (int j = 0; j < n; j++)
        if (std::fabs(double(mu[j]) - (mu[0] + j * dmu)) > 1e-5 * dmu)
            return; // not evenly spaced
    // skipped centres lie >= (K + 1/2) dmu - (rounding slack) from z, i.e. at
    // least cut + 1 sigma.  Default cut 5.5 (K = 6 at sigma = spacing): skipped
    // basis values are below exp(-21.1) ~ 2^-30 of the nearest one's, under the
    // fp32 rounding (2^-24) of every sum they would enter; option rbf_cut = 85
    // restores the 8.5-sigma window (K = 9, below 2^-52)
    const double cut = g_rbf_cut / 10.0;
    const int K = int(std::ceil(cut * g.sigma / dmu + 0.5 - 1e-6)); // sigma = spacing: K = 6 (9 at cut 8.5)
    const int win = 2 * K + 1;
    if (win >= n)
        return;
    g.win = win;
    g.mu0 = mu[0];
    g.inv_dmu = float(1.0 / dmu);
    g.dmu = float(dmu);
    g.q = float(std::exp(-dmu * dmu / (double(g.sigma) * g.sigma)));
}

void rbf_forward(cfloat* y, const cfloat* z, const cfloat* w, const float* mu, const RbfGeom& g)
{
    if (g.nw > kMaxW)
        throw ConfigError("rbf: more than 64 basis functions not supported on device");
    // algorithmic bytes: z in, y out (complex, 8 B each)
    ProfScope prof("rbf", 16.0 * double(g.inner) * g.nf * g.outer);
    pdl_launch(k_rbf_map, grid_for(g.inner * g.nf * g.outer), kT, sizeof(float) * g.nf * g.nw, ctx().stream, y, z, w, nullptr, mu, g, 0 | g_rbf_pair);
    KERNEL_CHECK();
}

void rbf_adjoint_z(cfloat* dz, const cfloat* dy, const cfloat* z, const cfloat* w, const float* mu, const RbfGeom& g)
{
    pdl_launch(k_rbf_map, grid_for(g.inner * g.nf * g.outer), kT, sizeof(float) * g.nf * g.nw, ctx().stream, dz, z, w, dy, mu, g, 1 | g_rbf_pair);
    KERNEL_CHECK();
}

void rbf_deriv_z(cfloat* dy, const cfloat* dz, const cfloat* z, const cfloat* w, const float* mu, const RbfGeom& g)
{
    pdl_launch(k_rbf_map, grid_for(g.inner * g.nf * g.outer), kT, sizeof(float) * g.nf * g.nw, ctx().stream, dy, z, w, dz, mu, g, 1 | g_rbf_pair);
    KERNEL_CHECK();
}

void rbf_deriv_w(cfloat* dy, const cfloat* dw, const cfloat* z, const float* mu, const RbfGeom& g)
{
    pdl_launch(k_rbf_map, grid_for(g.inner * g.nf * g.outer), kT, sizeof(float) * g.nf * g.nw, ctx().stream, dy, z, dw, nullptr, mu, g, 2);
    KERNEL_CHECK();
}

// dynamic shared memory of k_rbf_wgrad (windowed: per-thread sums [nw][kT])
size_t rbf_wgrad_smem(const RbfGeom& g)
{
    if (!g.win)
        return 0;
    const size_t bytes = sizeof(float) * kT * g.nw;
    static size_t granted = 48 * 1024;
    if (bytes > granted) {
        CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_rbf_wgrad),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
        granted = bytes;
    }
    return bytes;
}

// the K = 9 / K = 6 windowed weight-gradient kernels, or false when the geometry needs the generic one
template<int K>
void launch_wgrad_wk(double* part, const cfloat* dy, const cfloat* z, const float* mu, const RbfGeom& g, int nchunk,
                     cfloat* dz, const cfloat* w)
{
    const size_t bytes = sizeof(float) * kT * (g.nw + 2 * K);
    static size_t granted = 48 * 1024;
    if (bytes > granted) {
        CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_rbf_wgrad_w<K, true>),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
        CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_rbf_wgrad_w<K, false>),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
        granted = bytes;
    }
    pdl_launch(dz ? k_rbf_wgrad_w<K, true> : k_rbf_wgrad_w<K, false>, dim3(nchunk, unsigned(g.nf)), kT, bytes,
               ctx().stream, part, dy, z, mu, g, nchunk, dz, w);
    KERNEL_CHECK();
}

bool launch_wgrad_w9(double* part, const cfloat* dy, const cfloat* z, const float* mu, const RbfGeom& g, int nchunk,
                     cfloat* dz, const cfloat* w)
{
    if (g.win == 19)
        launch_wgrad_wk<9>(part, dy, z, mu, g, nchunk, dz, w);
    else if (g.win == 13)
        launch_wgrad_wk<6>(part, dy, z, mu, g, nchunk, dz, w);
    else
        return false;
    return true;
}

void rbf_adjoint_w(cfloat* dw, const cfloat* dy, const cfloat* z, const float* mu, const RbfGeom& g)
{
    auto& c = ctx();
    const long total = g.inner * g.outer;
    const int nchunk = int(std::max(1L, (total + kChunk - 1) / kChunk));
    double* part;
    CUDA_CHECK(cudaMallocAsync(&part, sizeof(double) * g.nf * g.nw * nchunk, c.stream));
    if (!launch_wgrad_w9(part, dy, z, mu, g, nchunk, nullptr, nullptr)) {
        pdl_launch(k_rbf_wgrad, dim3(nchunk, unsigned(g.nf)), kT, rbf_wgrad_smem(g), c.stream, part, dy, z, mu, g, nchunk, nullptr, nullptr);
        KERNEL_CHECK();
    }
    pdl_launch(k_rbf_wfinal, 4, 256, 0, c.stream, dw, part, g, nchunk);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(part, c.stream));
}

void rbf_adjoint_zw(cfloat* dz, cfloat* dw, const cfloat* dy, const cfloat* z, const cfloat* w, const float* mu,
                    const RbfGeom& g)
{
    auto& c = ctx();
    // algorithmic bytes: z and dy in, dz out (complex, 8 B each)
    ProfScope prof("rbf_adjoint", 24.0 * double(g.inner) * g.nf * g.outer);
    const long total = g.inner * g.outer;
    const int nchunk = int(std::max(1L, (total + kChunk - 1) / kChunk));
    double* part;
    CUDA_CHECK(cudaMallocAsync(&part, sizeof(double) * g.nf * g.nw * nchunk, c.stream));
    if (!launch_wgrad_w9(part, dy, z, mu, g, nchunk, dz, w)) {
        pdl_launch(k_rbf_wgrad, dim3(nchunk, unsigned(g.nf)), kT, rbf_wgrad_smem(g), c.stream, part, dy, z, mu, g, nchunk, dz, w);
        KERNEL_CHECK();
    }
    pdl_launch(k_rbf_wfinal, 4, 256, 0, c.stream, dw, part, g, nchunk);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(part, c.stream));
}

} // namespace mdnn
