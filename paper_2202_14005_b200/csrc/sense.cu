// SENSE operator A = P F C, its adjoint, the normal operator A^H A (+ lambda)
// and the data-consistency conjugate-gradient solve.
//
// Reference: build_sense (recon.hpp:82-123), sense_*_fragment
// (recon.hpp:345-418), modl_normal_plus_lambda (recon.hpp:807-820), cg_solve
// (recon.hpp:143-181).
//
// Network patterns are x-invariant ([1,Y], recon.hpp:24-29), so
//   F^H P F = I_x (x) (F_y^H P_y F_y)
// and the x-transform pair cancels exactly.  The fused kernel below therefore
// runs, per CTA, a strip of W image columns x all Y rows of one batch item:
// it reads x once, streams every coil map once, does coil-multiply -> y-FFT ->
// mask -> inverse y-FFT -> conj-coil accumulate entirely in shared memory,
// and writes A^H A x + lambda x once: 8*(C*M + 2M) bytes per pixel, the
// algorithmic minimum.  The CG variant additionally fuses
// p = r + beta p into the load and emits per-CTA partials of <p, Ap>.
#include "fft.cuh"
#include "kernels.h"
#include "profile.h"
#include "sm100.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cmath>

namespace mdnn {

using fftd::cconj;
using fftd::cmul;
using fftd::cmulc;

namespace {

constexpr int kT = 256;

int grid_for(long n)
{
    long blocks = (n + kT - 1) / kT;
    return int(std::max(1L, std::min(blocks, long(ctx().sm_count) * 8)));
}

struct PatStr {
    long sx, sy, sc, sb;
};

__global__ void k_coil_mul(cfloat* __restrict__ u, const cfloat* __restrict__ x, const cfloat* __restrict__ coils,
                           long XY, long C, long M, long B)
{
    MDNN_PDL_ENTRY();
    const long n = XY * C * B;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        long p = i % XY, c = (i / XY) % C, b = i / (XY * C);
        float2 acc{0.f, 0.f};
        for (long m = 0; m < M; m++) {
            float2 cv = coils[p + XY * (c + C * (m + M * b))];
            float2 xv = x[p + XY * (m + M * b)];
            acc.x += cv.x * xv.x - cv.y * xv.y;
            acc.y += cv.x * xv.y + cv.y * xv.x;
        }
        u[i] = acc;
    }
}

__global__ void k_coil_adj(cfloat* __restrict__ x, const cfloat* __restrict__ u, const cfloat* __restrict__ coils,
                           long XY, long C, long M, long B)
{
    MDNN_PDL_ENTRY();
    const long n = XY * M * B;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        long p = i % XY, m = (i / XY) % M, b = i / (XY * M);
        float2 acc{0.f, 0.f};
        for (long c = 0; c < C; c++) {
            float2 cv = coils[p + XY * (c + C * (m + M * b))];
            float2 uv = u[p + XY * (c + C * b)];
            acc.x += cv.x * uv.x + cv.y * uv.y;
            acc.y += cv.x * uv.y - cv.y * uv.x;
        }
        x[i] = acc;
    }
}

__global__ void k_pattern_mul(cfloat* __restrict__ out, const cfloat* __restrict__ u, const cfloat* __restrict__ pat,
                              long X, long Y, long C, long B, PatStr ps)
{
    MDNN_PDL_ENTRY();
    const long n = X * Y * C * B;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        long x = i % X, y = (i / X) % Y, c = (i / (X * Y)) % C, b = i / (X * Y * C);
        float2 pv = pat[x * ps.sx + y * ps.sy + c * ps.sc + b * ps.sb];
        float2 v = u[i];
        out[i] = float2{v.x * pv.x - v.y * pv.y, v.x * pv.y + v.y * pv.x};
    }
}

PatStr pat_strides(const SenseGeom& g)
{
    // pattern dims: [PX, PY, 1, PC, 1, ..., PB] with each 1 or full
    PatStr s{};
    s.sx = g.pat_x > 1 ? 1 : 0;
    s.sy = g.pat_y > 1 ? g.pat_x : 0;
    s.sc = g.pat_c > 1 ? g.pat_x * g.pat_y : 0;
    s.sb = g.pat_b > 1 ? g.pat_x * g.pat_y * g.pat_c : 0;
    return s;
}

// ---------------------------------------------------------------------------
// CG device state (recon.hpp:143-181).  Per-iteration scalars are stored by
// iteration index so that kernel k of iteration `it` only reads values written
// by earlier kernels: no intra-kernel races, no host synchronisation.
// ---------------------------------------------------------------------------
struct CgDev {
    double bnorm;
    double tol;
    int max_iter;
    int done_at;      // first iteration index that did not run (INT_MAX while running)
    int n_pap;        // partial count written by the S kernel
    int n_rr;         // partial count written by the update kernel
    double2* part_pap;
    double2* part_rr;
    double pap_sum;   // <p, Ap> of the current iteration, folded by the producer's last CTA
    double rr_sum;    // <r, r> after the latest update
    unsigned cnt_pap; // CTA arrival counters (reset by the folding CTA)
    unsigned cnt_rr;
    unsigned ws_bar;  // grid barrier of the fused CG update (k_normal_ws): G arrivals per iteration
    float* rs;        // [max_iter + 1]
    float* alpha;     // [max_iter]
    float* beta;      // [max_iter]
};


// Prologue of iteration `it` of the S kernel, run by thread 0 of every CTA
// (all CTAs compute bit-identical values).  Returns beta (or -1 to skip).
__device__ float cg_prologue(CgDev* st, int it, unsigned* errflags)
{
    if (st->done_at <= it)
        return -1.f;
    float rs_it;
    float beta = 0.f;
    if (it == 0) {
        rs_it = st->rs[0];
    } else {
        double sum = st->rr_sum;
        rs_it = float(sum);
        if (!isfinite(rs_it)) {
            if (blockIdx.x == 0) {
                atomicOr(errflags, unsigned(ERRF_CG_NONFINITE));
                st->done_at = it;
            }
            return -1.f;
        }
        beta = float(double(rs_it) / double(st->rs[it - 1]));
        if (blockIdx.x == 0) {
            st->rs[it] = rs_it;
            st->beta[it - 1] = beta;
        }
    }
    if (sqrt(double(rs_it)) <= st->tol * st->bnorm) {
        if (blockIdx.x == 0)
            st->done_at = it;
        return -1.f;
    }
    return beta;
}

__device__ float cg_alpha_sum(CgDev* st, int it, double s, unsigned* errflags)
{
    if (st->done_at <= it)
        return 0.f;
    float pap = float(s);
    if (!isfinite(pap) || pap <= 0.f) {
        if (blockIdx.x == 0) {
            atomicOr(errflags, unsigned(ERRF_CG_BREAKDOWN));
            st->done_at = it;
        }
        return 0.f;
    }
    float a = float(double(st->rs[it]) / double(pap));
    if (blockIdx.x == 0)
        st->alpha[it] = a;
    return a;
}

__device__ float cg_alpha(CgDev* st, int it, unsigned* errflags) { return cg_alpha_sum(st, it, st->pap_sum, errflags); }

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

// Every CTA of a partial-producing kernel calls this with its block sum (valid
// on thread 0).  The last CTA to arrive folds all partials in a fixed order
// (thread-strided, then the block tree) and publishes the real part, so the
// consumers read one scalar instead of re-summing gridDim partials per CTA.
__device__ void publish_partial(double2* parts, double* result, unsigned* counter, double2 part)
{
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        parts[blockIdx.x] = part;
        __threadfence();
        s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last)
        return;
    __threadfence();
    double2 v{0, 0};
    for (unsigned k = threadIdx.x; k < gridDim.x; k += blockDim.x)
        v.x += __ldcg(&parts[k].x);
    v = block_sum2(v);
    if (threadIdx.x == 0) {
        *result = v.x;
        *counter = 0;
    }
}

// ---------------------------------------------------------------------------
// Fused single-pass y-only normal operator.
//   mode 0: out = A^H A x + lam x
//   mode 1 (CG iteration it): p = (it ? r + beta p : p); out = Ap; partial <p,Ap>
// smem: xs[M][Y*W], acc[M][Y*W], buf a/b [Y*W]; layout [k*W + w].
// ---------------------------------------------------------------------------
struct NormalArgs {
    cfloat* out;
    const cfloat* x;     // mode 0: input image; mode 1: r
    cfloat* p;           // mode 1: search direction (read/write)
    const cfloat* coils;  // coil_mul maps
    const cfloat* coils2; // coil_adj maps (equal to coils after dedupe)
    const cfloat* pattern;
    const cfloat* lam;   // device complex scalar or null
    long X, Y, C, M, B;
    PatStr ps;
    int W;
    int nsplit;          // fast kernel: coil ranges per column strip (Ap planes)
    int mode;
    int it;
    CgDev* cg;
    unsigned* errflags;
};

__global__ void __launch_bounds__(kT) k_normal_y(NormalArgs a, fftd::Plan plan)
{
    MDNN_PDL_ENTRY();
    extern __shared__ float2 sm[];
    const int Y = int(a.Y), W = a.W, M = int(a.M);
    const int nYW = Y * W;
    float2* xs = sm;
    float2* acc = xs + size_t(M) * nYW;
    float2* ba = acc + size_t(M) * nYW;
    float2* bb = ba + nYW;
    __shared__ float s_beta;
    __shared__ float2 s_lam;

    const long nxb = (a.X + W - 1) / W;
    const long x0 = (blockIdx.x % nxb) * W;
    const long b = blockIdx.x / nxb;
    const long XY = a.X * a.Y;

    if (threadIdx.x == 0) {
        s_beta = a.mode == 1 ? cg_prologue(a.cg, a.it, a.errflags) : 0.f;
        s_lam = a.lam ? a.lam[0] : float2{0.f, 0.f};
    }
    __syncthreads();
    const float beta = s_beta;
    if (a.mode == 1 && beta < 0.f)
        return; // converged / stopped: uniform across the CTA

    // load x (or form p = r + beta p) and zero the accumulators
    for (int m = 0; m < M; m++) {
        for (int e = threadIdx.x; e < nYW; e += blockDim.x) {
            const int w = e % W, k = e / W;
            const long xx = x0 + w;
            float2 v{0.f, 0.f};
            if (xx < a.X) {
                const long gi = xx + a.X * (k + a.Y * (m + a.M * b));
                if (a.mode == 0) {
                    v = a.x[gi];
                } else {
                    if (a.it > 0) {
                        float2 r = a.x[gi], pv = a.p[gi];
                        v = float2{r.x + beta * pv.x, r.y + beta * pv.y};
                        a.p[gi] = v;
                    } else {
                        v = a.p[gi];
                    }
                }
            }
            xs[m * nYW + e] = v;
            acc[m * nYW + e] = float2{0.f, 0.f};
        }
    }
    __syncthreads();

    const float invY = 1.f / float(Y);
    for (long c = 0; c < a.C; c++) {
        // u = sum_m C_{c,m} x_m
        for (int e = threadIdx.x; e < nYW; e += blockDim.x) {
            const int w = e % W, k = e / W;
            const long xx = x0 + w;
            float2 u{0.f, 0.f};
            if (xx < a.X)
                for (int m = 0; m < M; m++) {
                    float2 cv = a.coils[xx + a.X * (k + a.Y * (c + a.C * (m + a.M * b)))];
                    float2 xv = xs[m * nYW + e];
                    u.x += cv.x * xv.x - cv.y * xv.y;
                    u.y += cv.x * xv.y + cv.y * xv.x;
                }
            ba[e] = u;
        }
        __syncthreads();
        float2* r = fftd::fft_smem(ba, bb, plan, W);
        float2* o = r == ba ? bb : ba;
        // mask, scale 1/Y (both unitary factors), conjugate for the inverse pass
        for (int e = threadIdx.x; e < nYW; e += blockDim.x) {
            const int k = e / W;
            float2 pv = a.pattern[k * a.ps.sy + b * a.ps.sb];
            float2 v = cmul(r[e], pv);
            r[e] = float2{v.x * invY, -v.y * invY};
        }
        __syncthreads();
        float2* r2 = fftd::fft_smem(r, o, plan, W);
        // acc_m += conj(C_{c,m}) * conj(r2)
        for (int e = threadIdx.x; e < nYW; e += blockDim.x) {
            const int w = e % W, k = e / W;
            const long xx = x0 + w;
            if (xx < a.X) {
                float2 v = cconj(r2[e]);
                for (int m = 0; m < M; m++) {
                    float2 cv = a.coils2[xx + a.X * (k + a.Y * (c + a.C * (m + a.M * b)))];
                    float2 t = cmulc(v, cv);
                    acc[m * nYW + e].x += t.x;
                    acc[m * nYW + e].y += t.y;
                }
            }
        }
        __syncthreads();
    }

    // epilogue
    double2 part{0, 0};
    for (int m = 0; m < M; m++)
        for (int e = threadIdx.x; e < nYW; e += blockDim.x) {
            const int w = e % W, k = e / W;
            const long xx = x0 + w;
            if (xx >= a.X)
                continue;
            const long gi = xx + a.X * (k + a.Y * (m + a.M * b));
            float2 v = acc[m * nYW + e];
            float2 xv = xs[m * nYW + e];
            if (a.mode == 0) {
                float2 lx = cmul(xv, s_lam);
                v.x += lx.x;
                v.y += lx.y;
            } else {
                float2 lx = cmul(xv, s_lam);
                v.x += lx.x;
                v.y += lx.y;
                // <p, Ap> = sum p * conj(Ap)
                part.x += double(xv.x) * v.x + double(xv.y) * v.y;
                part.y += double(xv.y) * v.x - double(xv.x) * v.y;
            }
            a.out[gi] = v;
        }
    if (a.mode == 1) {
        part = block_sum2(part);
        publish_partial(a.cg->part_pap, &a.cg->pap_sum, &a.cg->cnt_pap, part);
    }
    (void)XY;
}

} // namespace
} // namespace mdnn
#include <map>
#include <mutex>
namespace mdnn {
namespace {
#include "sense_fast.cuh"
#include "sense_rank.cuh"
#include "sense_ws.cuh"

bool fast_ok(const SenseGeom& g, const cfloat* coils, const cfloat* coils2)
{
    return g.M == 1 && coils2 == coils && g.pat_x == 1 && g.pat_c == 1 && fast_n1(g.Y) != 0;
}

int pick_w(long Y, int M)
{
    int W = 16;
    while (W > 1 && size_t(2 * M + 2) * Y * W * sizeof(float2) > 110 * 1024)
        W /= 2;
    return W;
}

bool fused_ok(const SenseGeom& g)
{
    return g.pat_x == 1 && g.pat_c == 1 && fft_supported(g.Y) && g.M <= 4
           && size_t(2 * g.M + 2) * g.Y * sizeof(float2) <= ctx().smem_optin;
}

void launch_normal_y(NormalArgs a, const SenseGeom& g)
{
    const auto& plan = fft_plan(int(g.Y));
    a.W = pick_w(g.Y, int(g.M));
    size_t smem = size_t(2 * g.M + 2) * g.Y * a.W * sizeof(float2);
    auto& c = ctx();
    allow_max_dyn_smem(reinterpret_cast<const void*>(k_normal_y));
    long nxb = (g.X + a.W - 1) / a.W;
    // algorithmic bytes: A^H A + lam reads x + coils and writes the
    // image; the CG launch also reads r and rewrites p (8 XYB (CM + 4M))
    const double xyb = double(g.X) * g.Y * g.B;
    const double work = 8.0 * xyb * (g.C * g.M + (a.mode == 1 ? 4 : 2) * g.M);
    ProfScope prof(a.mode == 1 ? "sense_normal_y_cg" : "sense_normal_y", work);
    pdl_launch(k_normal_y, unsigned(nxb * g.B), kT, smem, c.stream, a, plan);
    KERNEL_CHECK();
}

long normal_y_ctas(const SenseGeom& g)
{
    int W = pick_w(g.Y, int(g.M));
    return ((g.X + W - 1) / W) * g.B;
}

// ---- CG helper kernels -------------------------------------------------------
__global__ void k_cg_init(CgDev* st, const double2* bsum)
{
    MDNN_PDL_ENTRY();
    double s = bsum[0].x;
    st->bnorm = sqrt(s);
    st->rs[0] = float(s);
    st->done_at = (s == 0.0) ? 0 : INT_MAX;
}

// generic path: p-update (prologue) as its own kernel
__global__ void k_cg_pupdate(CgDev* st, int it, cfloat* p, const cfloat* r, long n, unsigned* errflags, int* skip)
{
    MDNN_PDL_ENTRY();
    __shared__ float s_beta;
    if (threadIdx.x == 0)
        s_beta = cg_prologue(st, it, errflags);
    __syncthreads();
    float beta = s_beta;
    if (blockIdx.x == 0 && threadIdx.x == 0)
        *skip = beta < 0.f ? 1 : 0;
    if (beta < 0.f || it == 0)
        return;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        float2 rv = r[i], pv = p[i];
        p[i] = float2{rv.x + beta * pv.x, rv.y + beta * pv.y};
    }
}

__global__ void k_cg_pap(CgDev* st, int it, const cfloat* p, const cfloat* ap, long n)
{
    MDNN_PDL_ENTRY();
    if (st->done_at <= it)
        return;
    double2 part{0, 0};
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        float2 a = p[i], b = ap[i];
        part.x += double(a.x) * b.x + double(a.y) * b.y;
        part.y += double(a.y) * b.x - double(a.x) * b.y;
    }
    part = block_sum2(part);
    publish_partial(st->part_pap, &st->pap_sum, &st->cnt_pap, part);
}

__global__ void k_cg_update(CgDev* st, int it, cfloat* x, cfloat* r, const cfloat* p, const cfloat* ap, long n,
                            unsigned* errflags)
{
    MDNN_PDL_ENTRY();
    __shared__ float s_alpha;
    if (threadIdx.x == 0)
        s_alpha = cg_alpha(st, it, errflags);
    __syncthreads();
    const float al = s_alpha;
    if (!(al > 0.f))
        return; // stopped, converged or broken down (flag raised)
    double2 part{0, 0};
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        float2 pv = p[i], av = ap[i], xv = x[i], rv = r[i];
        // md_axpy(x, alpha, p); md_axpy(r, -alpha, ap)  (mdarray.hpp:673-677)
        xv.x += al * pv.x;
        xv.y += al * pv.y;
        rv.x += -al * av.x;
        rv.y += -al * av.y;
        x[i] = xv;
        r[i] = rv;
        part.x += double(rv.x) * rv.x + double(rv.y) * rv.y;
    }
    part = block_sum2(part);
    publish_partial(st->part_rr, &st->rr_sum, &st->cnt_rr, part);
}

__global__ void k_cg_final(CgDev* st, double* status_out, unsigned* errflags)
{
    MDNN_PDL_ENTRY();
    // CgStatus after the loop (recon.hpp:176-178)
    int it = st->done_at;
    bool conv = false;
    float rs_last;
    if (it == INT_MAX) {
        it = st->max_iter;
        rs_last = float(st->rr_sum);
        if (!isfinite(rs_last))
            atomicOr(errflags, unsigned(ERRF_CG_NONFINITE));
    } else {
        rs_last = st->rs[it];
        conv = true; // loop left through the convergence test (breakdowns raise)
    }
    double rel = st->bnorm == 0 ? 0.0 : sqrt(double(rs_last)) / st->bnorm;
    conv = conv || rel <= st->tol;
    if (status_out) {
        status_out[0] = double(it);
        status_out[1] = rel;
        status_out[2] = conv ? 1.0 : 0.0;
    }
}

} // namespace

// ---------------------------------------------------------------------------

void launch_coil_mul(cfloat* u, const cfloat* x, const cfloat* coils, const SenseGeom& g)
{
    long XY = g.X * g.Y;
    pdl_launch(k_coil_mul, grid_for(XY * g.C * g.B), kT, 0, ctx().stream, u, x, coils, XY, g.C, g.M, g.B);
    KERNEL_CHECK();
}

void launch_coil_adj(cfloat* x, const cfloat* u, const cfloat* coils, const SenseGeom& g)
{
    long XY = g.X * g.Y;
    pdl_launch(k_coil_adj, grid_for(XY * g.M * g.B), kT, 0, ctx().stream, x, u, coils, XY, g.C, g.M, g.B);
    KERNEL_CHECK();
}

void launch_pattern_mul(cfloat* out, const cfloat* u, const cfloat* pattern, const SenseGeom& g)
{
    pdl_launch(k_pattern_mul, grid_for(g.X * g.Y * g.C * g.B), kT, 0, ctx().stream, out, u, pattern, g.X, g.Y, g.C, g.B,
                                                                             pat_strides(g));
    KERNEL_CHECK();
}

static Dims coil_img_dims(const SenseGeom& g)
{
    Dims d(max_rank, 1);
    d[0] = g.X;
    d[1] = g.Y;
    d[3] = g.C;
    d[15] = g.B;
    return d;
}

void sense_forward(cfloat* y, const cfloat* x, const cfloat* coils, const cfloat* pattern, const SenseGeom& g)
{
    launch_coil_mul(y, x, coils, g);
    fft_flags(y, y, coil_img_dims(g), 3UL, false);
    launch_pattern_mul(y, y, pattern, g);
}

void sense_adjoint(cfloat* x, const cfloat* y, const cfloat* coils, const cfloat* pattern, const SenseGeom& g)
{
    DArray t(coil_img_dims(g), false);
    launch_pattern_mul(t.data(), y, pattern, g);
    fft_flags(t.data(), t.data(), coil_img_dims(g), 3UL, true);
    launch_coil_adj(x, t.data(), coils, g);
}

// Rank-factorised A^H A + lambda (sense_rank.cuh / sense_ws.cuh), lambda from the
// device (lam) or by value (lam == nullptr: lamv).  Launches: the plan pass (split
// flags and, with check_pattern, the binary-pattern check folded in), the A^H A
// kernel, and the plane merge only when strips are shared.  false: shape unsupported.
static bool sense_normal_rank(cfloat* out, const cfloat* x, const cfloat* coils, const cfloat* pattern,
                              const cfloat* lam, float2 lamv, const SenseGeom& g, bool check_pattern)
{
    if (!rank_enabled())
        return false;
    const RankPlan rp = rank_plan(g, coils);
    if (!rp.ok)
        return false;
    const long n = g.X * g.Y * g.B;
    DArray plane1;
    if (rp.planes > 1)
        plane1 = DArray(Dims{n * (rp.planes - 1)}, false);
    DArray plans(Dims{long((rank_plan_bytes(g, rp) + 7) / 8)}, false);
    RankArgs a{};
    a.out = out;
    a.out1 = rp.planes > 1 ? plane1.data() : nullptr;
    a.pstride = n;
    a.x = x;
    a.pattern = pattern;
    a.lam = lam;
    a.lamv = lamv;
    a.ps = pat_strides(g);
    a.mode = 0;
    a.errflags = ctx().d_errflags;
    a.check_pattern = check_pattern ? 1 : 0;
    unsigned char* pl = reinterpret_cast<unsigned char*>(plans.data());
    launch_rank_plan(rp, a, g, pl);
    a.check_pattern = 0;
    launch_rank(rp, a, coils, g, pl);
    if (rp.planes > 1) {
        pdl_launch(k_rank_merge, grid_for(n), 256, 0, ctx().stream, out, plane1.data(), rank_split_flags(g, rp, pl),
                                                            int(g.X), int(g.Y * g.B), int(g.Y), int(rp.nxb),
                                                            rp.W == 8 ? 3 : 2, n);
        KERNEL_CHECK();
    }
    return true;
}

void sense_normal_value(cfloat* out, const cfloat* x, const cfloat* coils, const cfloat* pattern, float lambda,
                        const SenseGeom& g, bool check_pattern)
{
    if (sense_normal_rank(out, x, coils, pattern, nullptr, float2{lambda, 0.f}, g, check_pattern))
        return;
    if (check_pattern)
        launch_check_binary(pattern, g.pat_x * g.pat_y * g.pat_c * g.pat_b);
    DArray lam = DArray::scalar(lambda);
    sense_normal(out, x, coils, pattern, lam.data(), g);
}

void sense_normal(cfloat* out, const cfloat* x, const cfloat* coils, const cfloat* pattern, const cfloat* lam,
                  const SenseGeom& g, const cfloat* coils2)
{
    if (!coils2)
        coils2 = coils;
    if (coils2 == coils && sense_normal_rank(out, x, coils, pattern, lam, float2{0.f, 0.f}, g, false))
        return;
    if (fast_ok(g, coils, coils2)) {
        NormalArgs a{};
        a.out = out;
        a.x = x;
        a.coils = coils;
        a.coils2 = coils2;
        a.pattern = pattern;
        a.lam = lam;
        a.X = g.X;
        a.Y = g.Y;
        a.C = g.C;
        a.M = g.M;
        a.B = g.B;
        a.ps = pat_strides(g);
        a.mode = 0;
        a.errflags = ctx().d_errflags;
        a.nsplit = 1;
        if (dispatch_fast(a, nullptr, 0))
            return;
    }
    if (fused_ok(g)) {
        NormalArgs a{};
        a.out = out;
        a.x = x;
        a.coils = coils;
        a.coils2 = coils2;
        a.pattern = pattern;
        a.lam = lam;
        a.X = g.X;
        a.Y = g.Y;
        a.C = g.C;
        a.M = g.M;
        a.B = g.B;
        a.ps = pat_strides(g);
        a.mode = 0;
        a.errflags = ctx().d_errflags;
        launch_normal_y(a, g);
        return;
    }
    DArray k(coil_img_dims(g), false);
    sense_forward(k.data(), x, coils, pattern, g);
    sense_adjoint(out, k.data(), coils2, pattern, g);
    long n = g.X * g.Y * g.M * g.B;
    if (lam) {
        DArray lx(Dims{n}, false);
        launch_scale_dev(lx.data(), x, lam, false, n);
        launch_add(out, out, lx.data(), 1.f, n);
    }
}

namespace {

struct CgMem {
    char* mem = nullptr;
    CgDev* st = nullptr;
    CgDev h{};
};

CgMem cg_alloc(long max_iter, double tol, int n_pap, int n_upd)
{
    auto& c = ctx();
    CgMem m;
    size_t bytes = 256 + sizeof(float) * (3 * (max_iter + 2)) + sizeof(double2) * (n_pap + n_upd + 2) + 64;
    CUDA_CHECK(cudaMallocAsync(&m.mem, bytes, c.stream));
    m.h.tol = tol;
    m.h.max_iter = int(max_iter);
    m.h.done_at = INT_MAX;
    m.h.n_pap = n_pap;
    m.h.n_rr = n_upd;
    char* q = m.mem + 256;
    m.h.part_pap = reinterpret_cast<double2*>(q);
    q += sizeof(double2) * n_pap;
    m.h.part_rr = reinterpret_cast<double2*>(q);
    q += sizeof(double2) * n_upd;
    q += sizeof(double2) * 2; // bsum scratch
    m.h.rs = reinterpret_cast<float*>(q);
    m.h.alpha = m.h.rs + (max_iter + 2);
    m.h.beta = m.h.alpha + (max_iter + 2);
    m.st = reinterpret_cast<CgDev*>(m.mem);
    CUDA_CHECK(cudaMemcpyAsync(m.st, &m.h, sizeof(CgDev), cudaMemcpyHostToDevice, c.stream));
    return m;
}

double2* cg_bsum(const CgMem& m) { return reinterpret_cast<double2*>(reinterpret_cast<char*>(m.h.part_rr) + sizeof(double2) * m.h.n_rr); }

// x = 0, r = b, p = b, bnorm, rs0
void cg_start(const CgMem& m, cfloat* x, const cfloat* b, cfloat* r, cfloat* p, long n)
{
    auto& c = ctx();
    CUDA_CHECK(cudaMemsetAsync(x, 0, n * sizeof(cfloat), c.stream));
    launch_copy(r, b, n);
    launch_copy(p, b, n);
    launch_zdot(reinterpret_cast<double*>(cg_bsum(m)), b, b, n);
    pdl_launch(k_cg_init, 1, 1, 0, c.stream, m.st, cg_bsum(m));
    KERNEL_CHECK();
}

} // namespace

void cg_generic_device(cfloat* x, const cfloat* b, long n, const CgApply& apply, long max_iter, double tol,
                       double* status_out)
{
    auto& c = ctx();
    const int n_upd = grid_for(n);
    CgMem m = cg_alloc(max_iter, tol, n_upd, n_upd);
    DArray r(Dims{n}, false), p(Dims{n}, false), ap(Dims{n}, false);
    cg_start(m, x, b, r.data(), p.data(), n);
    int* d_skip = reinterpret_cast<int*>(cg_bsum(m) + 1);
    for (int it = 0; it < max_iter; it++) {
        pdl_launch(k_cg_pupdate, n_upd, kT, 0, c.stream, m.st, it, p.data(), r.data(), n, c.d_errflags, d_skip);
        KERNEL_CHECK();
        // S p is always evaluated; iterations after convergence are discarded
        // by the device-side state (no host synchronisation in the loop)
        apply(p.data(), ap.data());
        pdl_launch(k_cg_pap, n_upd, kT, 0, c.stream, m.st, it, p.data(), ap.data(), n);
        KERNEL_CHECK();
        pdl_launch(k_cg_update, n_upd, kT, 0, c.stream, m.st, it, x, r.data(), p.data(), ap.data(), n, c.d_errflags);
        KERNEL_CHECK();
    }
    pdl_launch(k_cg_final, 1, 1, 0, c.stream, m.st, status_out, c.d_errflags);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(m.mem, c.stream));
}

void cg_normal_device(cfloat* x, const cfloat* b, const cfloat* coils, const cfloat* pattern, const cfloat* lam,
                      const SenseGeom& g, long max_iter, double tol, double* status_out)
{
    const long n = g.X * g.Y * g.M * g.B;
    if (!fused_ok(g)) {
        cg_generic_device(
            x, b, n, [&](const cfloat* p, cfloat* ap) { sense_normal(ap, p, coils, pattern, lam, g); }, max_iter,
            tol, status_out);
        return;
    }
    auto& c = ctx();
    const int n_upd = grid_for(n);
    const RankPlan rp = rank_enabled() ? rank_plan(g, coils) : RankPlan{};
    if (rp.ok) {
        // persistent rank kernel: Ap in plane 0 (+ plane 1 for split strips);
        // p ping-pongs between two buffers (no CTA reads a p another rewrites)
        // few update CTAs: one contended counter atomic per CTA in publish_partial
        // Deferred x (up to 32 iterations): every direction p_it is kept (P[it + 1]),
        // the update kernel touches Ap and r only, and x is summed once at the end.
        const bool defer = max_iter <= 32 && g_cg_defer_x && n % 2 == 0;
        constexpr int UR = 2; // element pairs per thread in k_cg_update_r
        const long npair = n / 2;
        // deferred update: as few latency rounds per thread as 4 co-resident
        // 256-thread CTAs per SM allow, every round full (no partial last round)
        const long upd_round = 256L * UR * 4 * c.sm_count;
        const long upd_rounds = std::max(1L, (npair + upd_round - 1) / upd_round);
        const int n_updr = defer ? int((npair + 256L * UR * upd_rounds - 1) / (256L * UR * upd_rounds))
                                 : int(std::min<long>(2L * c.sm_count, g.Y * g.B));
        // fused update (ws kernel, deferred x): r -= alpha Ap after a grid barrier in
        // the A^H A launch itself, one launch per iteration
        const bool fuse = defer && rp.ws && g_cg_fuse != 0;
        CgMem m = cg_alloc(max_iter, tol, rp.G, std::max(n_updr, rp.G));
        DArray r(Dims{n}, false), pb(Dims{(defer ? max_iter + 1 : 2) * n}, false),
            ap(Dims{n * std::max(2, rp.planes)}, false);
        DArray plans(Dims{long((rank_plan_bytes(g, rp) + 7) / 8)}, false);
        unsigned char* pl = reinterpret_cast<unsigned char*>(plans.data());
        cfloat* P[2] = {pb.data(), pb.data() + n};
        auto pdir = [&](int k) { return defer ? pb.data() + long(k) * n : P[k & 1]; }; // p_(k-1) lives at pdir(k)
        cg_start(m, x, b, r.data(), pdir(1), n);
        {
            RankArgs a{};
            a.pattern = pattern;
            a.ps = pat_strides(g);
            launch_rank_plan(rp, a, g, pl);
        }
        for (int it = 0; it < max_iter; it++) {
            RankArgs a{};
            a.out = ap.data();
            a.out1 = ap.data() + n;
            a.pstride = n;
            a.x = r.data();
            a.p = pdir(it);
            a.p_out = pdir(it + 1);
            a.pattern = pattern;
            a.lam = lam;
            a.ps = pat_strides(g);
            a.mode = 1;
            a.it = it;
            a.cg = m.st;
            a.errflags = c.d_errflags;
            if (fuse) {
                a.r_upd = r.data();
                a.split = const_cast<unsigned char*>(rank_split_flags(g, rp, pl));
                a.upd_rows = int(g.Y * g.B);
                a.upd_Y = int(g.Y);
                a.upd_wshift = rp.W == 8 ? 3 : 2;
            }
            launch_rank(rp, a, coils, g, pl);
            if (fuse) {
                // (the update ran in the A^H A launch)
            } else if (defer) {
                ProfScope prof("cg_update_rank", 8.0 * n * 4);
                launch_maybe_pdl(g_cg_pdl && rp.ws, k_cg_update_r<UR>, dim3(n_updr), dim3(256), 0, m.st, it, r.data(),
                                 static_cast<const cfloat*>(ap.data()), static_cast<const cfloat*>(ap.data() + n),
                                 rank_split_flags(g, rp, pl), int(g.X), int(g.Y * g.B), int(g.Y), int(rp.nxb),
                                 rp.W == 8 ? 3 : 2, n, c.d_errflags);
            } else {
                ProfScope prof("cg_update_rank", 8.0 * n * 7);
                pdl_launch(k_cg_update_rank, n_updr, 512, 0, c.stream, m.st, it, x, r.data(), pdir(it + 1), ap.data(),
                                                              ap.data() + n, rank_split_flags(g, rp, pl), int(g.X),
                                                              int(g.Y * g.B), int(g.Y), int(rp.nxb),
                                                              rp.W == 8 ? 3 : 2, n, c.d_errflags);
            }
            KERNEL_CHECK();
        }
        if (defer) {
            pdl_launch(k_cg_x_sum, grid_for(n / 2), 256, 0, c.stream, m.st, x, pb.data(), n);
            KERNEL_CHECK();
        }
        pdl_launch(k_cg_final, 1, 1, 0, c.stream, m.st, status_out, c.d_errflags);
        KERNEL_CHECK();
        CUDA_CHECK(cudaFreeAsync(m.mem, c.stream));
        return;
    }
    if (fast_ok(g, coils, coils)) {
        // register-resident kernel, coils split over NS CTAs -> NS Ap planes
        // (NS picked against the wave tail); p ping-pongs between two buffers
        // (no CTA reads a p another rewrites)
        const int NS = fast_nsplit(g);
        CgMem m = cg_alloc(max_iter, tol, int(fast_ctas(g, NS)), n_upd);
        DArray r(Dims{n}, false), pb(Dims{2 * n}, false), ap(Dims{NS * n}, false);
        cfloat* P[2] = {pb.data(), pb.data() + n};
        cg_start(m, x, b, r.data(), P[1], n);
        for (int it = 0; it < max_iter; it++) {
            NormalArgs a{};
            a.out = ap.data();
            a.x = r.data();
            a.p = P[it & 1];
            a.coils = coils;
            a.coils2 = coils;
            a.pattern = pattern;
            a.lam = lam;
            a.X = g.X;
            a.Y = g.Y;
            a.C = g.C;
            a.M = g.M;
            a.B = g.B;
            a.ps = pat_strides(g);
            a.mode = 1;
            a.it = it;
            a.cg = m.st;
            a.errflags = c.d_errflags;
            a.nsplit = NS;
            dispatch_fast(a, P[(it + 1) & 1], n);
            pdl_launch(k_cg_update_planes, n_upd, kT, 0, c.stream, m.st, it, x, r.data(), P[(it + 1) & 1], ap.data(), n,
                                                          NS, n, c.d_errflags);
            KERNEL_CHECK();
        }
        pdl_launch(k_cg_final, 1, 1, 0, c.stream, m.st, status_out, c.d_errflags);
        KERNEL_CHECK();
        CUDA_CHECK(cudaFreeAsync(m.mem, c.stream));
        return;
    }
    const int n_pap = int(normal_y_ctas(g));
    CgMem m = cg_alloc(max_iter, tol, n_pap, n_upd);
    DArray r(Dims{n}, false), p(Dims{n}, false), ap(Dims{n}, false);
    cg_start(m, x, b, r.data(), p.data(), n);
    for (int it = 0; it < max_iter; it++) {
        NormalArgs a{};
        a.out = ap.data();
        a.x = r.data();
        a.p = p.data();
        a.coils = coils;
        a.coils2 = coils;
        a.pattern = pattern;
        a.lam = lam;
        a.X = g.X;
        a.Y = g.Y;
        a.C = g.C;
        a.M = g.M;
        a.B = g.B;
        a.ps = pat_strides(g);
        a.mode = 1;
        a.it = it;
        a.cg = m.st;
        a.errflags = c.d_errflags;
        launch_normal_y(a, g);
        pdl_launch(k_cg_update, n_upd, kT, 0, c.stream, m.st, it, x, r.data(), p.data(), ap.data(), n, c.d_errflags);
        KERNEL_CHECK();
    }
    pdl_launch(k_cg_final, 1, 1, 0, c.stream, m.st, status_out, c.d_errflags);
    KERNEL_CHECK();
    CUDA_CHECK(cudaFreeAsync(m.mem, c.stream));
}

namespace {
bool g_rank_enabled = true;
}
// rank-kernel CTA count override lives in sense_rank.cuh (g_rank_ctas)
void sense_rank_enable(bool on) { g_rank_enabled = on; }
void sense_rank_ctas(long g) { g_rank_ctas = g; }
void sense_ws_enable(bool on) { g_sense_ws = on; }
void cg_pdl_enable(bool on) { g_cg_pdl = on; }
void cg_fuse_enable(int mode) { g_cg_fuse = mode; }
void rank_rr_enable(bool on) { g_rank_rr = on; }
void rank_vh_set(int vh) { g_rank_vh = vh < 0 ? 0 : vh; }
void cg_defer_x_enable(bool on) { g_cg_defer_x = on; }
bool rank_enabled() { return g_rank_enabled; }

CgResult read_cg_status(const double* status_dev)
{
    double h[3];
    CUDA_CHECK(cudaMemcpyAsync(h, status_dev, sizeof(h), cudaMemcpyDeviceToHost, ctx().stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx().stream));
    return CgResult{long(h[0]), h[1], h[2] != 0.0};
}

} // namespace mdnn
