// Persistent, mask-pruned, register-resident A^H A (+ lambda) for Y = N1 * N2
// (included by sense.cu after sense_fast.cuh).  Replaces the operator chain of
// sense_normal_fragment + modl_normal_plus_lambda (recon.hpp:410-418,
// 807-820) for x-invariant patterns; same maths as sense_fast.cuh, different
// schedule:
//
//  * Work units are (column strip, coil) pairs.  G = min(2 * SMs, strips) CTAs
//    each take a contiguous unit range, so every SM gets the same number of
//    coil slices (no wave tail).  Ranges are >= C units, so a strip is shared by
//    at most two CTAs: the one owning its coil 0 writes plane 0 (and adds
//    lambda x), the other writes plane 1, and the consumer sums the planes of
//    split strips (rank_split()).  fp add is commutative, so the two-term sum
//    is bitwise deterministic.
//  * Coil slices (W columns x Y rows) arrive by TMA into a 2-slot ring, one
//    mbarrier per slot; no per-thread copy instructions.
//  * Stage B is the exact mask rewrite of sense_fast.cuh: per row k1 of the
//    16 x N2 factorisation, identity, or a few rank-1 terms, or (rows with
//    many terms) a full in-register DFT.  Term rows never leave registers:
//    thread (w, j) holds A[k1][j] for all k1 after its DFT over q, forms the
//    products A[k1][j] w_k[j] for every term, pairs them with a warp shuffle
//    and drops them in smem; one thread per (term, column) sums the pairs;
//    every thread then adds d_t conj(w_k[j]) back into its registers.  Full
//    rows go through smem to one thread per (row, column).  Two barriers per
//    coil and all threads busy in both long phases.
#pragma once

long g_rank_ctas = 0; // 0: 2 per SM (tests force fewer to exercise split strips)

constexpr int rank_nbox(int Y)
{
    int n = (Y + 255) / 256;
    while (Y % n)
        n++;
    return n;
}

template<int N1, int N2>
struct RankCfg {
    static constexpr int Y = N1 * N2;
    static constexpr int W = N2 <= 24 ? 8 : 4;             // columns per strip
    static constexpr int NT = ((W * N2 + 31) / 32) * 32;   // threads (w, j)
    static constexpr int JP = (N2 + 1) / 2;                // shuffle-paired j slots
    static constexpr int KMAX = (N2 % 2 == 1) ? 5 : 2;      // terms per row before a full DFT pays
    static constexpr int TMAX = 32;                        // terms per CTA
    static constexpr int NBOX = rank_nbox(Y);              // TMA boxes per coil slice (rows <= 256)
    static constexpr int BOXR = Y / NBOX;
    static constexpr int UNION = Y * W;                    // float2: term pairs + full rows (>= all-full)
    static constexpr size_t SLOT = size_t(Y) * W;          // float2 per ring slot
    // dynamic smem (float2): ring[2][Y*W] | xs[Y*W] | un[UNION] | D[TMAX*W] | ttw[TMAX*N2] | stw[Y] | spat[Y]
    static constexpr size_t SMEM = sizeof(float2) * (2 * SLOT + SLOT + UNION + TMAX * W + TMAX * N2 + 2 * Y) + 128;
    static constexpr int MINB = 2 * (SMEM + 4096) <= 228 * 1024 ? 2 : 1;
    static_assert(Y % NBOX == 0, "TMA box rows must tile Y");
};

struct RankArgs {
    cfloat* out;          // plane 0 (mode 0: the result; mode 1: Ap)
    cfloat* out1;         // plane 1 (split strips)
    const cfloat* x;      // mode 0: input image; mode 1: r
    cfloat* p;            // mode 1: previous search direction
    cfloat* p_out;        // mode 1: new search direction (== x source at it 0)
    const cfloat* pattern;
    const cfloat* lam;
    const float2* tw;     // exp(-2 pi i m / Y), m < Y
    long X, C, B;
    long nxb;             // strips per item
    long units;           // strips * C
    int G;                // CTAs
    PatStr ps;
    int mode, it;
    CgDev* cg;
    unsigned* errflags;
};

// CTA owning unit u, for ranges [floor(U g / G), floor(U (g+1) / G))
__host__ __device__ __forceinline__ long rank_owner(long u, long U, long G) { return ((u + 1) * G + U - 1) / U - 1; }
__host__ __device__ __forceinline__ bool rank_split(long s, long C, long U, long G)
{
    return rank_owner(s * C, U, G) != rank_owner(s * C + C - 1, U, G);
}

template<int N1, int N2>
__global__ void __launch_bounds__(RankCfg<N1, N2>::NT, RankCfg<N1, N2>::MINB)
    k_normal_rank(RankArgs a, const __grid_constant__ CUtensorMap tmap)
{
    using namespace fftd;
    using Cfg = RankCfg<N1, N2>;
    constexpr int Y = Cfg::Y, W = Cfg::W, NT = Cfg::NT, JP = Cfg::JP, KMAX = Cfg::KMAX, TMAX = Cfg::TMAX;
    extern __shared__ __align__(128) unsigned char rank_smem[];
    float2* ring = reinterpret_cast<float2*>((reinterpret_cast<uintptr_t>(rank_smem) + 127) & ~uintptr_t(127));
    float2* xs = ring + 2 * Cfg::SLOT;
    float2* un = xs + Cfg::SLOT;
    float2* Ds = un + Cfg::UNION;
    float2* ttw = Ds + TMAX * W;
    float2* stw = ttw + TMAX * N2;
    float2* spat = stw + Y;
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ float s_beta;
    __shared__ float2 s_lam;
    __shared__ int s_cnt[N1], s_bb[N1], s_mode[N1], s_off[N1], s_nt[N1];
    __shared__ int s_fullk1[N1], s_tk[TMAX], s_T, s_nfull;
    __shared__ float2 s_coef[TMAX];

    const int tid = threadIdx.x;
    const int w = tid % W, j0 = tid / W;
    const bool active = j0 < N2;
    const int j = active ? j0 : N2 - 1;
    const long U = a.units, C = a.C;
    const long u_begin = U * blockIdx.x / a.G, u_end = U * (blockIdx.x + 1) / a.G;

    auto issue = [&](long u, int slot) { // TMA of unit u's coil slice into ring slot
        const long s = u / C, c = u % C;
        const long b = s / a.nxb, xblk = s % a.nxb;
        const int row0 = int(Y * (c + C * b));
        sm100::mbar_arrive_expect_tx(&s_bar[slot], uint32_t(Cfg::SLOT * sizeof(float2)));
#pragma unroll
        for (int k = 0; k < Cfg::NBOX; k++)
            sm100::tma_load_2d(ring + slot * Cfg::SLOT + k * Cfg::BOXR * W, &tmap, &s_bar[slot], int(2 * W * xblk),
                               row0 + k * Cfg::BOXR);
    };
    if (tid == 0) {
        sm100::prefetch_tmap(&tmap);
        sm100::mbar_init(&s_bar[0], 1);
        sm100::mbar_init(&s_bar[1], 1);
        sm100::fence_barrier_init();
        for (long u = u_begin; u < u_end && u < u_begin + 2; u++)
            issue(u, int(u - u_begin));
        s_beta = a.mode == 1 ? cg_prologue(a.cg, a.it, a.errflags) : 0.f;
        s_lam = a.lam ? a.lam[0] : float2{0.f, 0.f};
    }
    for (int e = tid; e < Y; e += NT)
        stw[e] = a.tw[e];
    __syncthreads();
    const float beta = s_beta;
    if (a.mode == 1 && beta < 0.f) {
        // CG already stopped: drain the TMA ring before exiting
        for (long u = u_begin; u < u_end && u < u_begin + 2; u++)
            sm100::mbar_wait(&s_bar[u - u_begin], 0);
        return;
    }
    const bool upd = a.mode == 1 && a.it > 0;
    const float2 lam = s_lam;
    constexpr float invN1 = 1.f / float(N1), invN2 = 1.f / float(N2);

    double2 part{0, 0};
    long plan_b = -1;
    long u = u_begin;
    while (u < u_end) {
        const long s = u / C;
        const long b = s / a.nxb, xblk = s % a.nxb;
        const long c0 = u % C;
        const long seg_end = min(u_end, (s + 1) * C);
        const bool first = c0 == 0;
        const long xx = xblk * W + w;
        const bool colok = active && xx < a.X;

        // ---- row plan for item b (pattern may differ per item) --------------
        if (b != plan_b && (plan_b < 0 || a.ps.sb != 0)) {
            __syncthreads(); // previous plan no longer read
            for (int e = tid; e < Y; e += NT)
                spat[e] = a.pattern[e * a.ps.sy + b * a.ps.sb];
            __syncthreads();
            if (tid < N1) {
                const int k1 = tid;
                int nz = 0, n1 = 0;
                for (int k2 = 0; k2 < N2; k2++) {
                    const float2 pv = spat[k1 + N1 * k2];
                    nz += (pv.x != 0.f || pv.y != 0.f);
                    n1 += (pv.x != 1.f || pv.y != 0.f);
                }
                s_bb[k1] = nz <= n1 ? 0 : 1;
                s_cnt[k1] = min(nz, n1);
            }
            __syncthreads();
            if (tid == 0) {
                // term rows while the union buffer and TMAX allow (cheapest
                // rows first), the rest full; modes: 0 identity, 1 add terms,
                // 2 replace by terms, 3 full DFT
                int order[N1];
                for (int k = 0; k < N1; k++)
                    order[k] = k;
                for (int i = 1; i < N1; i++) {
                    const int r = order[i];
                    int k = i - 1;
                    while (k >= 0 && s_cnt[order[k]] > s_cnt[r]) {
                        order[k + 1] = order[k];
                        k--;
                    }
                    order[k + 1] = r;
                }
                int T = 0, nfull = 0, used = 0;
                const int row_full = N2 * W, term_sz = JP * W;
                for (int i = 0; i < N1; i++) {
                    const int k1 = order[i], n = s_cnt[k1];
                    const int remaining = N1 - i - 1; // rows still to place may all go full
                    const bool fit = n <= KMAX && T + n <= TMAX
                                     && used + n * term_sz + remaining * row_full <= Cfg::UNION;
                    if (n == 0) {
                        s_mode[k1] = s_bb[k1] ? 0 : 2;
                        s_nt[k1] = 0;
                        s_off[k1] = 0;
                    } else if (fit) {
                        s_mode[k1] = s_bb[k1] ? 1 : 2;
                        s_nt[k1] = n;
                        s_off[k1] = T;
                        T += n;
                        used += n * term_sz;
                    } else {
                        s_mode[k1] = 3;
                        s_nt[k1] = 0;
                        s_off[k1] = nfull;
                        s_fullk1[nfull++] = k1;
                        used += row_full;
                    }
                }
                s_T = T;
                s_nfull = nfull;
            }
            __syncthreads();
            if (tid < N1) {
                const int k1 = tid, bb = s_bb[k1];
                if (s_mode[k1] == 1 || s_mode[k1] == 2) {
                    int t = s_off[k1];
                    for (int k2 = 0; k2 < N2; k2++) {
                        const float2 pv = spat[k1 + N1 * k2];
                        if (pv.x != float(bb) || pv.y != 0.f) {
                            s_tk[t] = k1 + N1 * k2;
                            s_coef[t] = float2{(pv.x - float(bb)) * invN2, pv.y * invN2};
                            t++;
                        }
                    }
                }
            }
            __syncthreads();
            for (int e = tid; e < s_T * N2; e += NT) {
                const int t = e / N2, jj = e % N2;
                ttw[e] = stw[(jj * s_tk[t]) % Y];
            }
            __syncthreads();
            plan_b = b;
        }
        const int T = s_T, nfull = s_nfull;
        float2* Pbuf = un;                       // [T][JP][W]
        float2* Rbuf = un + T * JP * W;          // [nfull][N2][W]

        // ---- x (or p = r + beta p_prev) column strip -> xs ----------------------
        {
            const long img_base = xx + a.X * Y * b;
            float2 v[N1], pv[N1];
            const float2* src = a.mode == 0 ? a.x : (a.it == 0 ? a.p_out : a.x);
#pragma unroll
            for (int q = 0; q < N1; q++) {
                const long gi = img_base + a.X * (j + N2 * q);
                v[q] = colok ? src[gi] : float2{0.f, 0.f};
                pv[q] = (colok && upd) ? a.p[gi] : float2{0.f, 0.f};
            }
#pragma unroll
            for (int q = 0; q < N1; q++) {
                const int y = j + N2 * q;
                if (upd) {
                    v[q] = float2{v[q].x + beta * pv[q].x, v[q].y + beta * pv[q].y};
                    if (first && colok)
                        a.p_out[img_base + a.X * y] = v[q];
                }
                if (active)
                    xs[y * W + w] = v[q];
            }
        }

        float2 acc[N1];
#pragma unroll
        for (int q = 0; q < N1; q++)
            acc[q] = float2{0.f, 0.f};

        for (; u < seg_end; u++) {
            const long i = u - u_begin;
            const int slot = int(i & 1);
            const float2* cs = ring + slot * Cfg::SLOT;
            sm100::mbar_wait(&s_bar[slot], uint32_t((i >> 1) & 1));
            // ---- phase 1: coil multiply, DFT over q, term products / full rows
            float2 v[N1];
            {
                float2 cv[N1];
#pragma unroll
                for (int q = 0; q < N1; q++)
                    cv[q] = cs[(j + N2 * q) * W + w];
#pragma unroll
                for (int q = 0; q < N1; q++)
                    v[q] = active ? cmul(cv[q], xs[(j + N2 * q) * W + w]) : float2{0.f, 0.f};
            }
            dft_reg<N1, -1>(v);
#pragma unroll
            for (int k1 = 0; k1 < N1; k1++) {
                const int mode = s_mode[k1];
                if (mode == 3) {
                    if (active)
                        Rbuf[(s_off[k1] * N2 + j) * W + w] = v[k1];
                } else if (mode != 0 || s_nt[k1] > 0) {
                    const int off = s_off[k1], nt = s_nt[k1];
                    for (int t = off; t < off + nt; t++) {
                        float2 pr = cmul(v[k1], ttw[t * N2 + j]);
                        pr.x += __shfl_xor_sync(0xffffffffu, pr.x, W);
                        pr.y += __shfl_xor_sync(0xffffffffu, pr.y, W);
                        if (!(j0 & 1) && j0 < N2)
                            Pbuf[(t * JP + (j0 >> 1)) * W + w] = pr;
                    }
                }
            }
            __syncthreads();
            // both readers of this slot are done after the barrier of the next
            // unit's phase 1; refill the other slot now (its unit finished)
            if (tid == 0 && i >= 1 && u + 1 < u_end)
                issue(u + 1, slot ^ 1);
            // ---- phase 2: term sums (t, w) and full rows (r, w) -----------------
            for (int it2 = tid; it2 < (T + nfull) * W; it2 += NT) {
                const int ww = it2 % W, t = it2 / W;
                if (t < T) {
                    float2 d{0.f, 0.f};
#pragma unroll
                    for (int jp = 0; jp < JP; jp++) {
                        const float2 pv = Pbuf[(t * JP + jp) * W + ww];
                        d.x += pv.x;
                        d.y += pv.y;
                    }
                    Ds[t * W + ww] = cmul(d, s_coef[t]);
                } else {
                    const int r = t - T, k1 = s_fullk1[r];
                    float2* row = Rbuf + r * N2 * W + ww;
                    float2 uu[N2];
#pragma unroll
                    for (int jj = 0; jj < N2; jj++)
                        uu[jj] = row[jj * W];
#pragma unroll
                    for (int jj = 1; jj < N2; jj++)
                        uu[jj] = cmul(uu[jj], stw[jj * k1]);
                    dft_reg<N2, -1>(uu);
#pragma unroll
                    for (int k2 = 0; k2 < N2; k2++) {
                        const float2 pv = spat[k1 + N1 * k2];
                        uu[k2] = cmul(uu[k2], float2{pv.x * invN2, pv.y * invN2});
                    }
                    dft_reg<N2, +1>(uu);
#pragma unroll
                    for (int jj = 1; jj < N2; jj++)
                        uu[jj] = cmulc(uu[jj], stw[jj * k1]);
#pragma unroll
                    for (int jj = 0; jj < N2; jj++)
                        row[jj * W] = uu[jj];
                }
            }
            __syncthreads();
            // ---- phase 3: rows back into registers, inverse DFT, conj-coil accumulate
#pragma unroll
            for (int k1 = 0; k1 < N1; k1++) {
                const int mode = s_mode[k1];
                if (mode == 3) {
                    v[k1] = Rbuf[(s_off[k1] * N2 + j) * W + w];
                } else if (mode != 0) {
                    if (mode == 2)
                        v[k1] = float2{0.f, 0.f};
                    const int off = s_off[k1], nt = s_nt[k1];
                    for (int t = off; t < off + nt; t++) {
                        const float2 dt = Ds[t * W + w], tv = ttw[t * N2 + j]; // v += d conj(tv)
                        v[k1].x = fmaf(dt.x, tv.x, v[k1].x);
                        v[k1].y = fmaf(dt.y, tv.x, v[k1].y);
                        v[k1].x = fmaf(dt.y, tv.y, v[k1].x);
                        v[k1].y = fmaf(-dt.x, tv.y, v[k1].y);
                    }
                }
            }
            dft_reg<N1, +1>(v);
#pragma unroll
            for (int q = 0; q < N1; q++) {
                const float2 cv = cs[(j + N2 * q) * W + w];
                const float2 t = cmulc(v[q], cv);
                acc[q].x += t.x;
                acc[q].y += t.y;
            }
            (void)KMAX;
        }

        // ---- segment epilogue: 1/N1, + lambda x (plane 0), store, <p, Ap> -----
        {
            const long img_base = xx + a.X * Y * b;
            cfloat* dst = first ? a.out : a.out1;
#pragma unroll
            for (int q = 0; q < N1; q++) {
                const int y = j + N2 * q;
                const float2 xv = xs[y * W + w];
                float2 o{acc[q].x * invN1, acc[q].y * invN1};
                if (first) {
                    const float2 lx = cmul(xv, lam);
                    o.x += lx.x;
                    o.y += lx.y;
                }
                if (colok) {
                    dst[img_base + a.X * y] = o;
                    part.x += double(xv.x) * o.x + double(xv.y) * o.y;
                    part.y += double(xv.y) * o.x - double(xv.x) * o.y;
                }
            }
        }
        __syncthreads(); // xs / plan reuse by the next segment
    }
    if (a.mode == 1) {
        part = block_sum2(part);
        publish_partial(a.cg->part_pap, &a.cg->pap_sum, &a.cg->cnt_pap, part);
    }
}

// out (+)= plane 1 for pixels of split strips (mode 0 result assembly)
template<int W>
__global__ void k_rank_merge(cfloat* out, const cfloat* plane1, long X, long Y, long B, long nxb, long C, long U,
                             long G)
{
    const long n = X * Y * B;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        const long x = i % X, b = i / (X * Y);
        const long s = b * nxb + x / W;
        if (rank_split(s, C, U, G)) {
            float2 o = out[i];
            const float2 t = plane1[i];
            out[i] = float2{o.x + t.x, o.y + t.y};
        }
    }
}

// CG update with the two-plane Ap: x += alpha p ; r -= alpha Ap ; <r, r> partial
template<int W>
__global__ void k_cg_update_rank(CgDev* st, int it, cfloat* x, cfloat* r, const cfloat* p, const cfloat* ap,
                                 const cfloat* ap1, long X, long Y, long B, long nxb, long C, long U, long G,
                                 unsigned* errflags)
{
    __shared__ float s_alpha;
    if (threadIdx.x == 0)
        s_alpha = cg_alpha(st, it, errflags);
    __syncthreads();
    const float al = s_alpha;
    if (!(al > 0.f))
        return;
    const long n = X * Y * B;
    double2 part{0, 0};
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        const long xq = i % X, b = i / (X * Y);
        float2 av = ap[i];
        if (rank_split(b * nxb + xq / W, C, U, G)) {
            const float2 t = ap1[i];
            av.x += t.x;
            av.y += t.y;
        }
        float2 pv = p[i], xv = x[i], rv = r[i];
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

PFN_cuTensorMapEncodeTiled_v12000 rank_encode_fn()
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

// Geometry of one rank launch (shared by the kernel, the merge and the CG update)
struct RankPlan {
    int N1 = 0, N2 = 0, W = 0;
    long nxb = 0, strips = 0, units = 0;
    int G = 0;
    bool ok = false;
};

RankPlan rank_plan(const SenseGeom& g, const cfloat* coils)
{
    RankPlan r;
    int n1 = 0, n2 = 0;
    switch (g.Y) {
    case 128: n1 = 8; n2 = 16; break;
    case 256: n1 = 16; n2 = 16; break;
    case 320: n1 = 16; n2 = 20; break;
    case 368: n1 = 16; n2 = 23; break;
    case 512: n1 = 16; n2 = 32; break;
    case 640: n1 = 16; n2 = 40; break;
    default: return r;
    }
    if (g.M != 1 || g.pat_x != 1 || g.pat_c != 1 || (g.X & 1) || (reinterpret_cast<uintptr_t>(coils) & 15))
        return r;
    r.N1 = n1;
    r.N2 = n2;
    r.W = n2 <= 24 ? 8 : 4;
    r.nxb = (g.X + r.W - 1) / r.W;
    r.strips = r.nxb * g.B;
    r.units = r.strips * g.C;
    r.G = int(std::min<long>(g_rank_ctas > 0 ? g_rank_ctas : 2L * ctx().sm_count, r.strips));
    r.ok = g.Y * g.C * g.B < (1L << 31);
    return r;
}

template<int N1, int N2>
void launch_rank_t(RankArgs a, const cfloat* coils, const SenseGeom& g)
{
    using Cfg = RankCfg<N1, N2>;
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(2 * g.X), cuuint64_t(g.Y * g.C * g.B)};
    cuuint64_t strides[1] = {cuuint64_t(2 * g.X) * 4};
    cuuint32_t box[2] = {cuuint32_t(2 * Cfg::W), cuuint32_t(Cfg::BOXR)};
    cuuint32_t es[2] = {1, 1};
    CUresult res = rank_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<cfloat*>(coils), dims, strides,
                                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(coils) failed: " + std::to_string(int(res)));
    auto kern = k_normal_rank<N1, N2>;
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM)));
        attr = true;
    }
    const double xyb = double(g.X) * g.Y * g.B;
    const double work = 8.0 * xyb * (g.C + (a.mode == 1 ? 4 : 2));
    ProfScope prof(a.mode == 1 ? "sense_normal_y_cg" : "sense_normal_y", work);
    kern<<<a.G, Cfg::NT, Cfg::SMEM, ctx().stream>>>(a, m);
    KERNEL_CHECK();
}

void launch_rank(const RankPlan& rp, RankArgs a, const cfloat* coils, const SenseGeom& g)
{
    a.tw = fast_twiddles(rp.N1, rp.N2);
    a.X = g.X;
    a.C = g.C;
    a.B = g.B;
    a.nxb = rp.nxb;
    a.units = rp.units;
    a.G = rp.G;
    switch (g.Y) {
    case 128: launch_rank_t<8, 16>(a, coils, g); break;
    case 256: launch_rank_t<16, 16>(a, coils, g); break;
    case 320: launch_rank_t<16, 20>(a, coils, g); break;
    case 368: launch_rank_t<16, 23>(a, coils, g); break;
    case 512: launch_rank_t<16, 32>(a, coils, g); break;
    case 640: launch_rank_t<16, 40>(a, coils, g); break;
    default: throw Error("rank A^H A: unsupported Y");
    }
}
