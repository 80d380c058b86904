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

#include <type_traits>

bool g_cg_defer_x = true; // CG: keep every p, update r only per iteration, sum x once
long g_rank_ctas = 0; // 0: 2 per SM (tests force fewer to exercise split strips)
bool g_sense_ws = true; // warp-specialised kernel (sense_ws.cuh), one CTA per SM
// programmatic dependent launch of the CG loop's A^H A and update kernels: each
// kernel's launch and CTA start overlap the previous kernel's tail
bool g_cg_pdl = true;

// fused CG update inside the ws kernel (one launch per CG iteration; grid barrier):
// 0 off, 1 on, 2 on with a cooperative launch
int g_cg_fuse = 1;

// kernel launch on the library stream with optional programmatic serialisation
// (pdl) and cooperative residency (coop: every CTA co-resident, or the launch fails)
template<class... KArgs, class... Args>
void launch_ex(bool pdl, bool coop, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx().stream;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl && g_pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    if (coop) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na++].val.cooperative = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}
template<class... KArgs, class... Args>
void launch_maybe_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args)
{
    launch_ex(pdl, false, kern, grid, block, smem, std::forward<Args>(args)...);
}
bool g_rank_rr = true;
int g_rank_vh = 9;     // ws kernel: segment overhead ~2.25 units (RANK_VQ = 4; 0: equal unit counts)  // whole strips round robin for 32-B strips (RankPlan::rr)

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
#ifndef RANK_W
#define RANK_W 8
#endif
    static constexpr int W = N2 <= 24 ? RANK_W : 4;        // columns per strip
    static constexpr int NT = ((W * N2 + 31) / 32) * 32;   // threads (w, j)
    static constexpr int N2P = N2 + (N2 & 1);              // S / twiddle row pitch (even: unguarded halves)
    static constexpr int JH = N2P / 2;                     // j per half-row (stage-B thread pairs)
    static constexpr int TMAX = W == 8 ? 32 : 24;          // terms with precomputed twiddle rows
    static constexpr int NBOX = rank_nbox(Y);              // TMA boxes per coil slice (rows <= 256)
    static constexpr int BOXR = Y / NBOX;
    static constexpr size_t SLOT = size_t(Y) * W;          // float2 per ring slot / S / xs
    static constexpr size_t SSLOT = size_t(N1) * N2P * W;  // S (row pitch N2P)
    // dynamic smem (float2): ring[2][SLOT] | S[SSLOT] | xs[SLOT] | ttw[TMAX*N2P]
    static constexpr size_t SMEM = sizeof(float2) * (3 * SLOT + SSLOT + TMAX * N2P);
    // (W = 4 at 2 CTAs/SM, 255 registers, no spills: 240 vs 239 us at 512^2 x 32 x 4 -- no gain)
    static constexpr int MINB = 4 * (SMEM + 4096) <= 228 * 1024 ? 4 : 3 * (SMEM + 4096) <= 228 * 1024 ? 3
                              : 2 * (SMEM + 4096) <= 228 * 1024 ? 2 : 1;
    static_assert(Y % NBOX == 0, "TMA box rows must tile Y");
};

struct RankArgs {
    cfloat* out;          // plane 0 (mode 0: the result; mode 1: Ap)
    cfloat* out1;         // planes 1.. (strips shared by several CTAs), plane stride pstride
    long pstride;
    const cfloat* x;      // mode 0: input image; mode 1: r
    cfloat* p;            // mode 1: previous search direction
    cfloat* p_out;        // mode 1: new search direction (== x source at it 0)
    const cfloat* pattern;
    const cfloat* lam;    // device lambda, or nullptr: lamv
    float2 lamv;
    const float2* tw;     // exp(-2 pi i m / Y), m < Y
    long X, C, B;
    long nxb;             // strips per item
    long units;           // strips * C
    int G;                // CTAs
    int rr;               // 1: CTA g owns whole strips g, g + G, g + 2G, ... (no split strips)
    int vh;               // contiguous ranges: per-strip overhead weight (rank_ubegin; 0: equal unit counts)
    PatStr ps;
    int mode, it;
    CgDev* cg;
    unsigned* errflags;
    unsigned char* split; // k_rank_plan: split flag per strip (planes sharing it); ws fused update: read
    long strips;
    cfloat* r_upd;        // mode 1, k_normal_ws: fused CG update r -= alpha Ap (cg_defer_x path), or nullptr
    int upd_rows, upd_Y, upd_wshift;
    int check_pattern;    // k_rank_plan: also run the binary-pattern check
};

// Contiguous unit ranges.  vh = 0: [floor(U g / G), floor(U (g+1) / G)).
// vh > 0 (k_normal_ws): ranges of equal *cost*, where a unit weighs RANK_VQ and
// every strip an extra vh for its segment open + epilogue (x strip load, store,
// <p, Ap>): unit u = (s, c) sits at virtual position s (C RANK_VQ + vh) + vh +
// c RANK_VQ of V = strips (C RANK_VQ + vh), and CTA g owns the units whose
// position lies in [floor(V g / G), floor(V (g+1) / G)).  Equal unit counts
// left the CTAs that open one segment more ~6% behind the others, which the
// fused CG update's grid barrier turns into idle time on every CTA.
constexpr long RANK_VQ = 4;
__host__ __device__ __forceinline__ long rank_vpos(long u, long C, long vh)
{
    const long s = u / C;
    return s * (C * RANK_VQ + vh) + vh + (u - s * C) * RANK_VQ;
}
// CTA owning unit u
__host__ __device__ __forceinline__ long rank_owner(long u, long C, long U, long G, long vh)
{
    if (vh == 0)
        return ((u + 1) * G + U - 1) / U - 1;
    const long V = (U / C) * (C * RANK_VQ + vh), p = rank_vpos(u, C, vh);
    return ((p + 1) * G + V - 1) / V - 1;
}
// first unit of CTA g (g = G: U)
__host__ __device__ __forceinline__ long rank_ubegin(long g, long C, long U, long G, long vh)
{
    if (vh == 0)
        return U * g / G;
    const long SW = C * RANK_VQ + vh, v = (U / C) * SW * g / G;
    const long s = v / SW, o = v - s * SW;
    return s * C + (o <= vh ? 0 : (o - vh + RANK_VQ - 1) / RANK_VQ);
}
__host__ __device__ __forceinline__ bool rank_split(long s, long C, long U, long G, long vh)
{
    return rank_owner(s * C, C, U, G, vh) != rank_owner(s * C + C - 1, C, U, G, vh);
}
// number of CTAs (= Ap planes) sharing strip s (a CTA with an empty range never
// falls inside a strip's span: its range lies in the gap before a strip's first unit)
__host__ __device__ __forceinline__ int rank_planes(long s, long C, long U, long G, long vh)
{
    return int(rank_owner(s * C + C - 1, C, U, G, vh) - rank_owner(s * C, C, U, G, vh) + 1);
}
// destination of a segment's partial: plane 0 = out, plane k >= 1 = out1 + (k - 1) * pstride
__device__ __forceinline__ cfloat* rank_plane_dst(const RankArgs& a, int strip, int cta)
{
    if (a.rr)
        return a.out;
    const int k = cta - int(rank_owner(long(strip) * a.C, a.C, a.units, a.G, a.vh));
    return k == 0 ? a.out : a.out1 + long(k - 1) * a.pstride;
}

// Per-CTA row plan (shared memory), rebuilt when the item's pattern changes.
// Every non-identity row is a term row (min(#{p != 0}, #{p != 1}) <= N2 / 2
// terms); the first TMAX terms have precomputed twiddle rows (ttw), later
// ones index the Y-point table on the fly.
template<int N1, int N2>
struct RankPlanSm {
    static constexpr int TTOT = N1 * (N2 / 2);
    int nwork, T;
    int work_k1[N1];   // non-identity rows, fewest terms first
    int mode[N1];      // 0 identity, 1 identity + terms, 2 terms only
    int nt[N1], off[N1], key[N1];
    int tk[TTOT];
    float2 coef[TTOT];
};

// all threads; ends with a barrier
template<int N1, int N2>
__device__ void rank_build_plan(RankPlanSm<N1, N2>& pl, const RankArgs& a, int b, float2* ttw, const float2* stw)
{
    using Cfg = RankCfg<N1, N2>;
    constexpr int Y = Cfg::Y, NT = Cfg::NT, TMAX = Cfg::TMAX;
    constexpr float invN2 = 1.f / float(N2);
    const int tid = threadIdx.x;
    const long pb = long(b) * a.ps.sb;
    if (tid < N1) {
        int nz = 0, n1 = 0;
        for (int k2 = 0; k2 < N2; k2++) {
            const float2 pv = a.pattern[(tid + N1 * k2) * a.ps.sy + pb];
            nz += (pv.x != 0.f || pv.y != 0.f);
            n1 += (pv.x != 1.f || pv.y != 0.f);
        }
        const int n = min(nz, n1);
        pl.nt[tid] = n;
        pl.mode[tid] = n == 0 ? (n1 == 0 ? 0 : 2) : (nz <= n1 ? 2 : 1);
        pl.key[tid] = n1 == 0 ? -1 : n; // identity rows sort first and are skipped
    }
    __syncthreads();
    if (tid < N1) {
        int off = 0, rank = 0, nid = 0, T = 0;
        const int k = pl.key[tid];
        for (int r = 0; r < N1; r++) {
            off += r < tid ? pl.nt[r] : 0;
            T += pl.nt[r];
            const int kr = pl.key[r];
            rank += (kr < k) || (kr == k && r < tid);
            nid += kr < 0;
        }
        pl.off[tid] = off;
        if (k >= 0)
            pl.work_k1[rank - nid] = tid;
        if (tid == 0) {
            pl.nwork = N1 - nid;
            pl.T = T;
        }
        const int md = pl.mode[tid];
        if (md != 0) {
            const float bb = md == 1 ? 1.f : 0.f;
            int t = off;
            for (int k2 = 0; k2 < N2; k2++) {
                const float2 pv = a.pattern[(tid + N1 * k2) * a.ps.sy + pb];
                if (pv.x != bb || pv.y != 0.f) {
                    pl.tk[t] = tid + N1 * k2;
                    pl.coef[t] = float2{(pv.x - bb) * invN2, pv.y * invN2};
                    t++;
                }
            }
        }
    }
    __syncthreads();
    constexpr int N2P = Cfg::N2P;
    for (int e = tid; e < min(pl.T, TMAX) * N2P; e += NT) {
        const int t = e / N2P, jj = e % N2P;
        ttw[e] = jj < N2 ? stw[(jj * pl.tk[t]) % Y] : float2{0.f, 0.f}; // zero pad: no contribution
    }
    __syncthreads();
}

// Global plan record per pattern item: [RankPlanSm | ttw[TMAX * N2]], 16-B multiple.
template<int N1, int N2>
struct RankPlanRec {
    static constexpr size_t PL = (sizeof(RankPlanSm<N1, N2>) + 15) & ~size_t(15);
    static constexpr size_t BYTES = PL + sizeof(float2) * RankCfg<N1, N2>::TMAX * RankCfg<N1, N2>::N2P;
};

// one CTA per pattern item (grid = 1 for a broadcast pattern)
template<int N1, int N2>
__global__ void __launch_bounds__(RankCfg<N1, N2>::NT) k_rank_plan(RankArgs a, unsigned char* plans)
{
    MDNN_PDL_ENTRY();
    unsigned char* rec = plans + RankPlanRec<N1, N2>::BYTES * blockIdx.x;
    rank_build_plan<N1, N2>(*reinterpret_cast<RankPlanSm<N1, N2>*>(rec), a, int(blockIdx.x),
                            reinterpret_cast<float2*>(rec + RankPlanRec<N1, N2>::PL), a.tw);
    constexpr int NT = RankCfg<N1, N2>::NT;
    if (a.check_pattern) {
        // recon.hpp:67-77 on this item's pattern column (the plan reads exactly these
        // values), folded into the plan pass: ERRF_PATTERN is raised at the call's sync
        const long pb = long(blockIdx.x) * a.ps.sb;
        bool bad = false;
        for (int y = threadIdx.x; y < N1 * N2; y += NT) {
            const float2 pv = a.pattern[y * a.ps.sy + pb];
            bad |= pv.y != 0.f || (pv.x != 0.f && pv.x != 1.f);
        }
        if (__syncthreads_or(bad) && threadIdx.x == 0)
            atomicOr(a.errflags, unsigned(ERRF_PATTERN));
    }
    // split flag of every strip (planes sharing it; 1 for round-robin strips)
    for (long s = blockIdx.x * long(NT) + threadIdx.x; s < a.strips; s += long(gridDim.x) * NT)
        a.split[s] = a.rr ? 1 : (unsigned char)rank_planes(s, a.C, a.units, a.G, a.vh);
}

template<int N1, int N2>
__global__ void __launch_bounds__(RankCfg<N1, N2>::NT, RankCfg<N1, N2>::MINB)
    k_normal_rank(RankArgs a, const __grid_constant__ CUtensorMap tmap, const unsigned char* __restrict__ plans)
{
    MDNN_PDL_ENTRY();
    using namespace fftd;
    using Cfg = RankCfg<N1, N2>;
    constexpr int Y = Cfg::Y, W = Cfg::W, JH = Cfg::JH, TMAX = Cfg::TMAX, N2P = Cfg::N2P;
    static_assert(JH % 2 == 0, "stage-B half rows are read as float4 pairs");
    constexpr int NT = Cfg::NT; // threads of this CTA
    constexpr int NQ = N1;      // q points per thread
    extern __shared__ __align__(128) float2 rank_smem[];
    float2* ring = rank_smem;
    float2* S = ring + 2 * Cfg::SLOT;
    float2* xs = S + Cfg::SSLOT;
    float2* ttw = xs + Cfg::SLOT;
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ float s_beta;
    __shared__ float2 s_lam;
    __shared__ __align__(16) RankPlanSm<N1, N2> pl;

    const int tid = threadIdx.x;
    const int w = tid % W, j0 = tid / W;
    const bool active = j0 < N2;
    const int j = active ? j0 : N2 - 1;
    const int C = int(a.C), nxb = int(a.nxb);
    const int U = int(a.units);
    // contiguous unit ranges, or (a.rr) whole strips g, g + G, ...: the CTAs then
    // read neighbouring strips of the same coil at the same time, so the 128-B
    // DRAM lines of narrow (32-B) strips are fetched once
    const int u_begin = a.rr ? int(blockIdx.x) * C : int(long(U) * blockIdx.x / a.G);
    const int u_end = int(long(U) * (blockIdx.x + 1) / a.G);
    const int nstrips_rr = a.rr ? int((U / C - 1 - int(blockIdx.x)) / a.G + 1) : 0;
    const int n = a.rr ? nstrips_rr * C : u_end - u_begin;
    // global unit of local unit i
    auto unit_of = [&](int i) { return a.rr ? (int(blockIdx.x) + (i / C) * a.G) * C + i % C : u_begin + i; };

    auto issue = [&](int u, int slot) { // TMA of unit u's coil slice into ring slot
        const int s = u / C, c = u - s * C;
        const int b = s / nxb, xblk = s - b * nxb;
        const int row0 = Y * (c + C * b);
        sm100::mbar_arrive_expect_tx(&s_bar[slot], uint32_t(Cfg::SLOT * sizeof(float2)));
#pragma unroll
        for (int k = 0; k < Cfg::NBOX; k++)
            sm100::tma_load_2d(ring + slot * Cfg::SLOT + k * Cfg::BOXR * W, &tmap, &s_bar[slot], 2 * W * xblk,
                               row0 + k * Cfg::BOXR);
    };
    if (tid == 0) {
        sm100::prefetch_tmap(&tmap);
        sm100::mbar_init(&s_bar[0], 1);
        sm100::mbar_init(&s_bar[1], 1);
        sm100::fence_barrier_init();
        for (int i = 0; i < n && i < 2; i++)
            issue(unit_of(i), i);
        s_beta = a.mode == 1 ? cg_prologue(a.cg, a.it, a.errflags) : 0.f;
        s_lam = a.lam ? a.lam[0] : a.lamv;
    }
    if constexpr (N2P != N2) { // pad column of S stays zero (read by stage B, never by A/C)
        for (int e = tid; e < N1 * W; e += NT)
            S[((e / W) * N2P + N2) * W + e % W] = float2{0.f, 0.f};
    }
    __syncthreads();
    const float beta = s_beta;
    if (a.mode == 1 && beta < 0.f) {
        // CG already stopped: drain the TMA ring before exiting
        for (int i = 0; i < n && i < 2; i++)
            sm100::mbar_wait(&s_bar[i], 0);
        return;
    }
    const bool upd = a.mode == 1 && a.it > 0;
    const float2 lam = s_lam;
    constexpr float invN1 = 1.f / float(N1);

    int plan_b = -1;
    int n_items = 0, my_h = 0, my_k1 = 0, my_ww = 0, my_md = 0, my_nt = 0, my_off = 0;
    bool my_item = false;
    double2 part{0, 0};
    float2 acc[NQ], cv[NQ];
    int seg_s = u_begin / C;           // strip of the open segment
    int c_cur = u_begin - seg_s * C;   // coil of unit i
    bool seg_first = c_cur == 0;

    // iteration i: [C(unit i-1) (+ epilogue) ; A(unit i)] | barrier | B(unit i) | barrier
    for (int i = 0; i <= n; i++) {
        const bool opens = i < n && (i == 0 || c_cur == 0);
        if (i >= 1) {
            // ---- C(i-1): inverse DFT over k1, conj-coil accumulate
            float2 v[NQ];
#pragma unroll
            for (int m = 0; m < NQ; m++)
                v[m] = S[(m * N2P + j) * W + w];
            dft_reg<N1, +1>(v);
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                const float2 t = cmulc(v[q], cv[q]);
                acc[q].x += t.x;
                acc[q].y += t.y;
            }
            if (i == n || c_cur == 0) {
                // ---- segment epilogue: 1/N1, + lambda x (plane 0), store, <p, Ap>
                const int b = seg_s / nxb, xx = (seg_s - b * nxb) * W + w;
                const long img_base = xx + a.X * Y * long(b);
                cfloat* dst = rank_plane_dst(a, seg_s, blockIdx.x);
#pragma unroll
                for (int q = 0; q < NQ; q++) {
                    const int y = j + N2 * q;
                    const float2 xv = xs[y * W + w];
                    float2 o{acc[q].x * invN1, acc[q].y * invN1};
                    if (seg_first) {
                        const float2 lx = cmul(xv, lam);
                        o.x += lx.x;
                        o.y += lx.y;
                    }
                    if (active && xx < a.X) {
                        dst[img_base + a.X * y] = o;
                        part.x += double(xv.x) * o.x + double(xv.y) * o.y;
                        part.y += double(xv.y) * o.x - double(xv.x) * o.y;
                    }
                }
            }
        }
        if (i < n) {
            if (opens) {
                if (i > 0)
                    seg_s += a.rr ? a.G : 1;
                seg_first = c_cur == 0;
                const int b = seg_s / nxb;
                if (b != plan_b && (plan_b < 0 || a.ps.sb != 0)) {
                    // B(i-1) is done (barrier); C does not read the plan
                    using Rec = RankPlanRec<N1, N2>;
                    const int4* src = reinterpret_cast<const int4*>(plans + Rec::BYTES * (a.ps.sb != 0 ? b : 0));
                    int4* dpl = reinterpret_cast<int4*>(&pl);
                    for (int e = tid; e < int(Rec::PL / 16); e += NT)
                        dpl[e] = src[e];
                    const int4* src2 = reinterpret_cast<const int4*>(reinterpret_cast<const unsigned char*>(src) + Rec::PL);
                    int4* dtw = reinterpret_cast<int4*>(ttw);
                    for (int e = tid; e < int(TMAX * N2P * sizeof(float2) / 16); e += NT)
                        dtw[e] = src2[e];
                    __syncthreads();
                    plan_b = b;
                    // this thread's first stage-B item (the loop handles any others)
                    const int it0 = tid, nitems = pl.nwork * W * 2;
                    my_item = it0 < nitems;
                    my_h = it0 & 1;
                    my_k1 = my_item ? pl.work_k1[(it0 >> 1) / W] : 0;
                    my_ww = (it0 >> 1) % W;
                    my_md = pl.mode[my_k1];
                    my_nt = pl.nt[my_k1];
                    my_off = pl.off[my_k1];
                    n_items = nitems;
                }
                // ---- open a segment: x (or p = r + beta p_prev) strip -> xs
                const int xx = (seg_s - b * nxb) * W + w;
                const bool colok = active && xx < a.X;
                const long img_base = xx + a.X * Y * long(b);
                float2 v[NQ], pv[NQ];
                const float2* src = a.mode == 0 ? a.x : (a.it == 0 ? a.p_out : a.x);
#pragma unroll
                for (int q = 0; q < NQ; q++) {
                    const long gi = img_base + a.X * (j + N2 * q);
                    v[q] = colok ? src[gi] : float2{0.f, 0.f};
                    pv[q] = (colok && upd) ? a.p[gi] : float2{0.f, 0.f};
                }
#pragma unroll
                for (int q = 0; q < NQ; q++) {
                    const int y = j + N2 * q;
                    if (upd) {
                        v[q] = float2{v[q].x + beta * pv[q].x, v[q].y + beta * pv[q].y};
                        if (seg_first && colok)
                            a.p_out[img_base + a.X * y] = v[q];
                    }
                    if (active)
                        xs[y * W + w] = v[q];
                    acc[q] = float2{0.f, 0.f};
                }
            }
            // ---- A(i): coil multiply, DFT over q -> S (untwiddled)
            const int slot = i & 1;
            const float2* cs = ring + slot * Cfg::SLOT;
            sm100::mbar_wait(&s_bar[slot], uint32_t((i >> 1) & 1));
            float2 v[NQ];
            // padding threads (j clamped) compute on valid rows; their results are never stored
            const float2* csp = cs + j * W + w;
            const float2* xsp = xs + j * W + w;
#pragma unroll
            for (int q = 0; q < NQ; q++)
                cv[q] = csp[N2 * W * q];
#pragma unroll
            for (int q = 0; q < NQ; q++)
                v[q] = cmul(cv[q], xsp[N2 * W * q]);
            dft_reg<N1, -1>(v);
            if (active) {
#pragma unroll
                for (int m = 0; m < NQ; m++)
                    S[(m * N2P + j) * W + w] = v[m];
            }
        }
        __syncthreads();
        if (i >= n)
            break;
        c_cur = c_cur + 1 == C ? 0 : c_cur + 1;
        // slot i & 1 is consumed (coils now live in registers): refill it
        if (tid == 0 && i + 2 < n)
            issue(unit_of(i + 2), i & 1);
        // ---- B(i): per non-identity row, a thread pair (h = j half) per column:
        //   r = b A + sum_t coef_t (sum_j A_j w_t[j]) conj(w_t[j])
        for (int item = tid; item < n_items; item += NT) {
            int h = my_h, ww = my_ww, k1 = my_k1, md = my_md, nt = my_nt, off = my_off;
            if (item != tid) {
                h = item & 1;
                ww = (item >> 1) % W;
                k1 = pl.work_k1[(item >> 1) / W];
                md = pl.mode[k1];
                nt = pl.nt[k1];
                off = pl.off[k1];
            }
            float2* row = S + k1 * N2P * W + ww;
            const unsigned pmask = 3u << ((tid & 31) & ~1);
            const int jb = h * JH;
            float2 uu[JH];
#pragma unroll
            for (int jj = 0; jj < JH; jj++)
                uu[jj] = row[(jb + jj) * W]; // pad column: finite junk times a zero twiddle
            if (nt <= 2 && off + nt <= TMAX) {
                // common case (<= 2 terms, precomputed twiddle rows): both dot
                // products in one pass (4 independent chains), then in place
                const bool two = nt == 2;
                const float2* t0 = ttw + off * N2P + jb;
                const float2* t1 = ttw + (two ? off + 1 : off) * N2P + jb;
                float2 a0{0.f, 0.f}, a1{0.f, 0.f};
                const float4* t0v = reinterpret_cast<const float4*>(t0); // 16-B aligned: N2P, jb even
                const float4* t1v = reinterpret_cast<const float4*>(t1);
#pragma unroll
                for (int jj = 0; jj < JH; jj++) {
                    {
                        const float4 q0 = t0v[jj >> 1], q1 = t1v[jj >> 1];
                        const float2 p0 = (jj & 1) ? float2{q0.z, q0.w} : float2{q0.x, q0.y};
                        const float2 p1 = (jj & 1) ? float2{q1.z, q1.w} : float2{q1.x, q1.y};
                        a0.x = fmaf(uu[jj].x, p0.x, a0.x);
                        a0.y = fmaf(uu[jj].x, p0.y, a0.y);
                        a1.x = fmaf(uu[jj].x, p1.x, a1.x);
                        a1.y = fmaf(uu[jj].x, p1.y, a1.y);
                        a0.x = fmaf(-uu[jj].y, p0.y, a0.x);
                        a0.y = fmaf(uu[jj].y, p0.x, a0.y);
                        a1.x = fmaf(-uu[jj].y, p1.y, a1.x);
                        a1.y = fmaf(uu[jj].y, p1.x, a1.y);
                    }
                }
                a0.x += __shfl_xor_sync(pmask, a0.x, 1);
                a0.y += __shfl_xor_sync(pmask, a0.y, 1);
                a1.x += __shfl_xor_sync(pmask, a1.x, 1);
                a1.y += __shfl_xor_sync(pmask, a1.y, 1);
                a0 = nt > 0 ? cmul(a0, pl.coef[off]) : float2{0.f, 0.f};
                a1 = two ? cmul(a1, pl.coef[off + 1]) : float2{0.f, 0.f};
                auto scatter = [&](auto keep) { // u = b u + d conj(tw), b as a compile-time flag
#pragma unroll
                    for (int jj = 0; jj < JH; jj++) {
                        const float4 q0 = t0v[jj >> 1], q1 = t1v[jj >> 1];
                        const float2 p0 = (jj & 1) ? float2{q0.z, q0.w} : float2{q0.x, q0.y};
                        const float2 p1 = (jj & 1) ? float2{q1.z, q1.w} : float2{q1.x, q1.y};
                        float2 r;
                        if constexpr (decltype(keep)::value) {
                            r.x = fmaf(a0.x, p0.x, uu[jj].x);
                            r.y = fmaf(a0.y, p0.x, uu[jj].y);
                        } else {
                            r.x = a0.x * p0.x;
                            r.y = a0.y * p0.x;
                        }
                        r.x = fmaf(a0.y, p0.y, r.x);
                        r.y = fmaf(-a0.x, p0.y, r.y);
                        r.x = fmaf(a1.x, p1.x, r.x);
                        r.y = fmaf(a1.y, p1.x, r.y);
                        r.x = fmaf(a1.y, p1.y, r.x);
                        r.y = fmaf(-a1.x, p1.y, r.y);
                        row[(jb + jj) * W] = r;
                    }
                };
                if (md == 1)
                    scatter(std::true_type{});
                else
                    scatter(std::false_type{});
            } else {
                // general rows: any number of terms, twiddles indexed on the fly
                float2 rr[JH];
#pragma unroll
                for (int jj = 0; jj < JH; jj++)
                    rr[jj] = md == 1 ? uu[jj] : float2{0.f, 0.f};
                for (int t = off; t < off + nt; t++) {
                    const int k = pl.tk[t];
                    const int m00 = (jb * k) % Y;
                    int m0 = m00;
                    float2 e0{0.f, 0.f};
#pragma unroll
                    for (int jj = 0; jj < JH; jj++) {
                        if (jb + jj < N2) {
                            const float2 tv = __ldg(&a.tw[m0]);
                            e0.x = fmaf(uu[jj].x, tv.x, e0.x);
                            e0.y = fmaf(uu[jj].x, tv.y, e0.y);
                            e0.x = fmaf(-uu[jj].y, tv.y, e0.x);
                            e0.y = fmaf(uu[jj].y, tv.x, e0.y);
                        }
                        m0 += k;
                        m0 -= m0 >= Y ? Y : 0;
                    }
                    e0.x += __shfl_xor_sync(pmask, e0.x, 1);
                    e0.y += __shfl_xor_sync(pmask, e0.y, 1);
                    e0 = cmul(e0, pl.coef[t]);
                    m0 = m00;
#pragma unroll
                    for (int jj = 0; jj < JH; jj++) {
                        if (jb + jj < N2) {
                            const float2 tv = __ldg(&a.tw[m0]);
                            rr[jj].x = fmaf(e0.x, tv.x, rr[jj].x);
                            rr[jj].y = fmaf(e0.y, tv.x, rr[jj].y);
                            rr[jj].x = fmaf(e0.y, tv.y, rr[jj].x);
                            rr[jj].y = fmaf(-e0.x, tv.y, rr[jj].y);
                        }
                        m0 += k;
                        m0 -= m0 >= Y ? Y : 0;
                    }
                }
#pragma unroll
                for (int jj = 0; jj < JH; jj++)
                    if (jb + jj < N2)
                        row[(jb + jj) * W] = rr[jj];
            }
        }
        __syncthreads();
    }
    if (a.mode == 1) {
        part = block_sum2(part);
        publish_partial(a.cg->part_pap, &a.cg->pap_sum, &a.cg->cnt_pap, part);
    }
}

// out (+)= plane 1 for pixels of split strips (mode 0 result assembly)
__global__ void __launch_bounds__(256) k_rank_merge(cfloat* out, const cfloat* plane1,
                                                    const unsigned char* __restrict__ split, int X, int rows, int Y,
                                                    int nxb, int wshift, long pstride)
{
    MDNN_PDL_ENTRY();
    const int X2 = X >> 1;
    for (int row = blockIdx.x; row < rows; row += gridDim.x) {
        const int sb = (row / Y) * nxb;
        const long base = long(row) * X2;
        for (int xp = threadIdx.x; xp < X2; xp += blockDim.x) {
            const int np = split[sb + ((2 * xp) >> wshift)];
            if (np <= 1)
                continue;
            const long i = base + xp;
            float4 o = reinterpret_cast<float4*>(out)[i];
            for (int k = 1; k < np; k++) { // fixed plane order: bitwise deterministic
                const float4 t = reinterpret_cast<const float4*>(plane1)[i + long(k - 1) * (pstride / 2)];
                o.x += t.x;
                o.y += t.y;
                o.z += t.z;
                o.w += t.w;
            }
            reinterpret_cast<float4*>(out)[i] = o;
        }
    }
}

// CG update with the two-plane Ap: x += alpha p ; r -= alpha Ap ; <r, r> partial.
// Blocks walk whole image rows (no per-element division), two complex per
// thread (float4); split[s] flags strips whose Ap has a plane-1 part.
__global__ void __launch_bounds__(512) k_cg_update_rank(CgDev* st, int it, cfloat* __restrict__ x,
                                                        cfloat* __restrict__ r, const cfloat* __restrict__ p,
                                                        const cfloat* __restrict__ ap,
                                                        const cfloat* __restrict__ ap1,
                                                        const unsigned char* __restrict__ split, int X, int rows,
                                                        int Y, int nxb, int wshift, long pstride, unsigned* errflags)
{
    MDNN_PDL_ENTRY();
    __shared__ float s_alpha;
    if (threadIdx.x == 0)
        s_alpha = cg_alpha(st, it, errflags);
    const int X2 = X >> 1;
    const int npair = rows * X2;
    const int stride = gridDim.x * blockDim.x;
    const float4* ap4 = reinterpret_cast<const float4*>(ap);
    const float4* ap14 = reinterpret_cast<const float4*>(ap1);
    const float4* p4 = reinterpret_cast<const float4*>(p);
    float4* x4 = reinterpret_cast<float4*>(x);
    float4* r4 = reinterpret_cast<float4*>(r);
    constexpr int U = 2; // element pairs in flight per thread
    float4 av[U], t1[U], pv[U], xv[U], rv[U];
    int sp[U];
    bool ok[U];
    int i0 = blockIdx.x * blockDim.x + threadIdx.x;
    auto load = [&](int base) {
#pragma unroll
        for (int k = 0; k < U; k++) {
            const int i = base + k * stride;
            ok[k] = i < npair;
            const int ii = ok[k] ? i : 0;
            av[k] = ap4[ii];
            t1[k] = ap14[ii]; // junk outside split strips: not used there
            pv[k] = p4[ii];
            xv[k] = x4[ii];
            rv[k] = r4[ii];
            const int row = ii / X2, xp = ii - row * X2;
            sp[k] = split[(row / Y) * nxb + ((2 * xp) >> wshift)];
        }
    };
    load(i0);
    __syncthreads();
    const float al = s_alpha;
    if (!(al > 0.f))
        return;
    double2 part{0, 0};
    while (true) {
#pragma unroll
        for (int k = 0; k < U; k++) {
            if (!ok[k])
                continue;
            float4 a = av[k];
            if (sp[k] > 1) {
                a.x += t1[k].x;
                a.y += t1[k].y;
                a.z += t1[k].z;
                a.w += t1[k].w;
                for (int pk = 2; pk < sp[k]; pk++) { // rare: strips shared by 3+ CTAs
                    const float4 t = ap14[i0 + k * stride + long(pk - 1) * (pstride / 2)];
                    a.x += t.x;
                    a.y += t.y;
                    a.z += t.z;
                    a.w += t.w;
                }
            }
            float4 xx = xv[k], rr = rv[k];
            xx.x += al * pv[k].x;
            xx.y += al * pv[k].y;
            xx.z += al * pv[k].z;
            xx.w += al * pv[k].w;
            rr.x += -al * a.x;
            rr.y += -al * a.y;
            rr.z += -al * a.z;
            rr.w += -al * a.w;
            const int i = i0 + k * stride;
            x4[i] = xx;
            r4[i] = rr;
            part.x += double(rr.x) * rr.x + double(rr.y) * rr.y;
            part.x += double(rr.z) * rr.z + double(rr.w) * rr.w;
        }
        i0 += U * stride;
        if (i0 >= npair)
            break;
        load(i0);
    }
    part = block_sum2(part);
    publish_partial(st->part_rr, &st->rr_sum, &st->cnt_rr, part);
}

// r-only CG update (x deferred): r -= alpha Ap ; <r, r> partial.  With every
// search direction p_it kept, x = sum_it alpha_it p_it is formed once after the
// loop by k_cg_x_sum in the same fma order as the per-iteration update (bitwise
// identical), and each iteration streams 3 arrays instead of 5.
// r -= alpha Ap (Ap = plane 0 + the planes of split strips) over the pixel pairs
// i0, i0 + stride, ... ; returns this thread's <r, r> partial.  L2 loads: in the
// fused form (k_normal_ws) Ap was stored by other CTAs of the same grid.
template<int U>
__device__ __forceinline__ double2 cg_r_update_pairs(float al, cfloat* __restrict__ r, const cfloat* __restrict__ ap,
                                                     const cfloat* __restrict__ ap1,
                                                     const unsigned char* __restrict__ split, int X, int rows, int Y,
                                                     int nxb, int wshift, long pstride, int i0, int stride)
{
    const int X2 = X >> 1;
    const int npair = rows * X2;
    const float4* ap4 = reinterpret_cast<const float4*>(ap);
    const float4* ap14 = reinterpret_cast<const float4*>(ap1);
    float4* r4 = reinterpret_cast<float4*>(r);
    float4 av[U], t1[U], rv[U];
    int sp[U];
    bool ok[U];
    auto load = [&](int base) {
#pragma unroll
        for (int k = 0; k < U; k++) {
            const int i = base + k * stride;
            ok[k] = i < npair;
            const int ii = ok[k] ? i : 0;
            av[k] = __ldcg(ap4 + ii);
            t1[k] = __ldcg(ap14 + ii); // junk outside split strips: not used there
            rv[k] = __ldcg(r4 + ii);
            const int row = ii / X2, xp = ii - row * X2;
            sp[k] = split[(row / Y) * nxb + ((2 * xp) >> wshift)];
        }
    };
    double2 part{0, 0};
    if (i0 >= npair)
        return part;
    load(i0);
    while (true) {
#pragma unroll
        for (int k = 0; k < U; k++) {
            if (!ok[k])
                continue;
            float4 a = av[k];
            if (sp[k] > 1) {
                a.x += t1[k].x;
                a.y += t1[k].y;
                a.z += t1[k].z;
                a.w += t1[k].w;
                for (int pk = 2; pk < sp[k]; pk++) {
                    const float4 t = __ldcg(ap14 + i0 + k * stride + long(pk - 1) * (pstride / 2));
                    a.x += t.x;
                    a.y += t.y;
                    a.z += t.z;
                    a.w += t.w;
                }
            }
            float4 rr = rv[k];
            rr.x += -al * a.x;
            rr.y += -al * a.y;
            rr.z += -al * a.z;
            rr.w += -al * a.w;
            r4[i0 + k * stride] = rr;
            part.x += double(rr.x) * rr.x + double(rr.y) * rr.y;
            part.x += double(rr.z) * rr.z + double(rr.w) * rr.w;
        }
        i0 += U * stride;
        if (i0 >= npair)
            break;
        load(i0);
    }
    return part;
}

// r-only CG update (x deferred): r -= alpha Ap ; <r, r> partial.  With every
// search direction p_it kept, x = sum_it alpha_it p_it is formed once after the
// loop by k_cg_x_sum in the same fma order as the per-iteration update (bitwise
// identical), and each iteration streams 3 arrays instead of 5.
template<int U>
__global__ void __launch_bounds__(256) k_cg_update_r(CgDev* st, int it, cfloat* __restrict__ r,
                                                     const cfloat* __restrict__ ap, const cfloat* __restrict__ ap1,
                                                     const unsigned char* __restrict__ split, int X, int rows, int Y,
                                                     int nxb, int wshift, long pstride, unsigned* errflags)
{
    MDNN_PDL_ENTRY();
    __shared__ float s_alpha;
    if (threadIdx.x == 0)
        s_alpha = cg_alpha(st, it, errflags);
    __syncthreads();
    const float al = s_alpha;
    if (!(al > 0.f))
        return;
    double2 part = cg_r_update_pairs<U>(al, r, ap, ap1, split, X, rows, Y, nxb, wshift, pstride,
                                        int(blockIdx.x * blockDim.x + threadIdx.x), int(gridDim.x * blockDim.x));
    part = block_sum2(part);
    publish_partial(st->part_rr, &st->rr_sum, &st->cnt_rr, part);
}

// x += alpha_it p_it for every iteration that ran, in iteration order (the
// per-iteration update's fma sequence); P holds p_it at P + (it + 1) * n
__global__ void __launch_bounds__(256) k_cg_x_sum(const CgDev* __restrict__ st, cfloat* __restrict__ x,
                                                  const cfloat* __restrict__ P, long n)
{
    MDNN_PDL_ENTRY();
    const int nit = min(st->done_at, st->max_iter);
    const long npair = n >> 1;
    float4* x4 = reinterpret_cast<float4*>(x);
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < npair; i += long(gridDim.x) * blockDim.x) {
        float4 xv = x4[i];
        for (int it = 0; it < nit; it++) {
            const float al = st->alpha[it];
            if (!(al > 0.f))
                continue;
            const float4 pv = reinterpret_cast<const float4*>(P + (it + 1) * n)[i];
            xv.x = fmaf(al, pv.x, xv.x);
            xv.y = fmaf(al, pv.y, xv.y);
            xv.z = fmaf(al, pv.z, xv.z);
            xv.w = fmaf(al, pv.w, xv.w);
        }
        x4[i] = xv;
    }
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
    int planes = 1; // max CTAs sharing a strip (Ap planes)
    bool ws = false; // warp-specialised kernel (sense_ws.cuh)
    bool rr = false; // k_normal_rank with whole strips per CTA, round robin (32-B strips)
    int vh = 0;      // per-strip overhead weight of the cost-balanced ranges (ws kernel)
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
    r.W = n2 <= 24 ? RANK_W : 4;
    r.nxb = (g.X + r.W - 1) / r.W;
    r.strips = r.nxb * g.B;
    r.units = r.strips * g.C;
    int minb = 1;
    switch (g.Y) {
    case 128: minb = RankCfg<8, 16>::MINB; break;
    case 256: minb = RankCfg<16, 16>::MINB; break;
    case 320: minb = RankCfg<16, 20>::MINB; break;
    case 368: minb = RankCfg<16, 23>::MINB; break;
    case 512: minb = RankCfg<16, 32>::MINB; break;
    case 640: minb = RankCfg<16, 40>::MINB; break;
    }
    // warp-specialised kernel (k_normal_rank stays behind option sense_ws = 0).
    // N1 = 8 with twice the A/C warps was measured slower at Y = 368 (71.9 vs 63
    // us per CG launch): stage B then carries ~3.3 terms per row over 46-point rows.
    r.ws = g_sense_ws;
    if (r.ws)
        minb = 1;
    r.G = int(std::min<long>(g_rank_ctas > 0 ? g_rank_ctas : long(minb) * ctx().sm_count, r.units));
    // 32-B strips (W = 4): contiguous unit ranges put neighbouring strips of a
    // 128-B DRAM line on CTAs at different coils, and each line was fetched up to
    // 4x (1.09 GB for 302 MB algorithmic at 512^2 x 32 coils).  Whole strips
    // round robin keep neighbours in step; the load imbalance (ceil(strips / G))
    // is the smaller cost.
    r.rr = r.W == 4 && g_rank_rr && r.strips >= r.G;
    if (r.rr)
        r.G = int(std::min<long>(r.G, r.strips));
    r.vh = r.ws && !r.rr ? g_rank_vh : 0;
    r.planes = 1;
    if (!r.rr)
        for (long s = 0; s < r.strips; s++)
            r.planes = std::max(r.planes, rank_planes(s, g.C, r.units, r.G, r.vh));
    r.ok = r.units < (1L << 30) && g.Y * g.C * g.B < (1L << 30) && g.X * g.Y < (1L << 30) && r.planes < 250;
    return r;
}

template<int N1, int N2>
void launch_rank_t(RankArgs a, const cfloat* coils, const SenseGeom& g, const unsigned char* plans)
{
    using Cfg = RankCfg<N1, N2>;
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(2 * g.X), cuuint64_t(g.Y * g.C * g.B)};
    cuuint64_t strides[1] = {cuuint64_t(2 * g.X) * 4};
    cuuint32_t box[2] = {cuuint32_t(2 * Cfg::W), cuuint32_t(Cfg::BOXR)};
    cuuint32_t es[2] = {1, 1};
    // promote only to the box row: 32-B rows (W = 4) promoted to 128 B read the
    // neighbouring strips too, which other CTAs fetch again later (3.5x the
    // algorithmic DRAM bytes measured at 512^2 x 32 coils)
    CUresult res = rank_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<cfloat*>(coils), dims, strides,
                                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    Cfg::W * 8 >= 128  ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                    : Cfg::W * 8 >= 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                                       : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(coils) failed: " + std::to_string(int(res)));
    auto kern = k_normal_rank<N1, N2>;
    const int nthreads = Cfg::NT;
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_normal_rank<N1, N2>),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM)));
        attr = true;
    }
    const double xyb = double(g.X) * g.Y * g.B;
    const double work = 8.0 * xyb * (g.C + (a.mode == 1 ? 4 : 2));
    ProfScope prof(a.mode == 1 ? "sense_normal_y_cg" : "sense_normal_y", work);
    pdl_launch(kern, a.G, nthreads, Cfg::SMEM, ctx().stream, a, m, plans);
    KERNEL_CHECK();
}

// per-item row plans of the pattern (once per pattern, before the launches that use it)
template<int N1, int N2>
void launch_rank_plan_t(const RankArgs& a, unsigned char* plans, int nitems)
{
    pdl_launch(k_rank_plan<N1, N2>, nitems, RankCfg<N1, N2>::NT, 0, ctx().stream, a, plans);
    KERNEL_CHECK();
}

#define RANK_SHAPES(X_) X_(128, 8, 16) X_(256, 16, 16) X_(320, 16, 20) X_(368, 16, 23) X_(512, 16, 32) X_(640, 16, 40)
// (N1, N2) of every plan record layout: the k_normal_rank shapes and the ws shapes
#define PLAN_SHAPES(X_) RANK_SHAPES(X_)
#define WS_SHAPES(X_) RANK_SHAPES(X_)

// device memory for the per-item plans of a pattern
size_t rank_plan_record_bytes(const SenseGeom& g, const RankPlan& rp)
{
    const long items = g.pat_b > 1 ? g.pat_b : 1;
#define X_(YY, A1, A2) \
    if (rp.N1 == A1 && rp.N2 == A2) \
        return RankPlanRec<A1, A2>::BYTES * items;
    PLAN_SHAPES(X_)
#undef X_
    return 0;
}
// [per-item plan records | split flag per strip]
size_t rank_plan_bytes(const SenseGeom& g, const RankPlan& rp) { return rank_plan_record_bytes(g, rp) + size_t(rp.strips); }
const unsigned char* rank_split_flags(const SenseGeom& g, const RankPlan& rp, const unsigned char* plans)
{
    return plans + rank_plan_record_bytes(g, rp);
}

void fill_rank_args(const RankPlan& rp, RankArgs& a, const SenseGeom& g)
{
    a.tw = fast_twiddles(rp.N1, rp.N2);
    a.X = g.X;
    a.C = g.C;
    a.B = g.B;
    a.nxb = rp.nxb;
    a.units = rp.units;
    a.G = rp.G;
    a.rr = rp.rr ? 1 : 0;
    a.vh = rp.vh;
}

void launch_rank_plan(const RankPlan& rp, RankArgs a, const SenseGeom& g, unsigned char* plans)
{
    fill_rank_args(rp, a, g);
    const int items = int(g.pat_b > 1 ? g.pat_b : 1);
    a.split = plans + rank_plan_record_bytes(g, rp);
    a.strips = rp.strips;
#define X_(YY, A1, A2)                                \
    if (rp.N1 == A1 && rp.N2 == A2) {                 \
        launch_rank_plan_t<A1, A2>(a, plans, items); \
        return;                                       \
    }
    PLAN_SHAPES(X_)
#undef X_
    throw Error("rank A^H A: unsupported factorisation");
}

template<int N1, int N2>
void launch_ws_t(RankArgs a, const cfloat* coils, const SenseGeom& g, const unsigned char* plans);

void launch_rank(const RankPlan& rp, RankArgs a, const cfloat* coils, const SenseGeom& g,
                 const unsigned char* plans)
{
    fill_rank_args(rp, a, g);
    if (rp.ws) {
#define X_(YY, A1, A2)                               \
    if (rp.N1 == A1 && rp.N2 == A2) {                \
        launch_ws_t<A1, A2>(a, coils, g, plans);     \
        return;                                      \
    }
        WS_SHAPES(X_)
#undef X_
        throw Error("ws A^H A: unsupported factorisation");
    }
#define X_(YY, A1, A2) \
    case YY: launch_rank_t<A1, A2>(a, coils, g, plans); return;
    switch (g.Y) { RANK_SHAPES(X_) default: throw Error("rank A^H A: unsupported Y"); }
#undef X_
}
