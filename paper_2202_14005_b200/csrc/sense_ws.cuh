// Warp-specialised A^H A (+ lambda) for Y = N1 * N2, x-invariant patterns
// (included by sense.cu after sense_rank.cuh).  Same maths, work units, plan
// records and Ap-plane semantics as k_normal_rank (sense_rank.cuh), which
// replaces the operator chain of sense_normal_fragment + modl_normal_plus_lambda
// (recon.hpp:410-418, 807-820); different schedule:
//
//  * One CTA per SM, three warp roles joined by mbarriers instead of CTA-wide
//    barriers:
//      - a TMA producer warp streams coil slices (W columns x Y rows) of the
//        CTA's (strip, coil) units into an NSLOT-deep ring;
//      - the A/C warps (thread (w, j) as in k_normal_rank) own the x strip and
//        the coil accumulators in registers: A(i) = coil multiply + DFT over q
//        into S[i & 1]; C(i) = inverse DFT over k1 + conj-coil accumulate (the
//        coil slice is re-read from its ring slot, which is then released);
//        the loop runs A(i+1) before C(i) so the stage-B warps work on unit i
//        while the A/C warps transform unit i+1;
//      - the stage-B warps apply the mask-pruned row operators (identity rows
//        skipped, rank-1 terms) to S[i & 1], one thread per (row, column).
//  * Complex arithmetic is paired fp32 (FFMA2 / FADD2 / FMUL2 with broadcast,
//    swap and partial-negate operand modifiers): a complex multiply is two
//    instructions, a complex add one.
//  * The x strip of a new segment is loaded by A(i) while the epilogue of the
//    previous segment runs in C(i-1): the old strip is parked in a one-strip
//    stash in shared memory.
#pragma once

#include <algorithm>
#include <utility>

namespace cx2 {
// Complex arithmetic on float2.  WS_PAIRED = 1 (default) uses the paired-fp32
// forms (FFMA2/FADD2/FMUL2: half the instructions; one warp issues them only
// every ~3 cycles, tools/probes/ffma2_probe.cu); 0 uses scalar FFMA/FADD
// (~1.15 cycles per instruction per warp).  Measured on the C2 CG launch:
// paired 63.0 us, scalar 71.9 us.
#ifndef WS_PAIRED
#define WS_PAIRED 1
#endif
#if WS_PAIRED
__device__ __forceinline__ float2 add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
// a + DIR * i * b
template<int DIR>
__device__ __forceinline__ float2 addi(float2 a, float2 b)
{
    return DIR > 0 ? __fadd2_rn(a, make_float2(-b.y, b.x)) : __fadd2_rn(a, make_float2(b.y, -b.x));
}
// a * b
__device__ __forceinline__ float2 mul(float2 a, float2 b)
{
    const float2 t = __fmul2_rn(make_float2(a.y, a.x), make_float2(b.y, b.y));
    return __ffma2_rn(a, make_float2(b.x, b.x), make_float2(-t.x, t.y));
}
// acc + u * p
__device__ __forceinline__ float2 mac(float2 acc, float2 u, float2 p)
{
    const float2 t = __ffma2_rn(p, make_float2(u.x, u.x), acc);
    return __ffma2_rn(make_float2(-p.y, p.x), make_float2(u.y, u.y), t);
}
// acc + conj(c) * v
__device__ __forceinline__ float2 mac_conj(float2 acc, float2 c, float2 v)
{
    const float2 t = __ffma2_rn(v, make_float2(c.x, c.x), acc);
    return __ffma2_rn(make_float2(v.y, v.x), make_float2(c.y, -c.y), t);
}
// acc + d * conj(p), with e = (d.y, -d.x) precomputed
__device__ __forceinline__ float2 mac_dconj(float2 acc, float2 d, float2 e, float2 p)
{
    const float2 t = __ffma2_rn(d, make_float2(p.x, p.x), acc);
    return __ffma2_rn(e, make_float2(p.y, p.y), t);
}
__device__ __forceinline__ float2 scale(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }
// v * (c + i s), c and s compile-time constants
__device__ __forceinline__ float2 rotc(float2 v, float c, float s)
{
    const float2 t = __fmul2_rn(make_float2(v.y, v.x), make_float2(s, s));
    return __ffma2_rn(v, make_float2(c, c), make_float2(-t.x, t.y));
}
#else
__device__ __forceinline__ float2 add(float2 a, float2 b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ float2 sub(float2 a, float2 b) { return {a.x - b.x, a.y - b.y}; }
template<int DIR>
__device__ __forceinline__ float2 addi(float2 a, float2 b)
{
    return DIR > 0 ? float2{a.x - b.y, a.y + b.x} : float2{a.x + b.y, a.y - b.x};
}
__device__ __forceinline__ float2 mul(float2 a, float2 b)
{
    return {fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x)};
}
__device__ __forceinline__ float2 mac(float2 acc, float2 u, float2 p)
{
    return {fmaf(-u.y, p.y, fmaf(u.x, p.x, acc.x)), fmaf(u.y, p.x, fmaf(u.x, p.y, acc.y))};
}
__device__ __forceinline__ float2 mac_conj(float2 acc, float2 c, float2 v)
{
    return {fmaf(c.y, v.y, fmaf(c.x, v.x, acc.x)), fmaf(-c.y, v.x, fmaf(c.x, v.y, acc.y))};
}
__device__ __forceinline__ float2 mac_dconj(float2 acc, float2 d, float2 e, float2 p)
{
    return {fmaf(e.x, p.y, fmaf(d.x, p.x, acc.x)), fmaf(e.y, p.y, fmaf(d.y, p.x, acc.y))};
}
__device__ __forceinline__ float2 scale(float2 a, float s) { return {a.x * s, a.y * s}; }
__device__ __forceinline__ float2 rotc(float2 v, float c, float s)
{
    return {fmaf(v.x, c, -v.y * s), fmaf(v.x, s, v.y * c)};
}
#endif

// v * exp(DIR * 2 pi i m / R), exact for quarter turns
template<long M_, int R, int DIR>
__device__ __forceinline__ float2 rot(float2 v)
{
    constexpr long m = ((M_ % R) + R) % R;
    if constexpr (m == 0) {
        return v;
    } else if constexpr (2 * m == R) {
        return make_float2(-v.x, -v.y);
    } else if constexpr (4 * m == R) {
        return DIR > 0 ? make_float2(-v.y, v.x) : make_float2(v.y, -v.x);
    } else if constexpr (4 * m == 3 * R) {
        return DIR > 0 ? make_float2(v.y, -v.x) : make_float2(-v.y, v.x);
    } else {
        constexpr float c = float(fftd::cos2pi(m, R));
        constexpr float s = float(DIR * fftd::sin2pi(m, R));
        return rotc(v, c, s);
    }
}

template<int I, int N, class F>
__device__ __forceinline__ void sfor(F&& f)
{
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        sfor<I + 1, N>(f);
    }
}

template<int DIR>
__device__ __forceinline__ void dft4(float2& a0, float2& a1, float2& a2, float2& a3)
{
    const float2 s0 = add(a0, a2), d0 = sub(a0, a2), s1 = add(a1, a3), d1 = sub(a1, a3);
    a0 = add(s0, s1);
    a2 = sub(s0, s1);
    a1 = addi<DIR>(d0, d1);
    a3 = addi<-DIR>(d0, d1);
}

// in-register DFT of R = P * 4 points (P in {2, 4}), natural order in and out:
// X[k] = sum_n x[n] exp(DIR 2 pi i n k / R)
template<int R, int DIR>
__device__ __forceinline__ void dft(float2 (&v)[R])
{
    static_assert(R == 8 || R == 16, "paired-fp32 DFT: R = 8 or 16");
    constexpr int Q = 4, P = R / 4;
    // step 1: DFT-P over n1 of x[Q n1 + n2], in place (index Q k1 + n2)
    sfor<0, Q>([&](auto N2_) {
        constexpr int n2 = decltype(N2_)::value;
        if constexpr (P == 4) {
            dft4<DIR>(v[n2], v[Q + n2], v[2 * Q + n2], v[3 * Q + n2]);
        } else {
            const float2 a = v[n2], b = v[Q + n2];
            v[n2] = add(a, b);
            v[Q + n2] = sub(a, b);
        }
    });
    // step 2: twiddles W_R^(n2 k1)
    sfor<1, P>([&](auto K1_) {
        constexpr int k1 = decltype(K1_)::value;
        sfor<1, Q>([&](auto N2_) {
            constexpr int n2 = decltype(N2_)::value;
            v[Q * k1 + n2] = rot<long(n2) * k1, R, DIR>(v[Q * k1 + n2]);
        });
    });
    // step 3: DFT-4 over n2 for each k1 -> X[k1 + P k2] at Q k1 + k2
    sfor<0, P>([&](auto K1_) {
        constexpr int k1 = decltype(K1_)::value;
        dft4<DIR>(v[Q * k1], v[Q * k1 + 1], v[Q * k1 + 2], v[Q * k1 + 3]);
    });
    float2 o[R];
    sfor<0, P>([&](auto K1_) {
        constexpr int k1 = decltype(K1_)::value;
        sfor<0, Q>([&](auto K2_) {
            constexpr int k2 = decltype(K2_)::value;
            o[k1 + P * k2] = v[Q * k1 + k2];
        });
    });
#pragma unroll
    for (int k = 0; k < R; k++)
        v[k] = o[k];
}
} // namespace cx2

#ifndef WS_NTW
#define WS_NTW 12 // warps per CTA (at least)
#endif
template<int N1, int N2>
struct WsCfg {
    using RC = RankCfg<N1, N2>; // plan record layout (TMAX, N2P) and TMA boxes
    static constexpr int Y = N1 * N2;
    static constexpr int W = N2 <= 24 ? 8 : 4;                // as k_normal_rank (32-B strips past N2 = 24)
    static constexpr int N2P = RC::N2P;
    static constexpr int TMAX = RC::TMAX;
    static constexpr int NBOX = RC::NBOX, BOXR = RC::BOXR;
    static constexpr int NT_AC = ((W * N2 + 31) / 32) * 32;  // A/C threads (w, j)
    // stage B: BQ threads per (row, column), each JQ consecutive j (even: float4 twiddle pairs)
    static constexpr int BQ = N2 > 24 ? 4 : 2;
    static constexpr int jq(int v) { return (v * W) % 16 == 0 ? v : jq(v + 2); }
    static constexpr int JQ = jq((((N2P + BQ - 1) / BQ) + 1) & ~1); // parts start 16-float2 aligned
    // 12 warps in all: ptxas sizes the register budget for a multiple of 4 warps
    // (13 warps got the 16-warp cap of 128 registers and spilled)
    // one pass over the (row, column, part) items of the reference pattern family
    // (12 rows x W x BQ <= 192); with 13 warps ptxas budgets registers for 16 (128)
    static constexpr int NT_B = 32 * (WS_NTW - NT_AC / 32 - 1) >= 192 ? 32 * (WS_NTW - NT_AC / 32 - 1) : 192;
    static constexpr int NT = NT_AC + NT_B + 32;             // + TMA producer warp
    static constexpr int SLOT = Y * W;                        // float2 per coil slice / stash
    // S layout: element (row m, j, column w) at m * RP + SOFF(j) + w; j-part p
    // is shifted by 8 p float2 so the BQ parts of a stage-B item fall in
    // alternate halves of the banks (conflict-free)
    // (W = 4: + 4 more, so the two rows of a stage-B warp use opposite bank quarters)
    static constexpr int RP = N2P * W + 8 * BQ + (W == 4 ? 4 : 0);
    __host__ __device__ static constexpr int SOFF(int j) { return j * W + 8 * (j / JQ); }
    static constexpr int SBUF = N1 * RP;
    static constexpr int TTW = TMAX * N2P + 8;                // twiddle rows + zero pad (last part's reads)
    static constexpr size_t STATIC_EST = 4096;                // plan, barriers, reductions
    // 2 S buffers, stash, 2 staging strips (x or r, and p_prev), twiddle rows
    // (+ 16 float2 = 128 B: the stash's extra row Y, read only by padding threads;
    // keeps the TMA-written staging buffers 128-B aligned)
    static constexpr int STASH_PAD = 16;
    static constexpr size_t FIXED = sizeof(float2) * (size_t(2) * SBUF + 3 * size_t(SLOT) + STASH_PAD + size_t(TTW));
    static constexpr size_t SMEM_MAX = 227 * 1024;
    static constexpr int NSLOT_FIT = int((SMEM_MAX - STATIC_EST - FIXED) / (sizeof(float2) * SLOT));
    static constexpr int NSLOT = NSLOT_FIT > 6 ? 6 : NSLOT_FIT;
    static constexpr size_t SMEM = FIXED + sizeof(float2) * size_t(NSLOT) * SLOT;
    static_assert(NSLOT >= 3, "coil ring needs three slots");
    static_assert(N1 == 8 || N1 == 16, "paired DFT sizes");
    static_assert((JQ * W) % 16 == 0, "bank layout");
};

#ifdef WS_PROF
#define WS_WAIT(k, bar, ph)                        \
    do {                                           \
        const long long t0_ = clock64();           \
        sm100::mbar_wait(bar, ph);                 \
        wprof[k] += clock64() - t0_;               \
    } while (0)
#else
#define WS_WAIT(k, bar, ph) sm100::mbar_wait(bar, ph)
#endif

__device__ __forceinline__ void named_bar_sync(int id, int nthreads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Fused CG update of iteration a.it (cg_defer_x path; replaces the k_cg_update_r
// launch): every CTA stores its <p, Ap> partial and meets the others at a grid
// barrier (cooperative launch: all CTAs co-resident), folds the partials exactly
// as publish_partial's last CTA would (same order, same block size: bitwise the
// same alpha on every CTA), then updates r over a grid-stride range of pixel pairs
// and publishes its <r, r> partial.
__device__ void ws_cg_update(const RankArgs& a, double2 part)
{
    CgDev* st = a.cg;
    __shared__ float s_al;
    if (threadIdx.x == 0) {
        st->part_pap[blockIdx.x] = part;
        __threadfence();
        atomicAdd(&st->ws_bar, 1u);
        const unsigned target = unsigned(a.it + 1) * gridDim.x;
        // bounded spin (~seconds): a grid that is not co-resident raises an error
        // instead of hanging the device
        for (long spin = 0;; spin++) {
            unsigned v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&st->ws_bar) : "memory");
            if (v >= target)
                break;
            if (spin > (1L << 26)) {
                atomicOr(a.errflags, unsigned(ERRF_GRID_BARRIER));
                break;
            }
            __nanosleep(32);
        }
    }
    __syncthreads();
    double2 v{0, 0};
    for (unsigned k = threadIdx.x; k < gridDim.x; k += blockDim.x)
        v.x += __ldcg(&st->part_pap[k].x);
    v = block_sum2(v);
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0)
            st->pap_sum = v.x;
        s_al = cg_alpha_sum(st, a.it, v.x, a.errflags);
    }
    __syncthreads();
    const float al = s_al;
    if (!(al > 0.f))
        return;
    double2 pr = cg_r_update_pairs<2>(al, a.r_upd, a.out, a.out1, a.split, int(a.X), a.upd_rows, a.upd_Y,
                                      int(a.nxb), a.upd_wshift, a.pstride, int(blockIdx.x * blockDim.x + threadIdx.x),
                                      int(gridDim.x * blockDim.x));
    pr = block_sum2(pr);
    publish_partial(st->part_rr, &st->rr_sum, &st->cnt_rr, pr);
}

template<int N1, int N2>
__global__ void __launch_bounds__(WsCfg<N1, N2>::NT, 1)
    k_normal_ws(RankArgs a, const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tmx,
                const __grid_constant__ CUtensorMap tmp, const unsigned char* __restrict__ plans)
{
    MDNN_PDL_ENTRY();
    using Cfg = WsCfg<N1, N2>;
    constexpr int Y = Cfg::Y, W = Cfg::W, N2P = Cfg::N2P, TMAX = Cfg::TMAX, RP = Cfg::RP;
    constexpr int NT_AC = Cfg::NT_AC, NT_B = Cfg::NT_B, NSLOT = Cfg::NSLOT;
    constexpr int SLOT = Cfg::SLOT, SBUF = Cfg::SBUF;
    extern __shared__ __align__(128) float2 ws_smem[];
    float2* ring = ws_smem;
    float2* Sb = ring + size_t(NSLOT) * SLOT;
    float2* stash = Sb + 2 * SBUF;
    float2* stg = stash + SLOT + Cfg::STASH_PAD; // [2][SLOT]: strip of x (or r) and of p_prev, TMA-staged one segment ahead
    float2* ttw = stg + 2 * SLOT;
    __shared__ __align__(8) uint64_t bar_full[NSLOT], bar_empty[NSLOT], bar_sfull[2], bar_sdone[2], bar_xfull,
        bar_xempty;
    __shared__ float s_beta;
    __shared__ float2 s_lam;
    __shared__ __align__(16) RankPlanSm<N1, N2> pl;

    const int tid = threadIdx.x;
    const int C = int(a.C), nxb = int(a.nxb);
    const int U = int(a.units);
    // contiguous unit ranges, or (a.rr, 32-B strips) whole strips g, g + G, ...
    // so that neighbouring strips of one 128-B DRAM line are read together
    const int u_begin = a.rr ? int(blockIdx.x) * C : int(rank_ubegin(blockIdx.x, C, U, a.G, a.vh));
    const int n = a.rr ? C * ((U / C - 1 - int(blockIdx.x)) / a.G + 1)
                       : int(rank_ubegin(blockIdx.x + 1, C, U, a.G, a.vh)) - u_begin;
    const int sstep = a.rr ? a.G : 1; // strip step between segments
    // next segment's strip: (b, xb) advanced by sstep strips
    auto next_strip = [&](int& xb, int& b) {
        xb += sstep;
        while (xb >= nxb) {
            xb -= nxb;
            ++b;
        }
    };

    // (MDNN_PDL_ENTRY above: the previous kernel's r / p / CG scalars are read only
    // after its wait; from there on the next kernel may be scheduled)
    if (tid == 0) {
        for (int s = 0; s < NSLOT; s++) {
            sm100::mbar_init(&bar_full[s], 1);
            sm100::mbar_init(&bar_empty[s], NT_AC);
        }
        for (int b = 0; b < 2; b++) {
            sm100::mbar_init(&bar_sfull[b], NT_AC);
            sm100::mbar_init(&bar_sdone[b], NT_B);
        }
        sm100::mbar_init(&bar_xfull, 1);
        sm100::mbar_init(&bar_xempty, NT_AC);
        sm100::fence_barrier_init();
        s_beta = a.mode == 1 ? cg_prologue(a.cg, a.it, a.errflags) : 0.f;
        s_lam = a.lam ? a.lam[0] : a.lamv;
    }
    __syncthreads();
    const float beta = s_beta;
    if (a.mode == 1 && beta < 0.f)
        return; // CG already stopped (nothing issued yet)
    const bool upd = a.mode == 1 && a.it > 0;
    double2 part{0, 0};
#ifdef WS_PROF
    long long wprof[4] = {0, 0, 0, 0}, tprof[4] = {0, 0, 0, 0};
    const long long tstart = clock64();
#endif

    if (tid >= NT_AC + NT_B) {
        // ---------------- TMA producer ----------------
        if (tid == NT_AC + NT_B) {
            sm100::prefetch_tmap(&tmap);
            sm100::prefetch_tmap(&tmx);
            if (upd)
                sm100::prefetch_tmap(&tmp);
            int c, xblk, b;
            {
                const int s0 = u_begin / C;
                c = u_begin - s0 * C;
                b = s0 / nxb;
                xblk = s0 - b * nxb;
            }
            // x (or r, and p_prev) strips: segment k starts at unit seg_start(k); it is
            // staged as soon as segment k-1's strips were consumed (tested between
            // coil loads), at the latest just before its first unit
            const int c0 = c;
            auto seg_start = [&](int k) { return k == 0 ? 0 : (C - c0) + (k - 1) * C; };
            int nst = 0, st_b = b, st_xb = xblk;
            auto stage = [&]() {
                if (nst > 0)
                    WS_WAIT(0, &bar_xempty, uint32_t((nst - 1) & 1));
                sm100::mbar_arrive_expect_tx(&bar_xfull, uint32_t((upd ? 2 : 1) * SLOT * sizeof(float2)));
#pragma unroll
                for (int k = 0; k < Cfg::NBOX; k++) {
                    sm100::tma_load_2d(stg + k * Cfg::BOXR * W, &tmx, &bar_xfull, 2 * W * st_xb,
                                       Y * st_b + k * Cfg::BOXR);
                    if (upd)
                        sm100::tma_load_2d(stg + SLOT + k * Cfg::BOXR * W, &tmp, &bar_xfull, 2 * W * st_xb,
                                           Y * st_b + k * Cfg::BOXR);
                }
                nst++;
                next_strip(st_xb, st_b);
            };
            for (int i = 0; i < n; i++) {
                if (seg_start(nst) == i)
                    stage();
                const int slot = i % NSLOT;
                if (i >= NSLOT)
                    WS_WAIT(0, &bar_empty[slot], uint32_t((i / NSLOT - 1) & 1));
                const int row0 = Y * (c + C * b);
                const int xb_i = xblk;
                if (++c == C) {
                    c = 0;
                    next_strip(xblk, b);
                }
                sm100::mbar_arrive_expect_tx(&bar_full[slot], uint32_t(SLOT * sizeof(float2)));
#pragma unroll
                for (int k = 0; k < Cfg::NBOX; k++)
                    sm100::tma_load_2d(ring + size_t(slot) * SLOT + k * Cfg::BOXR * W, &tmap, &bar_full[slot],
                                       2 * W * xb_i, row0 + k * Cfg::BOXR);
                if (nst > 0 && seg_start(nst) < n && sm100::mbar_try(&bar_xempty, uint32_t((nst - 1) & 1)))
                    stage();
            }
        }
    } else if (tid >= NT_AC) {
        // ---------------- stage B: row operators on S ----------------
        const int bt = tid - NT_AC;
        int plan_b = -1;
        int w_c, w_xb, w_b;
        {
            const int s0 = u_begin / C;
            w_c = u_begin - s0 * C;
            w_b = s0 / nxb;
            w_xb = s0 - w_b * nxb;
        }
        for (int i = 0; i < n; i++) {
            const int b = w_b;
            if (++w_c == C) {
                w_c = 0;
                next_strip(w_xb, w_b);
            }
            if (b != plan_b && (plan_b < 0 || a.ps.sb != 0)) {
                using Rec = RankPlanRec<N1, N2>;
                named_bar_sync(1, NT_B); // every item of the previous unit is done with the old plan
                const int4* src = reinterpret_cast<const int4*>(plans + Rec::BYTES * (a.ps.sb != 0 ? b : 0));
                int4* dpl = reinterpret_cast<int4*>(&pl);
                for (int e = bt; e < int(Rec::PL / 16); e += NT_B)
                    dpl[e] = src[e];
                const int4* src2 = reinterpret_cast<const int4*>(reinterpret_cast<const unsigned char*>(src) + Rec::PL);
                int4* dtw = reinterpret_cast<int4*>(ttw);
                for (int e = bt; e < int(TMAX * N2P * sizeof(float2) / 16); e += NT_B)
                    dtw[e] = src2[e];
                for (int e = bt; e < Cfg::TTW - TMAX * N2P; e += NT_B)
                    ttw[TMAX * N2P + e] = float2{0.f, 0.f};
                named_bar_sync(1, NT_B);
                plan_b = b;
            }
            WS_WAIT(1, &bar_sfull[i & 1], uint32_t((i >> 1) & 1));
            float2* S = Sb + (i & 1) * SBUF;
            constexpr int BQ = Cfg::BQ, NJ = Cfg::JQ;
            const int nitems = BQ * pl.nwork * W;
            for (int item = bt; item < nitems; item += NT_B) {
                // BQ threads per (row, column): each NJ consecutive j in registers,
                // dot products combined with log2(BQ) shuffles
                const int h = item % BQ, pr = item / BQ;
                const int r = pr / W, ww = pr - r * W;
                const int k1 = pl.work_k1[r];
                const int md = pl.mode[k1], nt = pl.nt[k1], off = pl.off[k1];
                const int jb = h * NJ;
                float2* row = S + k1 * RP + Cfg::SOFF(jb) + ww; // element jb + jj at row[jj * W]
                const unsigned pmask = ((1u << BQ) - 1) << ((tid & 31) & ~(BQ - 1));
                auto qsum = [&](float2 d) {
#pragma unroll
                    for (int o = 1; o < BQ; o <<= 1) {
                        d.x += __shfl_xor_sync(pmask, d.x, o);
                        d.y += __shfl_xor_sync(pmask, d.y, o);
                    }
                    return d;
                };
                float2 u[NJ];
#pragma unroll
                for (int jj = 0; jj < NJ; jj++)
                    u[jj] = (jb + jj < N2) ? row[jj * W] : float2{0.f, 0.f};
                if (nt <= 4 && off + nt <= TMAX) {
                    // up to 4 terms with precomputed twiddle rows: all dot products in
                    // one pass over the part (2 chains per term), then one scatter pass
                    auto fast = [&](auto NTT_) {
                        constexpr int NTT = decltype(NTT_)::value;
                        // 16-B aligned: N2P and NJ even; reads past N2 meet zero u (or the zero pad)
                        const float4* tv[NTT > 0 ? NTT : 1];
#pragma unroll
                        for (int t = 0; t < NTT; t++)
                            tv[t] = reinterpret_cast<const float4*>(ttw + (off + t) * N2P + jb);
                        float2 da[NTT > 0 ? NTT : 1], db[NTT > 0 ? NTT : 1];
#pragma unroll
                        for (int t = 0; t < NTT; t++)
                            da[t] = db[t] = float2{0.f, 0.f};
#pragma unroll
                        for (int jj = 0; jj < NJ; jj += 2) {
#pragma unroll
                            for (int t = 0; t < NTT; t++) {
                                const float4 q = tv[t][jj >> 1];
                                da[t] = cx2::mac(da[t], u[jj], float2{q.x, q.y});
                                db[t] = cx2::mac(db[t], u[jj + 1], float2{q.z, q.w});
                            }
                        }
                        float2 d[NTT > 0 ? NTT : 1], e[NTT > 0 ? NTT : 1];
#pragma unroll
                        for (int t = 0; t < NTT; t++) {
                            d[t] = cx2::mul(qsum(cx2::add(da[t], db[t])), pl.coef[off + t]);
                            e[t] = float2{d[t].y, -d[t].x};
                        }
#pragma unroll
                        for (int jj = 0; jj < NJ; jj += 2) {
                            float4 q[NTT > 0 ? NTT : 1];
#pragma unroll
                            for (int t = 0; t < NTT; t++)
                                q[t] = tv[t][jj >> 1];
#pragma unroll
                            for (int hh = 0; hh < 2; hh++) {
                                if (jb + jj + hh < N2) {
                                    float2 r0 = md == 1 ? u[jj + hh] : float2{0.f, 0.f};
#pragma unroll
                                    for (int t = 0; t < NTT; t++)
                                        r0 = cx2::mac_dconj(r0, d[t], e[t],
                                                            hh ? float2{q[t].z, q[t].w} : float2{q[t].x, q[t].y});
                                    row[(jj + hh) * W] = r0;
                                }
                            }
                        }
                    };
                    switch (nt) {
                    case 0: fast(std::integral_constant<int, 0>{}); break;
                    case 1: fast(std::integral_constant<int, 1>{}); break;
                    case 2: fast(std::integral_constant<int, 2>{}); break;
                    case 3: fast(std::integral_constant<int, 3>{}); break;
                    default: fast(std::integral_constant<int, 4>{}); break;
                    }
                } else {
                    // general rows: any number of terms, twiddles indexed on the fly;
                    // the part row in shared memory is the running result
                    if (md != 1) {
#pragma unroll
                        for (int jj = 0; jj < NJ; jj++)
                            if (jb + jj < N2)
                                row[jj * W] = float2{0.f, 0.f};
                    }
                    for (int t = off; t < off + nt; t++) {
                        const int k = pl.tk[t];
                        const int m00 = (jb * k) % Y;
                        int m0 = m00;
                        float2 da{0.f, 0.f}, db{0.f, 0.f};
#pragma unroll
                        for (int jj = 0; jj < NJ; jj++) {
                            const float2 tv = (jb + jj < N2) ? __ldg(&a.tw[m0]) : float2{0.f, 0.f};
                            if (jj & 1)
                                db = cx2::mac(db, u[jj], tv);
                            else
                                da = cx2::mac(da, u[jj], tv);
                            m0 += k;
                            m0 -= m0 >= Y ? Y : 0;
                        }
                        const float2 d = cx2::mul(qsum(cx2::add(da, db)), pl.coef[t]);
                        const float2 e{d.y, -d.x};
                        m0 = m00;
#pragma unroll
                        for (int jj = 0; jj < NJ; jj++) {
                            if (jb + jj < N2)
                                row[jj * W] = cx2::mac_dconj(row[jj * W], d, e, __ldg(&a.tw[m0]));
                            m0 += k;
                            m0 -= m0 >= Y ? Y : 0;
                        }
                    }
                }
            }
            sm100::mbar_arrive(&bar_sdone[i & 1]);
        }
    } else {
        // ---------------- A/C warps ----------------
        const int w = tid % W, j0 = tid / W;
        const bool active = j0 < N2;
        const int j = active ? j0 : N2 - 1;
        constexpr float invN1 = 1.f / float(N1);
        const float2 lam = s_lam;
        int nseg = 0;
        float2 xr[N1], acc[N1];
#pragma unroll
        for (int q = 0; q < N1; q++)
            acc[q] = float2{0.f, 0.f};
        // unit walkers (no per-unit integer division): stage A leads, stage C trails by one
        int a_c, a_xb, a_b;
        {
            const int s0 = u_begin / C;
            a_c = u_begin - s0 * C;
            a_b = s0 / nxb;
            a_xb = s0 - a_b * nxb;
        }
        int c_c = a_c;
        int cur_s = u_begin / C, prev_s = cur_s;  // strip of xr / of the stash
        int cur_b = a_b, cur_xb = a_xb, prev_b = a_b, prev_xb = a_xb;
        bool cur_first = false, prev_first = false;
        bool opened = false;

        auto stage_a = [&](int i) {
#ifdef WS_PROF
            long long t0 = clock64();
#endif
            opened = i == 0 || a_c == 0;
            if (opened) {
                // open a segment: park the old strip, load x (or p = r + beta p_prev)
                if (i > 0 && active) {
#pragma unroll
                    for (int q = 0; q < N1; q++)
                        stash[(j + N2 * q) * W + w] = xr[q];
                }
                prev_s = cur_s;
                prev_first = cur_first;
                prev_b = cur_b;
                prev_xb = cur_xb;
                cur_s = i == 0 ? cur_s : cur_s + sstep;
                cur_first = a_c == 0;
                cur_b = a_b;
                cur_xb = a_xb;
                const int xx = a_xb * W + w;
                const bool colok = active && xx < a.X;
                const long img_base = xx + a.X * Y * long(a_b);
                WS_WAIT(0, &bar_xfull, uint32_t(nseg & 1));
                nseg++;
                // padding threads and columns past X read zeros from the TMA fill (j clamped rows are valid)
#pragma unroll
                for (int q = 0; q < N1; q++)
                    xr[q] = stg[(j + N2 * q) * W + w];
                if (upd) {
#pragma unroll
                    for (int q = 0; q < N1; q++) {
                        const float2 pv = stg[SLOT + (j + N2 * q) * W + w];
                        xr[q] = float2{xr[q].x + beta * pv.x, xr[q].y + beta * pv.y};
                    }
                }
                sm100::mbar_arrive(&bar_xempty);
                if (!colok) {
#pragma unroll
                    for (int q = 0; q < N1; q++)
                        xr[q] = float2{0.f, 0.f};
                }
                if (upd && cur_first && colok) {
#pragma unroll
                    for (int q = 0; q < N1; q++)
                        a.p_out[img_base + a.X * (j + N2 * q)] = xr[q];
                }
            }
            // advance the stage-A walker
            if (++a_c == C) {
                a_c = 0;
                next_strip(a_xb, a_b);
            }
            const int slot = i % NSLOT;
#ifdef WS_PROF
            tprof[0] += clock64() - t0;
#endif
            WS_WAIT(2, &bar_full[slot], uint32_t((i / NSLOT) & 1));
#ifdef WS_PROF
            t0 = clock64();
#endif
            const float2* csp = ring + size_t(slot) * SLOT + j * W + w;
            float2 v[N1];
#pragma unroll
            for (int q = 0; q < N1; q++)
                v[q] = cx2::mul(csp[N2 * W * q], xr[q]);
            cx2::dft<N1, -1>(v);
            if (active) {
                float2* S = Sb + (i & 1) * SBUF + Cfg::SOFF(j) + w;
#pragma unroll
                for (int m = 0; m < N1; m++)
                    S[m * RP] = v[m];
            }
            sm100::mbar_arrive(&bar_sfull[i & 1]);
#ifdef WS_PROF
            tprof[1] += clock64() - t0;
#endif
        };

        auto stage_c = [&](int i, bool from_stash) {
            WS_WAIT(3, &bar_sdone[i & 1], uint32_t((i >> 1) & 1));
#ifdef WS_PROF
            long long t0 = clock64();
#endif
            // padding threads (j0 >= N2; only N2 = 23, where j0 = N2 < N2P) read the
            // never-written pad column instead of their active twin's row (racecheck)
            const float2* S = Sb + (i & 1) * SBUF + Cfg::SOFF(j0) + w;
            const int slot = i % NSLOT;
            const float2* csp = ring + size_t(slot) * SLOT + j * W + w;
            float2 v[N1], cv[N1];
#pragma unroll
            for (int q = 0; q < N1; q++)
                cv[q] = csp[N2 * W * q];
#pragma unroll
            for (int m = 0; m < N1; m++)
                v[m] = S[m * RP];
            cx2::dft<N1, +1>(v);
#pragma unroll
            for (int q = 0; q < N1; q++)
                acc[q] = cx2::mac_conj(acc[q], cv[q], v[q]);
            sm100::mbar_arrive(&bar_empty[slot]);
            const bool closes = i == n - 1 || c_c == C - 1;
            if (++c_c == C)
                c_c = 0;
#ifdef WS_PROF
            tprof[2] += clock64() - t0;
            t0 = clock64();
#endif
            if (closes) {
                // segment epilogue: 1/N1, + lambda x (plane 0), store, <p, Ap>
                const int s = from_stash ? prev_s : cur_s;
                const bool first = from_stash ? prev_first : cur_first;
                const int b = from_stash ? prev_b : cur_b, xx = (from_stash ? prev_xb : cur_xb) * W + w;
                const long img_base = xx + a.X * Y * long(b);
                cfloat* dst = rank_plane_dst(a, s, blockIdx.x);
                // stash rows: y = j + N2 q; padding threads read the extra row Y (never
                // written) instead of rows their active twins rewrite at the next open
                const int sy0 = active ? j : Y, sdy = active ? N2 : 0;
#pragma unroll
                for (int q = 0; q < N1; q++) {
                    const int y = j + N2 * q;
                    const float2 xv = from_stash ? stash[(sy0 + sdy * q) * W + w] : xr[q];
                    float2 o = cx2::scale(acc[q], invN1);
                    if (first)
                        o = cx2::add(o, cx2::mul(xv, lam));
                    if (active && xx < a.X) {
                        dst[img_base + a.X * y] = o;
                        // Re <p, Ap> only (CG reads the real part; mode 0 ignores it)
                        part.x += double(xv.x) * o.x + double(xv.y) * o.y;
                    }
                    acc[q] = float2{0.f, 0.f};
                }
            }
#ifdef WS_PROF
            tprof[3] += clock64() - t0;
#endif
        };

        for (int i = 0; i < n; i++) {
            stage_a(i);
            if (i > 0)
                stage_c(i - 1, opened); // unit i opened a new segment: unit i-1's x is stashed
        }
        if (n > 0) // (cost-balanced ranges can leave a CTA without units)
            stage_c(n - 1, false);
    }
#ifdef WS_PROF
    if (blockIdx.x < 2 && (tid == 0 || tid == NT_AC || tid == NT_AC + NT_B))
        printf("ws cta %d role %s n %d total %lld wait empty %lld sfull %lld full %lld sdone %lld | open %lld A %lld C "
               "%lld epi %lld\n",
               int(blockIdx.x), tid == 0 ? "AC" : tid == NT_AC ? "B" : "P", n, clock64() - tstart, wprof[0], wprof[1],
               wprof[2], wprof[3], tprof[0], tprof[1], tprof[2], tprof[3]);
#endif
    if (a.mode == 1) {
        part = block_sum2(part);
        if (a.r_upd)
            ws_cg_update(a, part);
        else
            publish_partial(a.cg->part_pap, &a.cg->pap_sum, &a.cg->cnt_pap, part);
    } else {
        // keep every role resident until the A/C warps are done: letting the
        // producer and stage-B warps exit early made the mode-0 launch 1.7x
        // slower (96 vs 58 us at C2, coil-slice waits on some CTAs)
        __syncthreads();
    }
}

template<int N1, int N2>
void launch_ws_t(RankArgs a, const cfloat* coils, const SenseGeom& g, const unsigned char* plans)
{
    using Cfg = WsCfg<N1, N2>;
    // [2X floats, rows] strips of W columns x BOXR rows; promotion to the box row
    // only: a wider L2 fetch pulls in the neighbouring strip, which another CTA
    // reads much later
    auto strip_map = [&](const cfloat* base, long rows, const char* what) {
        CUtensorMap m;
        cuuint64_t dims[2] = {cuuint64_t(2 * g.X), cuuint64_t(rows)};
        cuuint64_t strides[1] = {cuuint64_t(2 * g.X) * 4};
        cuuint32_t box[2] = {cuuint32_t(2 * Cfg::W), cuuint32_t(Cfg::BOXR)};
        cuuint32_t es[2] = {1, 1};
        CUresult res = rank_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<cfloat*>(base), dims,
                                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        Cfg::W * 8 >= 128  ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                        : Cfg::W * 8 >= 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                                           : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (res != CUDA_SUCCESS)
            throw CudaError(std::string("cuTensorMapEncodeTiled(") + what + ") failed: " + std::to_string(int(res)));
        return m;
    };
    const CUtensorMap m = strip_map(coils, g.Y * g.C * g.B, "coils");
    const cfloat* src = a.mode == 0 ? a.x : (a.it == 0 ? a.p_out : a.x);
    const CUtensorMap mx = strip_map(src, g.Y * g.B, "x");
    const CUtensorMap mp = (a.mode == 1 && a.it > 0) ? strip_map(a.p, g.Y * g.B, "p") : mx;
    if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(a.mode == 1 ? a.p : src)) & 15)
        throw CudaError("A^H A: image arrays must be 16-byte aligned");
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_normal_ws<N1, N2>),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM)));
        attr = true;
    }
    const double xyb = double(g.X) * g.Y * g.B;
    // algorithmic bytes: coils once, x (r, p_prev, p_out) and Ap; the fused CG
    // update adds r and Ap read, r written
    const double work = 8.0 * xyb * (g.C + (a.mode == 1 ? 4 : 2) + (a.r_upd ? 3 : 0));
    ProfScope prof(a.mode == 1 ? "sense_normal_y_cg" : "sense_normal_y", work);
    launch_ex(g_cg_pdl, a.r_upd != nullptr && g_cg_fuse == 2, k_normal_ws<N1, N2>, dim3(a.G), dim3(Cfg::NT), size_t(Cfg::SMEM), a, m, mx, mp,
              plans);
    KERNEL_CHECK();
}
