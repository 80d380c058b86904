// k_normal_rank_tm: the rank A^H A kernel (sense_rank.cuh) re-laid-out for
// 3 CTAs (18 warps) per SM instead of 2 (12 warps): the per-thread coil
// accumulators and the x / p column strip live in tensor memory (TMEM, 64 of
// the 512 columns per CTA-warp group) instead of registers and shared memory,
// and the two TMA ring slots double as the stage-A/B/C work buffer (stage A
// overwrites the coil values it has read with its DFT outputs at the same
// addresses, so no separate S buffer).  The coil values stay in registers
// from A to C of the same unit; a slot is refilled once C of its unit is done.
// Same maths, plan, split-strip planes and CG fusion as k_normal_rank.
#pragma once

template<int N1, int N2>
struct RankTmCfg {
    using Base = RankCfg<N1, N2>;
    static constexpr int Y = N1 * N2, W = Base::W, NT = Base::NT, N2P = Base::N2P, JH = Base::JH;
    static constexpr int TMAX = Base::TMAX;
    static constexpr size_t SLOT = size_t(Y) * W;
    // dynamic smem (float2): slot[2][SLOT] | ttw[TMAX * N2P]
    static constexpr size_t SMEM = sizeof(float2) * (2 * SLOT + TMAX * N2P);
    static constexpr int MINB = 3;
    static_assert(N1 == 16, "TMEM layout assumes 16 points per thread");
};

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32])
{
    const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 16 complex values <-> 32 TMEM columns of this thread's lane
__device__ __forceinline__ void tm_load16(uint32_t taddr, float2 (&v)[16])
{
    float f[32];
    sm100::tmem_ld32(taddr, f);
    sm100::tmem_ld_wait();
#pragma unroll
    for (int q = 0; q < 16; q++)
        v[q] = float2{f[2 * q], f[2 * q + 1]};
}
__device__ __forceinline__ void tm_store16(uint32_t taddr, const float2 (&v)[16])
{
    float f[32];
#pragma unroll
    for (int q = 0; q < 16; q++) {
        f[2 * q] = v[q].x;
        f[2 * q + 1] = v[q].y;
    }
    tmem_st32(taddr, f);
    tmem_st_wait();
}

template<int N1, int N2>
__global__ void __launch_bounds__(RankCfg<N1, N2>::NT, 3)
    k_normal_rank_tm(RankArgs a, const __grid_constant__ CUtensorMap tmap, const unsigned char* __restrict__ plans)
{
    using namespace fftd;
    using Cfg = RankTmCfg<N1, N2>;
    constexpr int Y = Cfg::Y, W = Cfg::W, NT = Cfg::NT, JH = Cfg::JH, TMAX = Cfg::TMAX, N2P = Cfg::N2P;
    extern __shared__ __align__(128) float2 rank_tm_smem[];
    float2* ring = rank_tm_smem;                 // [2][SLOT]
    float2* ttw = ring + 2 * Cfg::SLOT;
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ float s_beta;
    __shared__ float2 s_lam;
    __shared__ uint32_t s_tmem;
    __shared__ __align__(16) RankPlanSm<N1, N2> pl;

    const int tid = threadIdx.x, warp = tid >> 5;
    const int w = tid % W, j0 = tid / W;
    const bool active = j0 < N2;
    const int j = active ? j0 : N2 - 1;
    const int C = int(a.C), nxb = int(a.nxb);
    const int U = int(a.units);
    const int u_begin = int(long(U) * blockIdx.x / a.G), u_end = int(long(U) * (blockIdx.x + 1) / a.G);
    const int n = u_end - u_begin;

    auto issue = [&](int u, int slot) {
        const int s = u / C, c = u - s * C;
        const int b = s / nxb, xblk = s - b * nxb;
        const int row0 = Y * (c + C * b);
        sm100::mbar_arrive_expect_tx(&s_bar[slot], uint32_t(Cfg::SLOT * sizeof(float2)));
#pragma unroll
        for (int k = 0; k < RankCfg<N1, N2>::NBOX; k++)
            sm100::tma_load_2d(ring + slot * Cfg::SLOT + k * RankCfg<N1, N2>::BOXR * W, &tmap, &s_bar[slot],
                               2 * W * xblk, row0 + k * RankCfg<N1, N2>::BOXR);
    };
    if (tid == 0) {
        sm100::prefetch_tmap(&tmap);
        sm100::mbar_init(&s_bar[0], 1);
        sm100::mbar_init(&s_bar[1], 1);
        sm100::fence_barrier_init();
        if (n > 0)
            issue(u_begin, 0);
        s_beta = a.mode == 1 ? cg_prologue(a.cg, a.it, a.errflags) : 0.f;
        s_lam = a.lam ? a.lam[0] : float2{0.f, 0.f};
    }
    if (warp == 0)
        sm100::tmem_alloc<128>(&s_tmem);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    // this thread's lane: warps 0-3 own lane quarters 0-3 at columns 0..63,
    // warps 4-5 lane quarters 0-1 at columns 64..127; acc at +0, x at +32
    const uint32_t tbase = s_tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * 64);
    const uint32_t t_acc = tbase, t_x = tbase + 32;
    const float beta = s_beta;
    const bool stop = a.mode == 1 && beta < 0.f;
    const bool upd = a.mode == 1 && a.it > 0;
    const float2 lam = s_lam;
    constexpr float invN1 = 1.f / float(N1);

    int plan_b = -1;
    int n_items = 0, my_h = 0, my_k1 = 0, my_ww = 0, my_md = 0, my_nt = 0, my_off = 0;
    bool my_item = false;
    double2 part{0, 0};
    float2 cv[N1];
    int seg_s = u_begin / C;
    int c_cur = u_begin - seg_s * C;
    bool seg_first = c_cur == 0;

    for (int i = 0; i <= n && !stop; i++) {
        const bool opens = i < n && (i == 0 || c_cur == 0);
        if (i >= 1) {
            // ---- C(i-1): inverse DFT over k1 (rows at the slot's own addresses), accumulate
            const float2* Sp = ring + ((i - 1) & 1) * Cfg::SLOT + j * W + w;
            float2 v[N1], acc[N1];
#pragma unroll
            for (int k1 = 0; k1 < N1; k1++)
                v[k1] = Sp[N2 * W * k1];
            dft_reg<N1, +1>(v);
            tm_load16(t_acc, acc);
#pragma unroll
            for (int q = 0; q < N1; q++) {
                const float2 t = cmulc(v[q], cv[q]);
                acc[q].x += t.x;
                acc[q].y += t.y;
            }
            if (i == n || c_cur == 0) {
                // ---- segment epilogue
                float2 xv[N1];
                tm_load16(t_x, xv);
                const int b = seg_s / nxb, xx = (seg_s - b * nxb) * W + w;
                const long img_base = xx + a.X * Y * long(b);
                cfloat* dst = rank_plane_dst(a, seg_s, blockIdx.x);
#pragma unroll
                for (int q = 0; q < N1; q++) {
                    const int y = j + N2 * q;
                    float2 o{acc[q].x * invN1, acc[q].y * invN1};
                    if (seg_first) {
                        const float2 lx = cmul(xv[q], lam);
                        o.x += lx.x;
                        o.y += lx.y;
                    }
                    if (active && xx < a.X) {
                        dst[img_base + a.X * y] = o;
                        part.x += double(xv[q].x) * o.x + double(xv[q].y) * o.y;
                        part.y += double(xv[q].y) * o.x - double(xv[q].x) * o.y;
                    }
                }
            } else {
                tm_store16(t_acc, acc);
            }
        }
        if (i < n) {
            if (opens) {
                if (i > 0)
                    seg_s++;
                seg_first = c_cur == 0;
                const int b = seg_s / nxb;
                if (b != plan_b && (plan_b < 0 || a.ps.sb != 0)) {
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
                // ---- open a segment: x (or p = r + beta p_prev) strip -> TMEM, acc = 0
                const int xx = (seg_s - b * nxb) * W + w;
                const bool colok = active && xx < a.X;
                const long img_base = xx + a.X * Y * long(b);
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
                    if (upd) {
                        v[q] = float2{v[q].x + beta * pv[q].x, v[q].y + beta * pv[q].y};
                        if (seg_first && colok)
                            a.p_out[img_base + a.X * (j + N2 * q)] = v[q];
                    }
                    pv[q] = float2{0.f, 0.f};
                }
                tm_store16(t_x, v);
                tm_store16(t_acc, pv);
            }
            // ---- A(i): coil multiply, DFT over q, in place in the slot
            const int slot = i & 1;
            float2* Sp = ring + slot * Cfg::SLOT + j * W + w;
            sm100::mbar_wait(&s_bar[slot], uint32_t((i >> 1) & 1));
            float2 v[N1];
            tm_load16(t_x, v);
#pragma unroll
            for (int q = 0; q < N1; q++)
                cv[q] = Sp[N2 * W * q];
#pragma unroll
            for (int q = 0; q < N1; q++)
                v[q] = cmul(cv[q], v[q]);
            dft_reg<N1, -1>(v);
            __syncwarp(); // padding lanes alias real rows: every lane has read before any writes
            if (active) {
#pragma unroll
                for (int k1 = 0; k1 < N1; k1++)
                    Sp[N2 * W * k1] = v[k1];
            }
        }
        __syncthreads();
        if (i >= n)
            break;
        c_cur = c_cur + 1 == C ? 0 : c_cur + 1;
        // unit i - 1 finished C: its slot takes unit i + 1
        if (tid == 0 && i + 1 < n)
            issue(u_begin + i + 1, (i + 1) & 1);
        // ---- B(i): rows at pitch N2 (row k1 = S[k1 * N2 * W ..]); half h = 1 has N2 - JH valid j
        float2* S = ring + (i & 1) * Cfg::SLOT;
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
            float2* row = S + k1 * N2 * W + ww;
            const unsigned pmask = 3u << ((tid & 31) & ~1);
            const int jb = h * JH;
            const bool last_ok = h == 0 || JH + JH - 1 < N2; // last j of the half exists
            float2 uu[JH];
#pragma unroll
            for (int jj = 0; jj < JH; jj++)
                uu[jj] = (jj < JH - 1 || last_ok) ? row[(jb + jj) * W] : float2{0.f, 0.f};
            if (nt <= 2 && off + nt <= TMAX) {
                const bool two = nt == 2;
                const float4* t0v = reinterpret_cast<const float4*>(ttw + off * N2P + jb);
                const float4* t1v = reinterpret_cast<const float4*>(ttw + (two ? off + 1 : off) * N2P + jb);
                float2 a0{0.f, 0.f}, a1{0.f, 0.f};
#pragma unroll
                for (int jj = 0; jj < JH; jj++) {
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
                a0.x += __shfl_xor_sync(pmask, a0.x, 1);
                a0.y += __shfl_xor_sync(pmask, a0.y, 1);
                a1.x += __shfl_xor_sync(pmask, a1.x, 1);
                a1.y += __shfl_xor_sync(pmask, a1.y, 1);
                a0 = nt > 0 ? cmul(a0, pl.coef[off]) : float2{0.f, 0.f};
                a1 = two ? cmul(a1, pl.coef[off + 1]) : float2{0.f, 0.f};
                auto scatter = [&](auto keep) {
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
                        if (jj < JH - 1 || last_ok)
                            row[(jb + jj) * W] = r;
                    }
                };
                if (md == 1)
                    scatter(std::true_type{});
                else
                    scatter(std::false_type{});
            } else {
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
    if (stop) {
        // CG already stopped: drain the TMA before leaving
        if (n > 0)
            sm100::mbar_wait(&s_bar[0], 0);
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        sm100::tc_fence_after();
        sm100::tmem_dealloc<128>(s_tmem);
    }
    if (a.mode == 1 && !stop) {
        part = block_sum2(part);
        publish_partial(a.cg->part_pap, &a.cg->pap_sum, &a.cg->cnt_pap, part);
    }
}

template<int N1, int N2>
void launch_rank_tm_t(RankArgs a, const cfloat* coils, const SenseGeom& g, const unsigned char* plans)
{
    using Cfg = RankTmCfg<N1, N2>;
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(2 * g.X), cuuint64_t(g.Y * g.C * g.B)};
    cuuint64_t strides[1] = {cuuint64_t(2 * g.X) * 4};
    cuuint32_t box[2] = {cuuint32_t(2 * Cfg::W), cuuint32_t(RankCfg<N1, N2>::BOXR)};
    cuuint32_t es[2] = {1, 1};
    CUresult res = rank_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<cfloat*>(coils), dims, strides,
                                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled(coils) failed: " + std::to_string(int(res)));
    auto kern = k_normal_rank_tm<N1, N2>;
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM)));
        attr = true;
    }
    const double xyb = double(g.X) * g.Y * g.B;
    const double work = 8.0 * xyb * (g.C + (a.mode == 1 ? 4 : 2));
    ProfScope prof(a.mode == 1 ? "sense_normal_y_cg" : "sense_normal_y", work);
    kern<<<a.G, Cfg::NT, Cfg::SMEM, ctx().stream>>>(a, m, plans);
    KERNEL_CHECK();
}
