// Register-resident fused A^H A (+ lambda) for Y = N1 * N2 (included by sense.cu).
//
// Per CTA: W image columns x all Y rows of one item, a contiguous range of
// coils (coil-split across nsplit CTAs against the wave tail; the partial
// results land in nsplit planes that the CG update sums, and <p, Ap> is linear
// in Ap so its per-CTA partials stay exact).  Per coil, with y = j + N2*q:
//   stage A  thread (w, j):   v[q] = C[y] x[y]  -> DFT_N1 over q -> twiddle
//                              W_Y^{j k1} -> smem S[k1][j]
//   stage B  thread (w, k1):  DFT_N2 over j -> spectrum X[k1 + N1 k2]
//                              -> mask P/Y -> IDFT_N2 -> conj twiddle -> S
//   stage C  thread (w, j):   IDFT_N1 over k1 -> acc[q] += conj(C[y]) v[q]
// Stage A and C threads own the same y positions, so the coil values read for
// stage A are reused for the combine and the accumulators never leave
// registers.  The next coil's W x Y slice is prefetched into shared memory
// with cp.async (zero-filled past the image edge) while stages B and C of the
// current coil run, so no warp waits on HBM inside the coil loop.  S is
// double-buffered by coil parity: 2 barriers per coil.
#pragma once

template<int N1, int N2, int W>
constexpr int fast_threads()
{
    return ((W * N2 + 31) / 32) * 32; // whole warps: block_sum2 needs full warps
}

__device__ __forceinline__ void cp_async8(float2* dst, const float2* src, bool valid)
{
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const int sz = valid ? 8 : 0; // src-size 0: zero fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// ---------------------------------------------------------------------------
// Mask-pruned stage B.  With k = k1 + N1 k2 the row k1 of stage B applies
//   M_k1 = sum_k2 (p_k / Y) w_k w_k^H,   w_k[j] = exp(+2 pi i j k / Y),
// to the untwiddled stage-A row A[k1][.] (stage A's W_Y^{j k1} twiddle and
// stage C's conjugate cancel into w_k).  Expanding against the identity,
// sum_k2 w_k w_k^H / Y = (N2 / Y) I, so with b in {0, 1}
//   M_k1 = (N2 / Y) (b I + sum_{k2 : p_k != b} ((p_k - b) / N2) w_k w_k^H),
// an exact rewrite with min(#{p != 0}, #{p != 1}) rank-1 terms.  A fully
// sampled row (every 4th line of the reference's make_pattern) is the
// identity and costs nothing; an ACL row costs one or two dot/axpy pairs of
// length N2; rows with more than KMAX terms run the full in-register DFT.
// The common factor N2 / Y = 1 / N1 is applied once in the epilogue.
// Per-CTA plan, built in the prologue from the (per-item) pattern:
//   s_nt[k1]   terms of row k1 (-1: full DFT row)
//   s_bb[k1]   b of row k1
//   s_toff[k1] first term index; term t: s_coef[t], twiddle row ttw[t][j]
//   s_row[s]   row of stage-B slot s, sorted by cost (warp-coherent loops)
// ---------------------------------------------------------------------------
template<int N2>
constexpr int prune_kmax()
{
    return (N2 % 2 == 1) ? 5 : 2; // rank-1 pair ~ 8 N2 FMA vs DFT pair cost
}
template<int N1>
constexpr int prune_tmax()
{
    return 3 * N1;
}

template<int N1, int N2, int W>
constexpr size_t fast_smem_bytes()
{
    return sizeof(float2) * (2 * N1 * N2 * W + 2 * N1 * N2 + 2 * N1 * N2 * W + prune_tmax<N1>() * N2);
}
// CTAs per SM the shared memory allows (register budget follows it)
template<int N1, int N2, int W>
constexpr int fast_min_blocks()
{
    return 2 * (fast_smem_bytes<N1, N2, W>() + 3 * 1024) <= 228 * 1024 ? 2 : 1;
}

template<int N1, int N2, int W>
__global__ void __launch_bounds__(fast_threads<N1, N2, W>(), (fast_min_blocks<N1, N2, W>()))
    k_normal_fast(NormalArgs a, const float2* __restrict__ tw, cfloat* __restrict__ p_out, long plane)
{
    MDNN_PDL_ENTRY();
    using namespace fftd;
    constexpr int Y = N1 * N2;
    constexpr int NT = fast_threads<N1, N2, W>();
    constexpr int KMAX = prune_kmax<N2>();
    constexpr int TMAX = prune_tmax<N1>();
    extern __shared__ float2 dsm[];
    float2* S0 = dsm;                 // [2][N1 * N2 * W]
    float2* stw = S0 + 2 * Y * W;     // [Y]  exp(-2 pi i m / Y)
    float2* spat = stw + Y;           // [Y]  p / N2 (full rows)
    float2* xs = spat + Y;            // [Y * W]
    float2* scoil = xs + Y * W;       // [Y * W] next coil slice
    float2* ttw = scoil + Y * W;      // [TMAX][N2] term twiddle rows
    __shared__ float s_beta;
    __shared__ float2 s_lam;
    __shared__ int s_nt[N1], s_bb[N1], s_toff[N1], s_row[N1], s_tk[TMAX], s_ntot;
    __shared__ float2 s_coef[TMAX];

    const int tid = threadIdx.x;
    const int w = tid % W, j0 = tid / W;
    const bool active = j0 < N2;      // padding lanes only join barriers / reductions
    const int j = active ? j0 : 0;
    const long nxb = (a.X + W - 1) / W;
    long blk = blockIdx.x;
    const int split = int(blk % a.nsplit);
    blk /= a.nsplit;
    const long x0 = (blk % nxb) * W, b = blk / nxb;
    const long xx = x0 + w;
    const bool colok = active && xx < a.X;
    const long c_begin = a.C * split / a.nsplit, c_end = a.C * (split + 1) / a.nsplit;
    const float invN2 = 1.f / float(N2);

    // prefetch the first coil slice (thread (w, j) copies the rows it will read)
    auto prefetch = [&](long c) {
        if (!active)
            return;
        const float2* src = a.coils + (colok ? xx : 0) + a.X * a.Y * (c + a.C * b);
#pragma unroll
        for (int q = 0; q < N1; q++)
            cp_async8(scoil + (j + N2 * q) * W + w, src + a.X * (j + N2 * q), colok);
    };
    if (c_begin < c_end)
        prefetch(c_begin);
    cp_async_commit();

    for (int e = tid; e < Y; e += NT) {
        stw[e] = tw[e];
        float2 pv = a.pattern[e * a.ps.sy + b * a.ps.sb];
        spat[e] = float2{pv.x * invN2, pv.y * invN2};
    }
    // ---- row plan: thread k1 classifies its row
    if (tid < N1) {
        const int k1 = tid;
        int nz = 0, n1 = 0;
        for (int k2 = 0; k2 < N2; k2++) {
            const float2 pv = a.pattern[(k1 + N1 * k2) * a.ps.sy + b * a.ps.sb];
            nz += (pv.x != 0.f || pv.y != 0.f);
            n1 += (pv.x != 1.f || pv.y != 0.f);
        }
        s_bb[k1] = nz <= n1 ? 0 : 1;
        s_nt[k1] = min(nz, n1);
    }
    if (tid == 0) {
        s_beta = a.mode == 1 ? cg_prologue(a.cg, a.it, a.errflags) : 0.f;
        s_lam = a.lam ? a.lam[0] : float2{0.f, 0.f};
    }
    __syncthreads();
    if (tid == 0) {
        // term slots in row order (rows over KMAX or past TMAX go full), then
        // slot order sorted by cost (insertion sort of N1 keys)
        int off = 0;
        int cost[N1];
        for (int k1 = 0; k1 < N1; k1++) {
            int nt = s_nt[k1];
            if (nt > KMAX || off + nt > TMAX)
                nt = -1;
            s_nt[k1] = nt;
            s_toff[k1] = off;
            off += nt > 0 ? nt : 0;
            cost[k1] = nt < 0 ? 1 << 20 : nt;
            s_row[k1] = k1;
        }
        for (int i = 1; i < N1; i++) {
            const int r = s_row[i], cr = cost[r];
            int k = i - 1;
            while (k >= 0 && cost[s_row[k]] > cr) {
                s_row[k + 1] = s_row[k];
                k--;
            }
            s_row[k + 1] = r;
        }
        s_ntot = off;
    }
    __syncthreads();
    if (tid < N1) {
        const int k1 = tid, nt = s_nt[k1], bb = s_bb[k1];
        int t = s_toff[k1];
        if (nt > 0)
            for (int k2 = 0; k2 < N2; k2++) {
                const float2 pv = a.pattern[(k1 + N1 * k2) * a.ps.sy + b * a.ps.sb];
                if (pv.x != float(bb) || pv.y != 0.f) {
                    s_tk[t] = k1 + N1 * k2;
                    s_coef[t] = float2{(pv.x - float(bb)) * invN2, pv.y * invN2};
                    t++;
                }
            }
    }
    __syncthreads();
    for (int e = tid; e < s_ntot * N2; e += NT) {
        const int t = e / N2, jj = e % N2;
        ttw[e] = stw[(jj * s_tk[t]) % Y];
    }
    const float beta = s_beta;
    if (a.mode == 1 && beta < 0.f) {
        cp_async_wait_all();
        return;
    }

    // image column strip (x, or p = r + beta p_prev) -> smem
    // all loads first (p_out may alias nothing we read, but the compiler
    // cannot know: interleaving the stores would serialise the loads)
    const long img_base = xx + a.X * a.Y * b;
    {
        float2 v[N1], pv[N1];
        const float2* src = a.mode == 0 ? a.x : (a.it == 0 ? p_out : a.x);
        const bool upd = a.mode == 1 && a.it > 0;
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
                if (split == 0 && colok)
                    p_out[img_base + a.X * y] = v[q];
            }
            if (active)
                xs[y * W + w] = v[q];
        }
    }
    cp_async_wait_all();
    __syncthreads();

    float2 acc[N1];
#pragma unroll
    for (int q = 0; q < N1; q++)
        acc[q] = float2{0.f, 0.f};

    // stage-B slot of this thread
    const int wb = tid % W, slot = tid / W;
    const int rowk1 = slot < N1 ? s_row[slot] : 0;
    const int row_nt = slot < N1 ? s_nt[rowk1] : 0;
    const int row_bb = slot < N1 ? s_bb[rowk1] : 1;
    const int row_off = slot < N1 ? s_toff[rowk1] : 0;
    const bool row_work = slot < N1 && !(row_nt == 0 && row_bb == 1); // identity rows: nothing to do

    for (long c = c_begin; c < c_end; c++) {
        float2* Sb = S0 + (c & 1) * (Y * W);
        // ---- stage A: coil multiply, DFT over q -> S (untwiddled)
        float2 cv[N1], v[N1];
#pragma unroll
        for (int q = 0; q < N1; q++)
            cv[q] = scoil[(j + N2 * q) * W + w];
#pragma unroll
        for (int q = 0; q < N1; q++)
            v[q] = cmul(cv[q], xs[(j + N2 * q) * W + w]);
        dft_reg<N1, -1>(v);
        if (active) {
#pragma unroll
            for (int k1 = 0; k1 < N1; k1++)
                Sb[(k1 * N2 + j) * W + w] = v[k1];
        }
        __syncthreads();
        // scoil is free: fetch the next coil while stages B and C run
        if (c + 1 < c_end)
            prefetch(c + 1);
        cp_async_commit();
        // ---- stage B: per row, identity / rank-1 terms / full DFT
        if (row_work) {
            float2* row = Sb + rowk1 * N2 * W + wb;
            float2 u[N2];
            if (row_nt < 0) {
#pragma unroll
                for (int jj = 0; jj < N2; jj++)
                    u[jj] = row[jj * W];
#pragma unroll
                for (int jj = 1; jj < N2; jj++)
                    u[jj] = cmul(u[jj], stw[jj * rowk1]);
                dft_reg<N2, -1>(u);
#pragma unroll
                for (int k2 = 0; k2 < N2; k2++)
                    u[k2] = cmul(u[k2], spat[rowk1 + N1 * k2]);
                dft_reg<N2, +1>(u);
#pragma unroll
                for (int jj = 1; jj < N2; jj++)
                    u[jj] = cmulc(u[jj], stw[jj * rowk1]);
            } else {
                float2 d[KMAX];
                if (row_nt > 0) {
#pragma unroll
                    for (int jj = 0; jj < N2; jj++)
                        u[jj] = row[jj * W];
                }
#pragma unroll
                for (int t = 0; t < KMAX; t++) {
                    if (t < row_nt) {
                        const float2* tt = ttw + (row_off + t) * N2;
                        float2 e0{0.f, 0.f}, e1{0.f, 0.f};
#pragma unroll
                        for (int jj = 0; jj < N2; jj += 2) {
                            const float2 tv = tt[jj];
                            e0.x = fmaf(u[jj].x, tv.x, e0.x);
                            e0.y = fmaf(u[jj].x, tv.y, e0.y);
                            e0.x = fmaf(-u[jj].y, tv.y, e0.x);
                            e0.y = fmaf(u[jj].y, tv.x, e0.y);
                            if (jj + 1 < N2) {
                                const float2 tv1 = tt[jj + 1];
                                e1.x = fmaf(u[jj + 1].x, tv1.x, e1.x);
                                e1.y = fmaf(u[jj + 1].x, tv1.y, e1.y);
                                e1.x = fmaf(-u[jj + 1].y, tv1.y, e1.x);
                                e1.y = fmaf(u[jj + 1].y, tv1.x, e1.y);
                            }
                        }
                        d[t] = cmul(float2{e0.x + e1.x, e0.y + e1.y}, s_coef[row_off + t]);
                    }
                }
                if (row_bb == 0) {
#pragma unroll
                    for (int jj = 0; jj < N2; jj++)
                        u[jj] = float2{0.f, 0.f};
                }
#pragma unroll
                for (int t = 0; t < KMAX; t++) {
                    if (t < row_nt) {
                        const float2* tt = ttw + (row_off + t) * N2;
                        const float2 dt = d[t];
#pragma unroll
                        for (int jj = 0; jj < N2; jj++) {
                            const float2 tv = tt[jj]; // u += d conj(tv)
                            u[jj].x = fmaf(dt.x, tv.x, u[jj].x);
                            u[jj].y = fmaf(dt.y, tv.x, u[jj].y);
                            u[jj].x = fmaf(dt.y, tv.y, u[jj].x);
                            u[jj].y = fmaf(-dt.x, tv.y, u[jj].y);
                        }
                    }
                }
            }
#pragma unroll
            for (int jj = 0; jj < N2; jj++)
                row[jj * W] = u[jj];
        }
        cp_async_wait_all();
        __syncthreads();
        // ---- stage C: inverse DFT over k1, conj-coil accumulate
#pragma unroll
        for (int k1 = 0; k1 < N1; k1++)
            v[k1] = Sb[(k1 * N2 + j) * W + w];
        dft_reg<N1, +1>(v);
#pragma unroll
        for (int q = 0; q < N1; q++) {
            const float2 t = cmulc(v[q], cv[q]);
            acc[q].x += t.x;
            acc[q].y += t.y;
        }
    }

    // ---- epilogue: common 1/N1, + lambda x (split 0), store plane, <p, Ap> partial
    constexpr float invN1 = 1.f / float(N1);
    double2 part{0, 0};
#pragma unroll
    for (int q = 0; q < N1; q++) {
        const int y = j + N2 * q;
        const float2 xv = xs[y * W + w];
        float2 o{acc[q].x * invN1, acc[q].y * invN1};
        if (split == 0) {
            const float2 lx = cmul(xv, s_lam);
            o.x += lx.x;
            o.y += lx.y;
        }
        if (colok) { // padding lanes: colok false, part stays 0
            a.out[plane * split + img_base + a.X * y] = o;
            part.x += double(xv.x) * o.x + double(xv.y) * o.y;
            part.y += double(xv.y) * o.x - double(xv.x) * o.y;
        }
    }
    if (a.mode == 1) {
        part = block_sum2(part);
        publish_partial(a.cg->part_pap, &a.cg->pap_sum, &a.cg->cnt_pap, part);
    }
}


// forward twiddles tw[m] = exp(-2 pi i m / Y), m < Y, double-accurate, per (device, Y)
const float2* fast_twiddles(int N1, int N2)
{
    static std::mutex mu;
    static std::map<std::pair<int, int>, float2*> cache;
    auto& c = ctx();
    const int Y = N1 * N2;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(c.device, Y * 1000 + N1);
    auto it = cache.find(key);
    if (it != cache.end())
        return it->second;
    std::vector<float2> h(Y);
    for (int m = 0; m < Y; m++) {
        const double ang = -2.0 * M_PI * double(m) / double(Y);
        h[m] = float2{float(std::cos(ang)), float(std::sin(ang))};
    }
    float2* d;
    CUDA_CHECK(cudaMalloc(&d, sizeof(float2) * Y));
    CUDA_CHECK(cudaMemcpy(d, h.data(), sizeof(float2) * Y, cudaMemcpyHostToDevice));
    cache[key] = d;
    return d;
}

template<int N1, int N2, int W>
void launch_fast(NormalArgs a, cfloat* p_out, long plane)
{
    auto kern = k_normal_fast<N1, N2, W>;
    constexpr size_t smem = fast_smem_bytes<N1, N2, W>();
    allow_max_dyn_smem(reinterpret_cast<const void*>(kern));
    const long nxb = (a.X + W - 1) / W;
    const double xyb = double(a.X) * a.Y * a.B;
    const double work = 8.0 * xyb * (a.C + (a.mode == 1 ? 4 : 2));
    ProfScope prof(a.mode == 1 ? "sense_normal_y_cg" : "sense_normal_y", work);
    pdl_launch(kern, unsigned(nxb * a.B * a.nsplit), fast_threads<N1, N2, W>(), smem, ctx().stream, a, fast_twiddles(N1, N2), p_out, plane);
    KERNEL_CHECK();
}

// (N1, N2) factorisation of Y handled by the register-resident kernel, or 0
int fast_n1(long Y)
{
    switch (Y) {
    case 128: case 256: case 320: case 368: case 512: case 640:
        return Y == 128 ? 8 : 16;
    default:
        return 0;
    }
}

bool dispatch_fast(NormalArgs a, cfloat* p_out, long plane)
{
    constexpr int W = 8;
    switch (a.Y) {
    case 128: launch_fast<8, 16, W>(a, p_out, plane); return true;
    case 256: launch_fast<16, 16, W>(a, p_out, plane); return true;
    case 320: launch_fast<16, 20, W>(a, p_out, plane); return true;
    case 368: launch_fast<16, 23, W>(a, p_out, plane); return true;
    case 512: launch_fast<16, 32, W>(a, p_out, plane); return true;
    case 640: launch_fast<16, 40, W>(a, p_out, plane); return true;
    default: return false;
    }
}

long fast_ctas(const SenseGeom& g, int nsplit) { return ((g.X + 7) / 8) * g.B * nsplit; }

// coil split minimising (waves) x (coils per CTA + ~1 coil of per-CTA overhead)
// at 2 resident CTAs per SM
int fast_nsplit(const SenseGeom& g)
{
    const long strips = (g.X + 7) / 8 * g.B, slots = 2L * ctx().sm_count;
    int best = 1;
    double best_t = 1e300;
    for (int ns = 1; ns <= std::min<long>(g.C, 8); ns++) {
        const double waves = double((strips * ns + slots - 1) / slots);
        const double t = waves * (double((g.C + ns - 1) / ns) + 1.0);
        if (t < best_t - 1e-9) {
            best_t = t;
            best = ns;
        }
    }
    return best;
}

// CG update with NSPLIT Ap planes: x += alpha p ; r -= alpha (sum of planes)
__global__ void k_cg_update_planes(CgDev* st, int it, cfloat* x, cfloat* r, const cfloat* p, const cfloat* ap,
                                   long n, int nplanes, long plane, unsigned* errflags)
{
    MDNN_PDL_ENTRY();
    __shared__ float s_alpha;
    if (threadIdx.x == 0)
        s_alpha = cg_alpha(st, it, errflags);
    __syncthreads();
    const float al = s_alpha;
    if (!(al > 0.f))
        return;
    double2 part{0, 0};
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        float2 av = ap[i];
        for (int s = 1; s < nplanes; s++) {
            const float2 t = ap[i + s * plane];
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
