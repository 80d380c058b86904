// Device FFT building blocks.
//
// Reference semantics (fft.hpp:23-226): unitary (1/sqrt n per axis),
// uncentred (DC at index 0) DFT, twiddles evaluated in double and rounded to
// float.  The reference runs radix-2 / Bluestein per line on one CPU thread;
// here every length is factored into compile-time radices:
//   * dft_reg<R,DIR>: an R-point DFT held entirely in registers, fully
//     unrolled with twiddle constants computed at compile time in double
//     (constexpr Taylor series) — composite R by in-register Cooley-Tukey,
//     prime R by the symmetric (x_j +- x_{R-j}) direct form, 4h^2 FMAs.
//   * smem Stockham autosort stages between radices (runtime plan), with
//     per-stage twiddle tables precomputed on the host in double.
#pragma once

#include <cuda_runtime.h>

namespace mdnn {
namespace fftd {

constexpr double kPi = 3.14159265358979323846264338327950288;

// accurate constexpr sin/cos of 2*pi*m/R (exact quadrant handling)
constexpr double cx_sin_small(double x)
{
    double term = x, sum = x;
    for (int n = 1; n < 16; n++) {
        term *= -x * x / double((2 * n) * (2 * n + 1));
        sum += term;
    }
    return sum;
}
constexpr double cx_cos_small(double x)
{
    double term = 1, sum = 1;
    for (int n = 1; n < 16; n++) {
        term *= -x * x / double((2 * n - 1) * (2 * n));
        sum += term;
    }
    return sum;
}
// cos(2 pi m / R)
constexpr double cos2pi(long m, long R)
{
    m %= R;
    if (m < 0)
        m += R;
    if (4 * m == R || 4 * m == 3 * R)
        return 0.0;
    if (2 * m == R)
        return -1.0;
    if (m == 0)
        return 1.0;
    double x = 2.0 * kPi * double(m) / double(R);
    if (x > kPi)
        x -= 2.0 * kPi;
    return cx_cos_small(x);
}
constexpr double sin2pi(long m, long R)
{
    m %= R;
    if (m < 0)
        m += R;
    if (m == 0 || 2 * m == R)
        return 0.0;
    if (4 * m == R)
        return 1.0;
    if (4 * m == 3 * R)
        return -1.0;
    double x = 2.0 * kPi * double(m) / double(R);
    if (x > kPi)
        x -= 2.0 * kPi;
    return cx_sin_small(x);
}

constexpr int smallest_factor(int R)
{
    if (R % 4 == 0 && R != 4)
        return 4;
    for (int f = 2; f * f <= R; f++)
        if (R % f == 0)
            return f;
    return R;
}

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return {a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) { return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y}; }
__device__ __forceinline__ float2 cconj(float2 a) { return {a.x, -a.y}; }

// multiply by exp(DIR * 2 pi i m / R), exact for multiples of a quarter turn
template<int M_, int R, int DIR>
__device__ __forceinline__ float2 rot(float2 v)
{
    constexpr long m = ((long(M_) % R) + R) % R;
    if constexpr (m == 0) {
        return v;
    } else if constexpr (2 * m == R) {
        return {-v.x, -v.y};
    } else if constexpr (4 * m == R) { // angle pi/2 * DIR
        return DIR > 0 ? float2{-v.y, v.x} : float2{v.y, -v.x};
    } else if constexpr (4 * m == 3 * R) {
        return DIR > 0 ? float2{v.y, -v.x} : float2{-v.y, v.x};
    } else {
        constexpr float c = float(cos2pi(m, R));
        constexpr float s = float(DIR * sin2pi(m, R));
        return {v.x * c - v.y * s, v.x * s + v.y * c};
    }
}

template<int R, int DIR>
struct Dft;

template<int R, int DIR>
__device__ __forceinline__ void dft_reg(float2 (&v)[R])
{
    Dft<R, DIR>::run(v);
}

template<int DIR>
struct Dft<1, DIR> {
    __device__ __forceinline__ static void run(float2 (&)[1]) {}
};

template<int DIR>
struct Dft<2, DIR> {
    __device__ __forceinline__ static void run(float2 (&v)[2])
    {
        float2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    }
};

template<int DIR>
struct Dft<4, DIR> {
    __device__ __forceinline__ static void run(float2 (&v)[4])
    {
        float2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
        float2 a2 = cadd(v[1], v[3]), a3 = csub(v[1], v[3]);
        // i*DIR*a3
        float2 ja3 = DIR > 0 ? float2{-a3.y, a3.x} : float2{a3.y, -a3.x};
        v[0] = cadd(a0, a2);
        v[2] = csub(a0, a2);
        v[1] = cadd(a1, ja3);
        v[3] = csub(a1, ja3);
    }
};

// prime (or generic odd) R: symmetric direct form.  j and k are template
// parameters so every cos/sin is a compile-time constant (FFMA immediates).
template<int R, int k, int j>
__device__ __forceinline__ void direct_acc(float2& A, float2& B, const float2* s, const float2* d)
{
    if constexpr (j <= (R - 1) / 2) {
        constexpr float c = float(cos2pi(long(j) * k, R));
        constexpr float sn = float(sin2pi(long(j) * k, R));
        A.x = fmaf(s[j].x, c, A.x);
        A.y = fmaf(s[j].y, c, A.y);
        B.x = fmaf(d[j].x, sn, B.x);
        B.y = fmaf(d[j].y, sn, B.y);
        direct_acc<R, k, j + 1>(A, B, s, d);
    }
}

template<int R, int DIR, int k>
__device__ __forceinline__ void direct_out(float2 (&v)[R], float2 x0, const float2* s, const float2* d)
{
    if constexpr (k <= (R - 1) / 2) {
        float2 A = x0, B = {0.f, 0.f};
        direct_acc<R, k, 1>(A, B, s, d);
        // X_k = A + i*DIR*B ; X_{R-k} = A - i*DIR*B
        float2 iB = DIR > 0 ? float2{-B.y, B.x} : float2{B.y, -B.x};
        v[k] = cadd(A, iB);
        v[R - k] = csub(A, iB);
        direct_out<R, DIR, k + 1>(v, x0, s, d);
    }
}

template<int R, int DIR, bool PRIME>
struct DftDirect {
    __device__ __forceinline__ static void run(float2 (&v)[R])
    {
        constexpr int h = (R - 1) / 2;
        float2 s[h + 1], d[h + 1];
#pragma unroll
        for (int j = 1; j <= h; j++) {
            s[j] = cadd(v[j], v[R - j]);
            d[j] = csub(v[j], v[R - j]);
        }
        float2 x0 = v[0];
        float2 sum = x0;
#pragma unroll
        for (int j = 1; j <= h; j++)
            sum = cadd(sum, s[j]);
        direct_out<R, DIR, 1>(v, x0, s, d);
        v[0] = sum;
    }
};

// composite R = F * M (in-register Cooley-Tukey, verified in DESIGN.md §FFT)
template<int R, int DIR, int F>
struct DftComposite {
    __device__ __forceinline__ static void run(float2 (&v)[R])
    {
        constexpr int M = R / F;
        float2 Y[M][F];
#pragma unroll
        for (int n2 = 0; n2 < M; n2++) {
            float2 t[F];
#pragma unroll
            for (int n1 = 0; n1 < F; n1++)
                t[n1] = v[M * n1 + n2];
            Dft<F, DIR>::run(t);
#pragma unroll
            for (int k1 = 0; k1 < F; k1++)
                Y[n2][k1] = t[k1];
        }
        twiddle<0, 0>(Y);
#pragma unroll
        for (int k1 = 0; k1 < F; k1++) {
            float2 t[M];
#pragma unroll
            for (int n2 = 0; n2 < M; n2++)
                t[n2] = Y[n2][k1];
            Dft<M, DIR>::run(t);
#pragma unroll
            for (int k2 = 0; k2 < M; k2++)
                v[k1 + F * k2] = t[k2];
        }
    }
    template<int n2, int k1>
    __device__ __forceinline__ static void twiddle(float2 (&Y)[R / F][F])
    {
        if constexpr (n2 < R / F) {
            if constexpr (k1 < F) {
                Y[n2][k1] = rot<n2 * k1, R, DIR>(Y[n2][k1]);
                twiddle<n2, k1 + 1>(Y);
            } else {
                twiddle<n2 + 1, 0>(Y);
            }
        }
    }
};

template<int R, int DIR>
struct Dft {
    __device__ __forceinline__ static void run(float2 (&v)[R])
    {
        constexpr int f = smallest_factor(R);
        if constexpr (f == R)
            DftDirect<R, DIR, true>::run(v);
        else
            DftComposite<R, DIR, f>::run(v);
    }
};

// ---------------------------------------------------------------------------
// Runtime plan for the smem Stockham path
// ---------------------------------------------------------------------------
constexpr int kMaxStages = 8;
struct Plan {
    int n;
    int nstages;
    int radix[kMaxStages];
    int ns[kMaxStages];            // product of previous radices
    const float2* tw[kMaxStages];  // [k*(R-1) + q-1] = exp(-2 pi i q k / (ns R)), k < ns
};

// One forward Stockham stage over W interleaved lines stored as buf[k*W + w].
template<int R>
__device__ __forceinline__ void stockham_stage(const float2* __restrict__ in, float2* __restrict__ out, int n, int ns,
                                               const float2* __restrict__ tw, int W, int tid, int nthreads)
{
    const int nb = n / R;
    for (int e = tid; e < nb * W; e += nthreads) {
        const int w = e % W;
        const int j = e / W;
        const int k = j % ns;
        float2 v[R];
#pragma unroll
        for (int q = 0; q < R; q++)
            v[q] = in[(j + q * nb) * W + w];
        if (ns > 1) {
#pragma unroll
            for (int q = 1; q < R; q++)
                v[q] = cmul(v[q], __ldg(&tw[k * (R - 1) + q - 1]));
        }
        dft_reg<R, -1>(v);
        const int dst = (j / ns) * ns * R + k;
#pragma unroll
        for (int q = 0; q < R; q++)
            out[(dst + q * ns) * W + w] = v[q];
    }
}

// Dispatch a stage by runtime radix (warp-uniform).
__device__ __forceinline__ void run_stage(int R, const float2* in, float2* out, int n, int ns, const float2* tw, int W,
                                          int tid, int nthreads)
{
    switch (R) {
    case 2: stockham_stage<2>(in, out, n, ns, tw, W, tid, nthreads); break;
    case 3: stockham_stage<3>(in, out, n, ns, tw, W, tid, nthreads); break;
    case 4: stockham_stage<4>(in, out, n, ns, tw, W, tid, nthreads); break;
    case 5: stockham_stage<5>(in, out, n, ns, tw, W, tid, nthreads); break;
    case 7: stockham_stage<7>(in, out, n, ns, tw, W, tid, nthreads); break;
    case 8: stockham_stage<8>(in, out, n, ns, tw, W, tid, nthreads); break;
    case 11: stockham_stage<11>(in, out, n, ns, tw, W, tid, nthreads); break;
    case 13: stockham_stage<13>(in, out, n, ns, tw, W, tid, nthreads); break;
    case 16: stockham_stage<16>(in, out, n, ns, tw, W, tid, nthreads); break;
    case 17: stockham_stage<17>(in, out, n, ns, tw, W, tid, nthreads); break;
    case 19: stockham_stage<19>(in, out, n, ns, tw, W, tid, nthreads); break;
    case 23: stockham_stage<23>(in, out, n, ns, tw, W, tid, nthreads); break;
    case 29: stockham_stage<29>(in, out, n, ns, tw, W, tid, nthreads); break;
    case 31: stockham_stage<31>(in, out, n, ns, tw, W, tid, nthreads); break;
    default: break; // rejected at plan time
    }
}

// Forward FFT of W lines in smem (buf layout [k*W + w]); returns the buffer
// holding the result (a or b).  Unnormalised.
__device__ __forceinline__ float2* fft_smem(float2* a, float2* b, const Plan& p, int W)
{
    float2* in = a;
    float2* out = b;
    for (int s = 0; s < p.nstages; s++) {
        run_stage(p.radix[s], in, out, p.n, p.ns[s], p.tw[s], W, threadIdx.x, blockDim.x);
        __syncthreads();
        float2* t = in;
        in = out;
        out = t;
    }
    return in;
}

} // namespace fftd

// host: cached plan for length n (device twiddle tables live for the process)
const fftd::Plan& fft_plan(int n);
bool fft_supported(long n);

} // namespace mdnn
