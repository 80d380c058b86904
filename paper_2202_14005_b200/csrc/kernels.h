// Launchers for every device kernel of the hot path.  All launch on the
// current device context's stream (core.h); none synchronises.
#pragma once

#include "core.h"

#include <functional>
#include <vector>

namespace mdnn {

// ---- generic md helpers (ew.cu) -------------------------------------------
// dst[p.sd] = src[p.ss] over dims (strides in complex elements)
void launch_strided_copy(const Dims& dims, cfloat* dst, const Dims& sd, const cfloat* src, const Dims& ss);
void launch_layout_convert(const DArray& in, const DArray& out);

// out = a + s * b (n complex); s real
void launch_add(cfloat* out, const cfloat* a, const cfloat* b, float s, long n);
// y += alpha * x
void launch_axpy(cfloat* y, cfloat alpha, const cfloat* x, long n);
// out = s * in (complex s)
void launch_scale(cfloat* out, const cfloat* in, cfloat s, long n);
// out = scalar[0] * in, scalar read on the device; conj_s conjugates it
void launch_scale_dev(cfloat* out, const cfloat* in, const cfloat* scalar, bool conj_s, long n);
void launch_conj(cfloat* out, const cfloat* in, long n);
// out = (factor * Re(scalar[0])) * in
void launch_scale_dev_real(cfloat* out, const cfloat* in, const cfloat* scalar, float factor, long n);
// out[0] = (factor * Re(in[0]), 0)
void launch_real_scalar(cfloat* out, const cfloat* in, float factor);
void launch_real(cfloat* out, const cfloat* in, long n);
void launch_crelu(cfloat* out, const cfloat* in, long n);
void launch_crelu_mask(cfloat* out, const cfloat* d, const cfloat* x, long n);
void launch_exp_real(cfloat* out, const cfloat* in, long n);
void launch_mul_real_real(cfloat* out, const cfloat* y, const cfloat* d, long n); // out = (Re y * Re d, 0)
void launch_neg(cfloat* out, const cfloat* in, long n);

// complex split/join on a channel dim (RealChan / ChanCplx, ops.hpp:318-411):
// in [.., 1(chan), ..] -> out [.., 2, ..]; inner = prod dims before chan, outer = after
void launch_real_chan_split(cfloat* out, const cfloat* in, long inner, long outer);
void launch_real_chan_join(cfloat* out, const cfloat* in, long inner, long outer);

// Broadcast binary op over out dims with per-operand strides (0 = broadcast).
// op: 0 = a + b, 1 = a * b, 2 = a * conj(b)
void launch_bcast_binary(const Dims& dims, cfloat* out, const cfloat* a, const Dims& sa, const cfloat* b,
                         const Dims& sb, int op);

// "ISO" reductions: data viewed as [inner][stat][outer] (column-major, inner
// fastest); out[stat] = sum over inner,outer of f(a, b) computed in double,
// deterministic two-stage tree.  mode: 0 sum a; 1 sum a*conj(b); 2 sum |a|^2 (real)
void launch_iso_reduce(cfloat* out, const cfloat* a, const cfloat* b, long inner, long nstat, long outer, int mode,
                       float scale);

// Batch-global complex dot <a,b> = sum a conj(b) accumulated in double
// (mdarray.hpp:679-708) into a device double2 (no host sync).
void launch_zdot(double* out2, const cfloat* a, const cfloat* b, long n);
double host_znorm(const cfloat* a, long n);

// generic TenMul contraction (md_fmac2 / md_zfmacc2, mdarray.hpp:485-523):
// out[p.so] += in1[p.s1] * (conj?)in2[p.s2], out zeroed by the caller
void launch_fmac_generic(const Dims& iter, cfloat* out, const Dims& so, const cfloat* in1, const Dims& s1,
                         const cfloat* in2, const Dims& s2, bool conj2);

// ---- FFT (fft.cu) -----------------------------------------------------------
// unitary (1/sqrt n) uncentred DFT along one dim of a column-major array
void launch_fft_dim(cfloat* out, const cfloat* in, const Dims& dims, int dim, bool inverse);
// true if every prime factor of n has a device radix (<= 31) and n fits smem
bool fft_supported(long n);
// multi-dim dft (fft.hpp:180-226): out may equal in
void fft_flags(cfloat* out, const cfloat* in, const Dims& dims, unsigned long flags, bool inverse);

// ---- SENSE (sense.cu) ---------------------------------------------------------
struct SenseGeom {
    long X, Y, C, M, B;             // image x, y, coils, map sets, batch
    long pat_x, pat_y, pat_c, pat_b; // pattern extents (each 1 = broadcast, or full)
};
// coil images u[x,y,c,b] = sum_m C[x,y,c,m,b] x[x,y,m,b]
void launch_coil_mul(cfloat* u, const cfloat* x, const cfloat* coils, const SenseGeom& g);
// x[x,y,m,b] = sum_c conj(C[x,y,c,m,b]) u[x,y,c,b]
void launch_coil_adj(cfloat* x, const cfloat* u, const cfloat* coils, const SenseGeom& g);
// u *= pattern (broadcast over x if pattern_xinv, over coils always)
void launch_pattern_mul(cfloat* out, const cfloat* u, const cfloat* pattern, const SenseGeom& g);
// A x  = P F C x       (recon.hpp:100-110): out [X,Y,1,C,1..,B]
void sense_forward(cfloat* y, const cfloat* x, const cfloat* coils, const cfloat* pattern, const SenseGeom& g);
// A^H y = C^H F^H P y  (recon.hpp:111-121)
void sense_adjoint(cfloat* x, const cfloat* y, const cfloat* coils, const cfloat* pattern, const SenseGeom& g);
// out = A^H A x + lam * x; lam is a device complex scalar (may be null = 0).
// Uses the fused single-pass y-only kernel when the pattern is x-invariant.
// coils2 (nullable) = the maps of the adjoint coil combine when they differ
void sense_normal(cfloat* out, const cfloat* x, const cfloat* coils, const cfloat* pattern, const cfloat* lam,
                  const SenseGeom& g, const cfloat* coils2 = nullptr);
// A^H A + lambda with lambda by value (the C ABI's call); check_pattern: also raise
// ERRF_PATTERN for a non-binary pattern (recon.hpp:67-77), folded into the plan pass
void sense_normal_value(cfloat* out, const cfloat* x, const cfloat* coils, const cfloat* pattern, float lambda,
                        const SenseGeom& g, bool check_pattern);
// CG on S = A^H A + lam (recon.hpp:143-181), device-resident state and scalars.
struct CgResult {
    long iterations;
    double rel_residual;
    bool converged;
};
// status_out (device, nullable): [iterations, rel_residual, converged] as doubles
void cg_normal_device(cfloat* x, const cfloat* b, const cfloat* coils, const cfloat* pattern, const cfloat* lam,
                      const SenseGeom& g, long max_iter, double tol, double* status_out);
CgResult read_cg_status(const double* status_dev);
// CG for an arbitrary Hermitian positive-definite map given as a callback
// (InverseNode over a user graph, recon.hpp:295-304); same device state machine.
using CgApply = std::function<void(const cfloat* p, cfloat* ap)>;
void cg_generic_device(cfloat* x, const cfloat* b, long n, const CgApply& apply, long max_iter, double tol,
                       double* status_out);

// ---- conv (conv.cu) -----------------------------------------------------------
struct ConvGeom {
    long X, Y, B;      // spatial extent (same padding) and batch
    long Cin, Cout;    // complex channels
    long KX, KY;       // kernel extents
    long px, py;       // corner offsets ((k-1)/2)
    // storage of the Cin-channel tensor (x / dx) and the Cout-channel tensor
    // (y / dy): false = CANON, true = CHLAST; *_tf32: operand already RN-rounded
    bool in_chlast = false, out_chlast = false;
    bool in_tf32 = false, out_tf32 = false;
    // forward only: per-channel partial sums of y from the conv epilogue when
    // the kernel form provides them (*stats_blocks = blocks written, else 0)
    double* stats = nullptr;
    int* stats_blocks = nullptr;
    // operands whose imaginary parts are known zero on the host: 1 = x (Cin side),
    // 2 = w, 4 = dy (Cout side); skips the device-side scan for the real-operand kernels
    int real_known = 0;
    // bwd-data only: batch-norm backward partial sums of the produced
    // cotangent for the BN block that consumes it (*bnb_blocks = blocks, else 0)
    const struct BnBwdHint* bnb = nullptr;
    double* bnb_part = nullptr;
    int* bnb_blocks = nullptr;
};
// y[p,f] = sum_{t,c} x[p+t-c0, c] w[t,c,f]
void conv_fwd(cfloat* y, const cfloat* x, const cfloat* w, const ConvGeom& g);
// dx[q,c] = sum_{t,f} dy[q-t+c0, f] conj(w[t,c,f])
void conv_bwd_data(cfloat* dx, const cfloat* dy, const cfloat* w, const ConvGeom& g);
// dw[t,c,f] = sum_p dy[p,f] conj(x[p+t-c0, c])
void conv_bwd_weight(cfloat* dw, const cfloat* x, const cfloat* dy, const ConvGeom& g);
// VarNet 11 x 11 layers (Cin = 2, Cout <= 24, CANON) of real operands on the
// tensor cores (conv_vn_tc.cu): mode 0 = forward, 1 = bwd-data.  `imag` is a
// device flag (nonzero: an operand has imaginary parts -> the kernel exits and
// the caller's CUDA-core complex kernel of the same pair does the work)
bool conv_vn_tc_supported(const ConvGeom& g);
void conv_vn_tc_run(cfloat* out, const cfloat* in, const cfloat* w, const ConvGeom& g, int mode, const unsigned* imag);
// weight gradient dw[t, c, f] = sum_p dy[p, f] x[p + t - 5, c] (the imag flag covers x and dy)
void conv_vn_tc_wgrad(cfloat* dw, const cfloat* x, const cfloat* dy, const ConvGeom& g, const unsigned* imag);
void conv_vn_tc_enable(bool on);
// tcgen05 TF32 implicit-GEMM path (conv_tc.cu) for 3x3 layers with 32/64 channels
void conv_tc_enable(bool on);
void conv_tc_debug(int mode);
int conv_tc_stat_slots(); // epilogue partial-sum blocks per CTA (ConvGeom::stats / bnb_part sizing)
// batch-norm work folded into the tensor-core conv epilogues (forward
// statistics, backward reduction); option "conv_bn_fuse", default on
void conv_bn_fuse_enable(bool on);
bool conv_bn_fuse();
// persistent mask-pruned A^H A kernel (sense_rank.cuh); off = sense_fast.cuh path
void sense_rank_enable(bool on);
void sense_rank_ctas(long g);
void sense_ws_enable(bool on);
void cg_pdl_enable(bool on); // programmatic dependent launch in the CG loop
void cg_fuse_enable(int mode); // CG r-update fused into the ws A^H A launch (grid barrier)
void rank_rr_enable(bool on);
void rank_vh_set(int vh); // ws A^H A: per-strip overhead weight of the cost-balanced unit ranges (0: equal counts)
void cg_defer_x_enable(bool on);
bool rank_enabled();
// test hook: auto-layout convs store multi-channel activations channels-last
void conv_force_chlast(bool on);
bool conv_chlast_forced();
bool conv_tc_supported(long cin, long cout, long kx, long ky);
void conv_tc_run(cfloat* out, const cfloat* in, const cfloat* w, const ConvGeom& g, int mode);
bool conv_tc_wgrad_supported(long cin, long cout, long kx, long ky);
// thin layers (one side 1 channel, wide side CHLAST): conv_thin.cu
bool conv_thin_supported(const ConvGeom& g);
long conv_thin_epi_blocks(const ConvGeom& g, int mode);
// F -> 1 (3x3, F = 64) on the tensor cores; false when the shape is not covered
bool thin_reduce_tc(cfloat* out, const float* wide, const float2* U, long X, long Y, long B, int F, int KK, int ox,
                    int oy);
void conv_thin_tc_enable(bool on);
void conv_thin_tc_expand_enable(bool on);
long thin_expand_tc_blocks(); // statistics partial slots the tensor-core expand may write
// 1 -> F (3x3, F = 64) on the tensor cores (+ BN statistics partials when stats != nullptr)
bool thin_expand_tc(float* out, const cfloat* thin, const float2* U, long X, long Y, long B, int F, int KK, int ox,
                    int oy, double* stats, int* stats_blocks, const BnBwdHint* bnb = nullptr, double* bpart = nullptr,
                    int* bblocks = nullptr);
void conv_thin_tc_bnb_enable(bool on);
bool conv_thin_tc_bnb();
// upper bound on the epilogue partial blocks a conv launch writes into
// ConvGeom::stats (mode 0) / bnb_part (mode 1); 0 = that path has none
long conv_epi_blocks(const ConvGeom& g, int mode);
void conv_thin_run(cfloat* out, const cfloat* in, const cfloat* w, const ConvGeom& g, int mode);
void conv_thin_wgrad(cfloat* dw, const cfloat* x, const cfloat* dy, const ConvGeom& g);
void conv_tc_wgrad(cfloat* dw, const cfloat* x, const cfloat* dy, const ConvGeom& g);

// ---- batch norm (bn.cu) ----------------------------------------------------------
struct IsoGeom {
    long inner, nstat, outer;
};
// train forward: mean, var (biased, E|x-mu|^2), u = x - mu, istd, y = u * istd,
// moving stats out = (1-mom) in + mom batch  (ops.hpp:1104-1136)
void bn_train_forward(cfloat* y, cfloat* u, cfloat* istd, cfloat* mean_out, cfloat* var_out, const cfloat* x,
                      const cfloat* mean_in, const cfloat* var_in, const IsoGeom& g, float eps, float mom);
void bn_infer_forward(cfloat* y, cfloat* u, cfloat* istd, const cfloat* x, const cfloat* mean_in,
                      const cfloat* var_in, const IsoGeom& g, float eps);
// train adjoint wrt x (ops.hpp:1245-1263)
void bn_train_adjoint_x(cfloat* dx, const cfloat* g_in, const cfloat* u, const cfloat* istd, const IsoGeom& g);
// train tangent wrt x (ops.hpp:1172-1190)
void bn_train_deriv_x(cfloat* dy, const cfloat* dx, const cfloat* u, const cfloat* istd, const IsoGeom& g);
// per-stat broadcast multiply out = in * s[stat] (conj optional)
void launch_stat_mul(cfloat* out, const cfloat* in, const cfloat* s, const IsoGeom& g, bool conj_s);
// out = in + b[stat]
void launch_stat_add(cfloat* out, const cfloat* in, const cfloat* b, const IsoGeom& g);
// out = s[stat]*c : out[i] = u[i] * f(stat) -- helper for BN adjoint wrt stats
void launch_stat_mul_u_f(cfloat* out, const cfloat* u, const cfloat* f, const IsoGeom& g);
// out[i] = (in[i], 0)
void launch_real_to_complex(cfloat* out, const float* in, long n);

// ---- fused BN + gamma + beta + CReLU on CHLAST activations (bnblock.cu) --------------
// forward state of a BN block that a producer of its output cotangent needs to
// fold the backward reduction (S1 = sum gz, S2 = sum gz conj(yhat)) into its epilogue
struct BnBwdHint {
    const float* x = nullptr; // BN input, CHLAST
    const float2* mu = nullptr;
    const float* istd = nullptr;
    const float2* gamma = nullptr;
    const float2* beta = nullptr;
    long npix = 0;
    int C = 0;
};
// x, out, dx, gout: CHLAST floats of npix pixels x C channels; mu/istd: per-channel
// device scratch kept by the node for the backward pass
void bnblock_forward(float* out, float2* mu, float* istd, float2* mean_out, float2* var_out, const float* x,
                     const float2* mean_in, const float2* var_in, const float2* gamma, const float2* beta, long npix,
                     int C, float eps, float mom, bool round_tf32, const double* pre_part = nullptr,
                     int pre_blocks = 0);
void bnblock_backward(float* dx, float2* dgamma, float2* dbeta, const float* gout, const float* x, const float2* mu,
                      const float* istd, const float2* gamma, const float2* beta, long npix, int C, bool round_tf32,
                      const double* pre_part = nullptr, int pre_blocks = 0);

// ---- RBF (rbf.cu, ops.hpp:1308-1427) -------------------------------------------------
struct RbfGeom {
    long inner, nf, outer; // z viewed [inner][filter][outer]
    int nw;
    float sigma;
    // evenly spaced centres: only the `win` centres around the nearest one are
    // evaluated (every skipped basis value is below 2^-52 of the nearest one,
    // i.e. under fp32 rounding of the sum); win = 0 evaluates all nw
    int win = 0;
    float mu0 = 0.f, inv_dmu = 0.f, dmu = 0.f;
    float q = 0.f; // exp(-dmu^2 / sigma^2): ratio of consecutive recurrence factors
};
void rbf_forward(cfloat* y, const cfloat* z, const cfloat* w, const float* mu, const RbfGeom& g);
// decides g.win for the centres (host); honours the rbf_window option
void rbf_set_window(RbfGeom& g, const std::vector<float>& mu);
void rbf_window_enable(bool on);
void rbf_cut_set(int tenths_sigma); // windowed RBF cut-off in tenths of sigma (55: K = 6 at sigma = spacing)
void rbf_pair_enable(bool on); // paired-fp32 windowed RBF map (forward / z-adjoint)
void rbf_adjoint_z(cfloat* dz, const cfloat* dy, const cfloat* z, const cfloat* w, const float* mu, const RbfGeom& g);
void rbf_deriv_z(cfloat* dy, const cfloat* dz, const cfloat* z, const cfloat* w, const float* mu, const RbfGeom& g);
void rbf_adjoint_w(cfloat* dw, const cfloat* dy, const cfloat* z, const float* mu, const RbfGeom& g);
// both adjoints in one pass (dz and dw of the same cotangent)
void rbf_adjoint_zw(cfloat* dz, cfloat* dw, const cfloat* dy, const cfloat* z, const cfloat* w, const float* mu,
                    const RbfGeom& g);
void rbf_deriv_w(cfloat* dy, const cfloat* dw, const cfloat* z, const float* mu, const RbfGeom& g);

// ---- loss / optimiser (train.cu) ------------------------------------------------------
// mse: out scalar = (1/n) sum |p - r|^2 (double accumulate), diff = p - r
void mse_forward(cfloat* loss, cfloat* diff, const cfloat* p, const cfloat* r, long n);
// complex Adam (optim.hpp:81-108) on a flat complex range
void adam_update(cfloat* theta, cfloat* m, float* v, const cfloat* g, long n, float lr, float b1, float b2,
                 float eps, float c1, float c2, float gscale, bool real_weights, bool nonneg_prox);
// flat gradient gather/scatter
void launch_copy(cfloat* dst, const cfloat* src, long n);
void launch_check_finite(const cfloat* a, long n); // sets ERRF_NONFINITE_GRAD
void launch_check_binary(const cfloat* a, long n); // sets ERRF_PATTERN unless every value is 0 or 1
// sgd_step with the clip scale, realify and NonNegProx folded in
void sgd_update(cfloat* theta, const cfloat* g, long n, float lr, float gscale, bool real_weights, bool nonneg_prox);
// NonNegProx (nn.hpp:57-64): v = (max(Re v, 0), 0)
void launch_prox_nonneg(cfloat* w, long n);

} // namespace mdnn
