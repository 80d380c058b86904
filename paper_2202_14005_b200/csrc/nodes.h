// Node factories: the reference's atoms (ops.hpp, linop.hpp) plus the fused
// B200 nodes that replace whole reference fragments on the hot path.
#pragma once

#include "nlop.h"

namespace mdnn {

// ---- atoms (reference names) ----------------------------------------------
NodePtr node_dft(const Dims& dims, unsigned long flags, bool inverse);             // linop_dft (fft.hpp:180)
NodePtr node_pad(const Dims& in, const Dims& out, const Dims& corner, bool crop);   // linop_pad / its adjoint
NodePtr node_tenmul(const std::string& name, const Dims& iter, const Dims& od, const Dims& so, const Dims& i1,
                    const Dims& s1, const Dims& i2, const Dims& s2);               // TenMulNode (ops.hpp:69)
NodePtr node_add(const Dims& dims, bool subtract);                                 // AddNode
NodePtr node_bcast_add(const Dims& x, const Dims& b);                              // BroadcastAddNode
NodePtr node_fork(const Dims& dims, int n);                                        // ForkNode
NodePtr node_zconj(const Dims& dims);
NodePtr node_zreal(const Dims& dims);
NodePtr node_real_chan(const Dims& in_dims, int chan_dim);
NodePtr node_chan_cplx(const Dims& in_dims, int chan_dim);
NodePtr node_crelu(const Dims& dims);
NodePtr node_exp_real(const Dims& dims);
NodePtr node_mse(const Dims& dims);
NodePtr node_batchnorm(const Dims& dims, unsigned long flags, bool train, double eps, double mom);
NodePtr node_rbf(const Dims& z, int filter_dim, const std::vector<float>& centers, float sigma);
// fused train-mode BatchNorm(x, y, batch) -> gamma -> beta -> CReLU block of the
// MoDL denoiser (recon.hpp:748-776): inputs (x, mean, var, g, beta),
// outputs (mean', var', out) — the reference chain's argument / output order.
// round_out / round_dx: RN-round the output / input cotangent to TF32 for a
// tensor-core convolution consumer.
NodePtr node_bnblock(const Dims& dims, bool round_out, bool round_dx, double eps = 1e-5, double mom = 0.1);
bool bnblock_supported(long channels);

// ---- fused SENSE nodes ----------------------------------------------------
struct SenseDims {
    long x = 0, y = 0, coils = 1, maps = 1, batch = 1;
    Dims image() const { return make(1, maps); }
    Dims coil_img() const { return make(coils, 1); }
    Dims coil_maps() const { return make(coils, maps); }
    Dims pattern() const
    {
        Dims d(max_rank, 1);
        d[dim_y] = y;
        return d;
    }
    Dims make(long nc, long nm) const
    {
        Dims d(max_rank, 1);
        d[dim_x] = x;
        d[dim_y] = y;
        d[dim_coil] = nc;
        d[dim_maps] = nm;
        d[dim_batch] = batch;
        return d;
    }
};
// A^H A as sense_normal_fragment (recon.hpp:412-418): inputs (x, coils, pattern, coils)
NodePtr node_sense_normal(const SenseDims& sd);
// A^H A + lambda as modl_normal_plus_lambda (recon.hpp:807-820): (x, coils, pattern, lambda)
NodePtr node_sense_normal_lambda(const SenseDims& sd);
// A^H y as sense_adjoint_fragment (recon.hpp:402-408): (y, pattern, coils)
NodePtr node_sense_adjoint(const SenseDims& sd);
// A x as sense_forward_fragment (recon.hpp:394-400): (x, coils, pattern)
NodePtr node_sense_forward(const SenseDims& sd);

// CheckpointNode (nlop.hpp:439-513): forward keeps only the inputs (shared
// immutable device arrays, no clones) and evaluates the inner graph without
// derivative state; every derivative batch re-runs the inner forward first.
NodePtr node_checkpoint(const Nlop& inner);
// re-executions of the first checkpoint node in h (-1: none)
long checkpoint_reexecutions(const Nlop& h);

// InverseNode (recon.hpp:211-329)
NodePtr node_inverse(const Nlop& s, long max_iter, double tol);
bool inverse_status(const Nlop& h, long* iterations, double* rel_residual, int* converged);

// ---- conv (conv_layer core, nn.hpp:344-426) ----------------------------------
struct ConvSpec {
    Dims in_dims;
    std::vector<int> axes;
    Dims kernel;
    int chan_dim = -1;
    long out_channels = 1;
    bool pad_same = false;
    bool transposed = false;
    // storage hint for multi-channel activations (not part of the reference
    // spec): 0 = auto (channels-last iff the tensor-core path applies),
    // 1 = channels-last (MoDL denoiser chain), -1 = reference layout
    int chlast_hint = 0;
    Dims weight_dims() const;
    Dims out_dims() const;
};
// the whole conv core (pad + TenMul, or zconj + scatter + crop for transposed)
// as one Nlop: inputs (x, w) forward, (w, x) transposed
Nlop conv_core(const std::string& name, const ConvSpec& spec);

} // namespace mdnn
