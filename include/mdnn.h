/*
 * mdnn.h — C ABI of the B200-native MoDL / VarNet hot path.
 *
 * This is the drop-in boundary for the reference's nlop operator API
 * (/root/reference/proj/include/mdnn/nlop.hpp:18-83 NlopNode, :89-437 Nlop,
 * nn.hpp:68-222 Model algebra, recon.hpp:82-904 SENSE/CG/MoDL/VarNet
 * constructors, optim.hpp:81-108,314-399 Adam + run_step).  The same header is
 * implemented twice:
 *
 *   libmdnn_b200.so   — the product: C++ host graph over device arrays and
 *                       hand-written sm_100a kernels (paper_2202_14005_b200/csrc)
 *   libmdnn_ref.so    — test oracle only: a thin shim over the unmodified
 *                       reference headers (oracle/ref_shim.cpp, built into
 *                       oracle/_ref/), used by tests/ and bench.py --impl reference.
 *
 * Conventions (reference: common.hpp:58-68, mdarray.hpp:23-200):
 *   - every array is complex64 interleaved (re, im), column-major, rank 1..16,
 *     strides counted in complex elements;
 *   - `device` = -1 for host memory, >= 0 for a CUDA device pointer (GPU build);
 *   - all calls are synchronous with respect to host buffers; device buffers
 *     are ordered on the library's stream for that device.
 *
 * Errors: every int-returning call returns 0 on success or one of MDNN_ERR_*
 * (the reference's exception taxonomy, common.hpp:15-26, with the CLI's exit
 * codes, cli.hpp:357-371); the message is in mdnn_last_error() (thread-local).
 * Handle-returning calls return NULL on error.
 */
#ifndef MDNN_H
#define MDNN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDNN_MAX_RANK 16

enum mdnn_status {
    MDNN_OK = 0,
    MDNN_ERR_OTHER = 1,
    MDNN_ERR_SHAPE = 2,  /* ShapeError */
    MDNN_ERR_IO = 3,     /* IoError */
    MDNN_ERR_CONFIG = 4, /* ConfigError */
    MDNN_ERR_SOLVER = 5, /* SolverError */
    MDNN_ERR_BOUNDS = 6, /* BoundsError */
    MDNN_ERR_ALIAS = 7,  /* AliasError */
    MDNN_ERR_STALE = 8,  /* StaleDerivativeError */
    MDNN_ERR_CUDA = 9    /* device failure (GPU build only) */
};

typedef struct mdnn_array {
    float* data;                   /* interleaved complex64 */
    int rank;                      /* 1..16 */
    int device;                    /* -1 host, >=0 CUDA ordinal */
    long dims[MDNN_MAX_RANK];
    long strides[MDNN_MAX_RANK];   /* complex elements; ignored if has_strides == 0 */
    int has_strides;               /* 0: default column-major strides */
} mdnn_array;

typedef struct mdnn_nlop mdnn_nlop;   /* refcounted graph handle (shares nodes) */
typedef struct mdnn_model mdnn_model; /* Model<R>: nlop + named args + outputs */
typedef struct mdnn_trainer mdnn_trainer;

/* ---- library ------------------------------------------------------------ */
const char* mdnn_last_error(void);
const char* mdnn_backend(void);            /* "b200-sm100a" or "reference-cpu" */
int mdnn_set_device(int device);           /* GPU build: selects device + stream */
int mdnn_synchronize(void);
/* "conv_tc" (1 = tcgen05 TF32 convolutions where supported, 0 = fp32 CUDA
   cores), "conv_chlast" (1 = auto-layout convolutions keep multi-channel
   activations channels-last; test hook for the thin-conv kernels),
   "conv_tc_form" (1 = channel-major transposed tcgen05 kernel for 64-channel
   outputs, 0 = pixel-major), "conv_tc_pair" (1 = CTA-pair cta_group::2
   pixel-major kernel), "conv_tc_debug" (diagnostics: 1 = no epilogue stores,
   2 = no epilogue; results invalid), "conv_bn_fuse" (1 = batch-norm
   statistics / backward reductions folded into the tensor-core conv
   epilogues), "conv_thin_tc" (1 = F -> 1 convolutions as tcgen05 tap
   projections + gather), "conv_wgrad_mc", "conv_tc_pair", "cg_defer_x",
   "sense_rank_split", "sense_rank" / "sense_rank_ctas" /
   "sense_rank_tm" (A^H A kernel selection) */
int mdnn_set_option(const char* key, long value);
/* the library's CUDA stream on the current device (cudaStream_t), so callers
   can order collectives / events with its kernels; NULL in the CPU shim */
void* mdnn_stream(void);
/* live per-kernel timing (CUDA events on the library stream) for tagged
   launch sites, e.g. "sense_normal_y", "conv_fwd"; used by bench.py */
int mdnn_profile_enable(int on);
/* total_work: summed algorithmic bytes (SENSE/CG tags) or flops (conv tags) */
int mdnn_profile_read(const char* tag, long* launches, double* total_ms, double* total_work);
int mdnn_profile_reset(void);
/* number of device kernels this library has launched (all devices) */
long mdnn_launch_count(void);

/* ---- Nlop (nlop.hpp:89-437) --------------------------------------------- */
void mdnn_nlop_free(mdnn_nlop* h);
mdnn_nlop* mdnn_nlop_ref(mdnn_nlop* h);    /* new handle sharing the same graph */
int mdnn_nlop_n_in(const mdnn_nlop* h);
int mdnn_nlop_n_out(const mdnn_nlop* h);
int mdnn_nlop_in_dims(const mdnn_nlop* h, int i, int* rank, long* dims);
int mdnn_nlop_out_dims(const mdnn_nlop* h, int o, int* rank, long* dims);

/* apply (nlop.hpp:125): outputs are written into caller buffers */
int mdnn_nlop_apply(mdnn_nlop* h, int n_in, const mdnn_array* in, int n_out, mdnn_array* out);
/* dy = D_i F_o dx at the last forward (nlop.hpp:158) */
int mdnn_nlop_derivative(mdnn_nlop* h, int o, int i, const mdnn_array* dx, mdnn_array* dy);
/* dx = (D_i F_o)^H dy (nlop.hpp:247) */
int mdnn_nlop_adjoint(mdnn_nlop* h, int o, int i, const mdnn_array* dy, mdnn_array* dx);
/* one reverse sweep (nlop.hpp:206); wanted[i]==0 skips input i (its dx is
   left untouched); wanted == NULL means all inputs */
int mdnn_nlop_adjoint_all(mdnn_nlop* h, int o, const mdnn_array* dy, int n_in, mdnn_array* dx,
                          const uint8_t* wanted);

/* composition algebra (nlop.hpp:265-350) — new handles, inputs unchanged */
mdnn_nlop* mdnn_nlop_combine(const mdnn_nlop* f, const mdnn_nlop* g);
mdnn_nlop* mdnn_nlop_link(const mdnn_nlop* h, int o, int i);
mdnn_nlop* mdnn_nlop_duplicate(const mdnn_nlop* h, int i, int j);
mdnn_nlop* mdnn_nlop_chain(const mdnn_nlop* f, const mdnn_nlop* g);

/* ---- atoms on the hot path (ops.hpp:1433-1485 factories + nodes) -------- */
mdnn_nlop* mdnn_nlop_dft(int rank, const long* dims, unsigned long flags, int inverse); /* linop_dft, linop.hpp:132 */
mdnn_nlop* mdnn_nlop_tenmul(int rank, const long* iter, const long* out_dims, const long* so,
                            const long* in1_dims, const long* s1, const long* in2_dims, const long* s2); /* ops.hpp:69 */
mdnn_nlop* mdnn_nlop_add(int rank, const long* dims, int subtract);            /* ops.hpp:122 */
mdnn_nlop* mdnn_nlop_bcast_add(int rank, const long* x_dims, const long* b_dims); /* ops.hpp:153 */
mdnn_nlop* mdnn_nlop_fork(int rank, const long* dims, int n);                  /* ops.hpp:214 */
mdnn_nlop* mdnn_nlop_zconj(int rank, const long* dims);                        /* ops.hpp:246 */
mdnn_nlop* mdnn_nlop_zreal(int rank, const long* dims);                        /* ops.hpp:266 */
mdnn_nlop* mdnn_nlop_real_chan(int rank, const long* dims, int chan_dim);      /* ops.hpp:318 */
mdnn_nlop* mdnn_nlop_chan_cplx(int rank, const long* dims, int chan_dim);      /* ops.hpp:376 */
mdnn_nlop* mdnn_nlop_crelu(int rank, const long* dims);                        /* ops.hpp:451 */
mdnn_nlop* mdnn_nlop_exp_real(int rank, const long* dims);                     /* ops.hpp:672 */
mdnn_nlop* mdnn_nlop_mse(int rank, const long* dims);                          /* ops.hpp:874 */
mdnn_nlop* mdnn_nlop_batchnorm(int rank, const long* dims, unsigned long flags, int train,
                               double eps, double momentum);                   /* ops.hpp:1070 */
mdnn_nlop* mdnn_nlop_rbf(int rank, const long* z_dims, int filter_dim, int n_centers,
                         const float* centers, float sigma);                   /* ops.hpp:1308 */
mdnn_nlop* mdnn_nlop_pad(int rank, const long* in_dims, const long* out_dims, const long* corner); /* linop.hpp:142 */

/* SENSE (recon.hpp:18-42 SenseDims) */
typedef struct mdnn_sense_dims {
    long x, y, coils, maps, batch;
} mdnn_sense_dims;
/* inverse of S with x = input 0 (recon.hpp:211-329, make_inverse_nlop :326) */
mdnn_nlop* mdnn_nlop_inverse(const mdnn_nlop* s, long max_iter, double tol);
/* checkpoint(f) (nlop.hpp:439-522): forward keeps only the inputs, every
 * derivative batch re-runs the inner forward; reexecutions() of its node */
mdnn_nlop* mdnn_nlop_checkpoint(const mdnn_nlop* f);
long mdnn_nlop_checkpoint_reexecutions(const mdnn_nlop* h); /* -1: no checkpoint node */
/* last CG status of an inverse node graph (recon.hpp:136-140): first InverseNode found */
int mdnn_nlop_cg_status(const mdnn_nlop* h, long* iterations, double* rel_residual, int* converged);

/* plain CG-SENSE linop applications on one array set (recon.hpp:82-195) */
int mdnn_sense_forward(const mdnn_array* coils, const mdnn_array* pattern, const mdnn_array* x, mdnn_array* y);
int mdnn_sense_adjoint(const mdnn_array* coils, const mdnn_array* pattern, const mdnn_array* y, mdnn_array* x);
int mdnn_sense_normal(const mdnn_array* coils, const mdnn_array* pattern, float lambda, const mdnn_array* x, mdnn_array* y);
int mdnn_cg_normal_solve(const mdnn_array* coils, const mdnn_array* pattern, float lambda, const mdnn_array* b,
                         long max_iter, double tol, mdnn_array* x, long* iterations, double* rel_residual);
/* dft on one array (fft.hpp:180) */
int mdnn_dft(const mdnn_array* in, unsigned long flags, int inverse, mdnn_array* out);

/* ---- Model (nn.hpp:68-222) ------------------------------------------------ */
enum mdnn_arg_kind { MDNN_ARG_DATA = 0, MDNN_ARG_WEIGHTS = 1, MDNN_ARG_MOVING_STATS = 2 };

void mdnn_model_free(mdnn_model* m);
mdnn_nlop* mdnn_model_nlop(const mdnn_model* m); /* new handle; caller frees */
int mdnn_model_n_args(const mdnn_model* m);
const char* mdnn_model_arg_name(const mdnn_model* m, int i);
int mdnn_model_arg_kind(const mdnn_model* m, int i);
int mdnn_model_arg_real(const mdnn_model* m, int i);
int mdnn_model_n_outs(const mdnn_model* m);
const char* mdnn_model_out_name(const mdnn_model* m, int o);
int mdnn_model_arg_index(const mdnn_model* m, const char* name);
int mdnn_model_output_index(const mdnn_model* m, const char* name);
long mdnn_model_num_real_params(const mdnn_model* m);
/* seeded init of one weights/moving-stats argument (nn.hpp:117-145), host or device out */
int mdnn_model_init_weight(const mdnn_model* m, uint64_t seed, const char* name, mdnn_array* out);

/* model algebra */
mdnn_model* mdnn_model_chain(const mdnn_model* a, const mdnn_model* b, const char* b_in, int a_out);
mdnn_model* mdnn_model_link(const mdnn_model* m, int out_idx, const char* arg);
mdnn_model* mdnn_model_combine(const mdnn_model* a, const mdnn_model* b);
mdnn_model* mdnn_model_dedupe(const mdnn_model* m);

/* layers (nn.hpp:344-453) */
typedef struct mdnn_conv_spec {
    int rank;
    long in_dims[MDNN_MAX_RANK];
    int n_axes;
    int axes[4];
    long kernel[4];
    int chan_dim;
    long out_channels;
    int pad_same;
    int transposed;
} mdnn_conv_spec;
mdnn_model* mdnn_conv_layer(const char* name, const mdnn_conv_spec* spec, int bias);
mdnn_model* mdnn_batchnorm_layer(const char* name, int rank, const long* dims, unsigned long flags,
                                 int train, double eps, double momentum);

/* networks (recon.hpp:499-904).  The constructors build the reference's
   graphs with the two wiring fixes documented in DESIGN.md §Oracle. */
typedef struct mdnn_modl_cfg {
    long iterations, layers, filters, kernel, cg_iter;
    double cg_tol, lambda_init;
    long im_x, im_y, coils, maps, batch;
    int train_mode;
} mdnn_modl_cfg;
typedef struct mdnn_varnet_cfg {
    long iterations, filters, kernel, rbf;
    long im_x, im_y, coils, maps, batch;
} mdnn_varnet_cfg;
void mdnn_modl_cfg_default(mdnn_modl_cfg* c);
void mdnn_varnet_cfg_default(mdnn_varnet_cfg* c);
mdnn_model* mdnn_build_modl(const mdnn_modl_cfg* cfg);
mdnn_model* mdnn_build_varnet(const mdnn_varnet_cfg* cfg);
/* Model::rebatch (nn.hpp:82, used by train's minibatching optim.hpp:237-276):
   the same network rebuilt for `batch` items (NULL + error 4 when the model has
   no rebatch, e.g. hand-assembled fragments) */
mdnn_model* mdnn_model_rebatch(const mdnn_model* m, long batch);
/* per-block fragments of the networks (parity units of the C2 / C3 configs):
   the MoDL CNN denoiser D_W(x) = x + CNN(x) of one unroll (modl_denoiser_fragment,
   recon.hpp:714-803, with the output-by-name fix) and the VarNet regulariser
   sum_f K^T Phi'(Re K x) of stage "it0" (varnet_reg_fragment, recon.hpp:522-609) */
mdnn_model* mdnn_modl_denoiser(const mdnn_modl_cfg* cfg);
/* the train-mode BN -> gamma -> beta -> CReLU chain of one denoiser layer
   (recon.hpp:748-776) as a model: args x, <name>_bn_mean, <name>_bn_var,
   <name>_g, <name>_beta; outputs <name>_bn_mean, <name>_bn_var, out.  The
   product runs it as one fused channels-last node (bnblock.cu) */
mdnn_model* mdnn_bn_block(const char* name, int rank, const long* dims);
mdnn_model* mdnn_varnet_reg(const mdnn_varnet_cfg* cfg);
/* SENSE fragments as models (recon.hpp:394-418, :807-820) */
mdnn_model* mdnn_sense_normal_fragment(const mdnn_sense_dims* sd);
mdnn_model* mdnn_sense_adjoint_fragment(const mdnn_sense_dims* sd);
mdnn_model* mdnn_modl_normal_plus_lambda(const mdnn_sense_dims* sd);
mdnn_model* mdnn_loss_model_mse(int rank, const long* dims);

/* ---- simulation fixtures (simulate.hpp:40-133) --------------------------- */
/* draw_phantom/draw_coils for item s with seed (hash_rand(seed,2s) / 2s+1) into
   host arrays of dims [X,Y,1,1,...] and [X,Y,1,C,...] */
int mdnn_sim_item(uint64_t seed, long item, long x, long y, long coils, float* phantom, float* coil_maps);
int mdnn_sim_pattern(long y, long accel, long acl, float* pattern);

/* ---- training (optim.hpp:20-108, :218-415) ------------------------------- */
typedef struct mdnn_train_cfg {
    double lr, beta1, beta2, eps, clip;
    int algo;                        /* OptAlgo (optim.hpp:10): 0 sgd, 1 adam (default), 2 ipalm */
    double ipalm_alpha, ipalm_beta;  /* IpalmParams (optim.hpp:26-29) */
} mdnn_train_cfg;
void mdnn_train_cfg_default(mdnn_train_cfg* c);
/* joins model output "out" with an MSE loss against data arg "reference" */
mdnn_trainer* mdnn_trainer_create(const mdnn_model* model, const mdnn_train_cfg* cfg, uint64_t seed);
void mdnn_trainer_free(mdnn_trainer* t);
int mdnn_trainer_set_data(mdnn_trainer* t, const char* name, const mdnn_array* a);
/* input prefetch (the reconet loader's next-batch staging): queue a dense
   host batch for data arg `name`; the copy runs asynchronously on a copy
   stream and the next forward pass takes the oldest queued batch of each
   name.  The host buffer (pinned for true overlap) must stay valid until that
   forward pass has been issued.  The CPU shim copies synchronously. */
int mdnn_trainer_stage_data(mdnn_trainer* t, const char* name, const mdnn_array* a);
int mdnn_trainer_set_weight(mdnn_trainer* t, const char* name, const mdnn_array* a);
int mdnn_trainer_get_weight(mdnn_trainer* t, const char* name, mdnn_array* out);
int mdnn_trainer_get_grad(mdnn_trainer* t, const char* name, mdnn_array* out);
/* forward + backward: loss (host double, synchronising) and gradients into the
   flat gradient buffer; no weight update */
int mdnn_trainer_forward_backward(mdnn_trainer* t, double* loss);
/* flat fp32 gradient buffer (device pointer in the GPU build) for all-reduce */
int mdnn_trainer_grad_buffer(mdnn_trainer* t, float** ptr, long* n_floats);
/* scale gradients (e.g. 1/world), realify/clip, Adam, prox, moving stats */
int mdnn_trainer_update(mdnn_trainer* t, float grad_scale);
/* run_step = forward_backward + update(1); with a communicator attached
   (mdnn_trainer_set_comm): forward_backward with the bucketed all-reduce,
   then update_dp(world) */
int mdnn_trainer_step(mdnn_trainer* t, double* loss);

/* ---- data parallelism (BART batch stacking) ----
 * Per-shard semantics: each replica runs the reference's run_step on its own
 * batch shard (optim.hpp:314-399); gradients are summed over replicas and
 * every replica applies the same update with 1/world, and the BN moving
 * statistics (update_stats, optim.hpp:403-415) become the replica mean, so
 * replicas stay bitwise identical.  The sync buffer is the whole payload:
 * [weight gradients (grad_buffer's floats) | moving statistics], fp32. */
int mdnn_trainer_sync_buffer(mdnn_trainer* t, float** ptr, long* n_floats);
/* after the sync buffer was summed over `world` replicas (caller's collective) */
int mdnn_trainer_update_dp(mdnn_trainer* t, int world);
/* in-library NCCL: rank 0 creates the 128-byte id, the caller distributes it,
   every rank attaches; mdnn_trainer_step then all-reduces gradient buckets on
   a comm stream as the reverse sweep finalises them (CPU reference: error 4) */
int mdnn_nccl_unique_id(uint8_t* id128);
int mdnn_trainer_set_comm(mdnn_trainer* t, const uint8_t* id128, int nranks, int rank);
int mdnn_trainer_n_weights(const mdnn_trainer* t);
const char* mdnn_trainer_weight_name(const mdnn_trainer* t, int k);

/* ---- cfl files and weight bundles (cfl.hpp:15-142) -----------------------
 * Byte-compatible with the reference: <base>.hdr ("# Dimensions" + 16 dims)
 * and <base>.cfl (interleaved complex64, column-major).  Bundles: a directory
 * of cfl pairs + manifest.txt ("format 1", sorted meta, "array <name>"). */
int mdnn_cfl_dims(const char* base, long* dims16);                     /* cfl_read header, cfl.hpp:53-73 */
int mdnn_cfl_read(const char* base, mdnn_array* out);                  /* cfl_read, cfl.hpp:53-88 */
int mdnn_cfl_write(const char* base, const mdnn_array* a);             /* cfl_write, cfl.hpp:19-51 */
/* WeightsBundle::save of every trainer weight plus n_meta key/value pairs (cfl.hpp:97-111) */
int mdnn_weights_save(mdnn_trainer* t, const char* dir, int n_meta, const char* const* keys,
                      const char* const* vals);
/* WeightsBundle::load (cfl.hpp:113-135) into the trainer's weights by name */
int mdnn_weights_load(mdnn_trainer* t, const char* dir);
/* WeightsBundle::meta_or: copies the value (or fallback) into buf, NUL-terminated (cfl.hpp:137-141) */
int mdnn_weights_meta(const char* dir, const char* key, const char* fallback, char* buf, long buflen);

/* ---- reconet driver (cli.hpp:52-265) ------------------------------------
 * The train / apply command either side of the training step, on cfl files.
 * Fields mirror ReconetOptions (cli.hpp:52-65); -1 / NULL mean "default" or
 * "take it from the weights bundle".  Strings are not copied past the call. */
typedef struct mdnn_reconet_opts {
    const char* network;       /* "varnet" | "modl" */
    int do_train, do_apply;    /* exactly one */
    int normalize;             /* per-item 1 / max |A^H y| (recon.hpp:464-493) */
    const char* pattern_file;  /* NULL / "": estimate_pattern from k-space (cli.hpp:28-50) */
    const char* init_weights;  /* warm-start bundle for --train */
    long iterations, filters, kernel, rbf, layers, cg_iter;
    long epochs, batch_size;
    double lr;                 /* <= 0: 1e-2 varnet, 1e-3 modl */
    const char* optimizer;     /* NULL / "": ipalm for varnet, adam for modl */
    uint64_t seed;
    int verbose;               /* print "epoch k loss v" per epoch */
    const char* kspace_file;
    const char* coils_file;
    const char* weights_dir;   /* bundle written by --train, read by --apply */
    const char* target_file;   /* --train: reference images; --apply: output */
} mdnn_reconet_opts;
void mdnn_reconet_opts_default(mdnn_reconet_opts* o);
int mdnn_reconet(const mdnn_reconet_opts* o);                                    /* cmd_reconet, cli.hpp:94-265 */
int mdnn_estimate_pattern(const mdnn_array* kspace, mdnn_array* pattern);       /* cli.hpp:28-50 */

#ifdef __cplusplus
}
#endif
#endif /* MDNN_H */
