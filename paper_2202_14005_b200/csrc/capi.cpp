// extern "C" boundary (include/mdnn.h) of the B200 library.  Every entry
// point maps C++ exceptions to the reference's error codes (common.hpp:15-26,
// cli.hpp:357-371) and keeps the message in a thread-local string.
#include "../../include/mdnn.h"

#include "cfl.h"
#include "reconet.h"
#include "kernels.h"
#include "profile.h"
#include "train.h"

#include <cstring>
#include <fstream>

using namespace mdnn;

struct mdnn_nlop {
    Nlop op;
};
struct mdnn_model {
    Model m;
};
struct mdnn_trainer {
    std::unique_ptr<Trainer> t;
};

namespace {

thread_local std::string g_err;

template<class F>
int guard(F&& f)
{
    try {
        f();
        return MDNN_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code();
    } catch (const std::exception& e) {
        g_err = e.what();
        return MDNN_ERR_OTHER;
    }
}

template<class T, class F>
T* guard_ptr(F&& f)
{
    T* out = nullptr;
    if (guard([&] { out = f(); }) != MDNN_OK)
        return nullptr;
    return out;
}

Dims mk(int rank, const long* d)
{
    if (rank < 1 || rank > max_rank)
        throw ShapeError("rank must be in 1..16");
    return Dims(d, d + rank);
}

HostView hv(const mdnn_array& a)
{
    HostView v;
    v.data = a.data;
    v.device = a.device;
    v.dims = Dims(a.dims, a.dims + a.rank);
    if (a.has_strides)
        v.strides = Dims(a.strides, a.strides + a.rank);
    if (a.device >= 0 && a.device != ctx().device)
        throw ConfigError("array on device " + std::to_string(a.device) + " but library is on device "
                          + std::to_string(ctx().device));
    return v;
}

DArray in_arr(const mdnn_array& a) { return import_array(hv(a)); }
// inputs of calls that do not keep them: dense device arrays are used in place
DArray in_view(const mdnn_array& a) { return borrow_array(hv(a)); }
// output buffer: the caller's dense device array in place, else a fresh array
// copied out by out_arr
DArray out_target(mdnn_array& a, const Dims& d)
{
    const HostView v = hv(a);
    if (v.device == ctx().device && v.dims == d && (v.strides.empty() || v.strides == default_strides(d)))
        return borrow_array(v);
    return DArray(d, false);
}
void out_arr_if_needed(const DArray& d, mdnn_array& a)
{
    if (d.buf->owned)
        export_array(d, hv(a));
}
void out_arr(const DArray& d, mdnn_array& a) { export_array(d, hv(a)); }

mdnn_nlop* wrap(Nlop op) { return new mdnn_nlop{std::move(op)}; }
mdnn_model* wrapm(Model m) { return new mdnn_model{std::move(m)}; }

SenseDims to_sd(const mdnn_sense_dims* s) { return SenseDims{s->x, s->y, s->coils, s->maps, s->batch}; }

// geometry of a standalone SENSE call from the coil and pattern arrays
SenseGeom geom_from(const DArray& coils, const DArray& pattern)
{
    if (coils.rank() != max_rank || pattern.rank() != max_rank)
        throw ShapeError("sense: coils/pattern must have rank 16");
    SenseGeom g{};
    g.X = coils.dims[dim_x];
    g.Y = coils.dims[dim_y];
    g.C = coils.dims[dim_coil];
    g.M = coils.dims[dim_maps];
    g.B = coils.dims[dim_batch];
    const Dims& p = pattern.dims;
    for (int d = 0; d < max_rank; d++)
        if (d != dim_x && d != dim_y && d != dim_coil && d != dim_batch && p[d] != 1)
            throw ShapeError("sense: pattern dims must be [X|1, Y|1, 1, C|1, 1, ..., B|1]");
    auto chk = [](long pv, long full) {
        if (pv != 1 && pv != full)
            throw ShapeError("sense: pattern not broadcastable to k-space");
        return pv;
    };
    g.pat_x = chk(p[dim_x], g.X);
    g.pat_y = chk(p[dim_y], g.Y);
    g.pat_c = chk(p[dim_coil], g.C);
    g.pat_b = chk(p[dim_batch], g.B);
    return g;
}

void check_binary(const DArray& pattern)
{
    // recon.hpp:67-77, evaluated on the device (no host round trip per call): a
    // non-binary pattern sets ERRF_PATTERN, which the call's closing
    // sync_and_check() raises as the reference's ConfigError
    launch_check_binary(pattern.data(), pattern.size());
}

Dims img_dims(const SenseGeom& g)
{
    Dims d(max_rank, 1);
    d[0] = g.X;
    d[1] = g.Y;
    d[dim_maps] = g.M;
    d[dim_batch] = g.B;
    return d;
}

Dims kspace_dims(const SenseGeom& g)
{
    Dims d(max_rank, 1);
    d[0] = g.X;
    d[1] = g.Y;
    d[dim_coil] = g.C;
    d[dim_batch] = g.B;
    return d;
}

} // namespace

extern "C" {

const char* mdnn_last_error(void) { return g_err.c_str(); }
const char* mdnn_backend(void) { return "b200-sm100a"; }

int mdnn_set_device(int device)
{
    return guard([&] { set_device(device); });
}

int mdnn_synchronize(void)
{
    return guard([] { sync_and_check(); });
}

int mdnn_set_option(const char* key, long value)
{
    return guard([&] {
        std::string k = key ? key : "";
        if (k == "conv_tc")
            conv_tc_enable(value != 0);
        else if (k == "sense_rank")
            sense_rank_enable(value != 0);
        else if (k == "rbf_window")
            rbf_window_enable(value != 0);
        else if (k == "rbf_pair")
            rbf_pair_enable(value != 0);
        else if (k == "rbf_cut")
            rbf_cut_set(int(value));
        else if (k == "rank_rr")
            rank_rr_enable(value != 0);
        else if (k == "rank_vh")
            rank_vh_set(int(value));
        else if (k == "sense_ws")
            sense_ws_enable(value != 0);
        else if (k == "cg_pdl")
            cg_pdl_enable(value != 0);
        else if (k == "cg_fuse")
            cg_fuse_enable(int(value));
        else if (k == "pdl")
            g_pdl = value != 0;
        else if (k == "sense_rank_ctas")
            sense_rank_ctas(value);
        else if (k == "cg_defer_x")
            cg_defer_x_enable(value != 0);
        else if (k == "conv_thin_tc")
            conv_thin_tc_enable(value != 0);
        else if (k == "conv_thin_tc_expand")
            conv_thin_tc_expand_enable(value != 0);
        else if (k == "conv_thin_tc_bnb")
            conv_thin_tc_bnb_enable(value != 0);
        else if (k == "conv_chlast")
            conv_force_chlast(value != 0);
        else if (k == "conv_tc_debug")
            conv_tc_debug(int(value));
        else if (k == "conv_vn_tc")
            conv_vn_tc_enable(value != 0);
        else if (k == "conv_bn_fuse")
            conv_bn_fuse_enable(value != 0);
        else
            throw ConfigError("unknown option '" + k + "'");
    });
}

void* mdnn_stream(void)
{
    void* s = nullptr;
    guard([&] { s = static_cast<void*>(ctx().stream); });
    return s;
}

int mdnn_profile_enable(int on)
{
    return guard([&] { prof_enable(on != 0); });
}

int mdnn_profile_read(const char* tag, long* launches, double* total_ms, double* total_work)
{
    return guard([&] { prof_read(tag, launches, total_ms, total_work); });
}

long mdnn_launch_count(void) { return launch_count(); }

int mdnn_profile_reset(void)
{
    return guard([] { prof_reset(); });
}

void mdnn_nlop_free(mdnn_nlop* h) { delete h; }
mdnn_nlop* mdnn_nlop_ref(mdnn_nlop* h) { return new mdnn_nlop{h->op}; }
int mdnn_nlop_n_in(const mdnn_nlop* h) { return h->op.n_in(); }
int mdnn_nlop_n_out(const mdnn_nlop* h) { return h->op.n_out(); }

int mdnn_nlop_in_dims(const mdnn_nlop* h, int i, int* rank, long* dims)
{
    return guard([&] {
        const auto& d = h->op.in_dims(i);
        *rank = int(d.size());
        std::copy(d.begin(), d.end(), dims);
    });
}

int mdnn_nlop_out_dims(const mdnn_nlop* h, int o, int* rank, long* dims)
{
    return guard([&] {
        const auto& d = h->op.out_dims(o);
        *rank = int(d.size());
        std::copy(d.begin(), d.end(), dims);
    });
}

int mdnn_nlop_apply(mdnn_nlop* h, int n_in, const mdnn_array* in, int n_out, mdnn_array* out)
{
    return guard([&] {
        std::vector<DArray> args;
        for (int i = 0; i < n_in; i++)
            args.push_back(in_arr(in[i]));
        auto res = h->op.apply(args);
        if (n_out != int(res.size()))
            throw ShapeError("apply: expected " + std::to_string(res.size()) + " outputs");
        for (int o = 0; o < n_out; o++)
            if (out[o].data)
                out_arr(res[o], out[o]);
        sync_and_check();
    });
}

int mdnn_nlop_derivative(mdnn_nlop* h, int o, int i, const mdnn_array* dx, mdnn_array* dy)
{
    return guard([&] {
        out_arr(h->op.derivative(o, i, in_arr(*dx)), *dy);
        sync_and_check();
    });
}

int mdnn_nlop_adjoint(mdnn_nlop* h, int o, int i, const mdnn_array* dy, mdnn_array* dx)
{
    return guard([&] {
        out_arr(h->op.adjoint_derivative(o, i, in_arr(*dy)), *dx);
        sync_and_check();
    });
}

int mdnn_nlop_adjoint_all(mdnn_nlop* h, int o, const mdnn_array* dy, int n_in, mdnn_array* dx, const uint8_t* wanted)
{
    return guard([&] {
        std::vector<char> want(h->op.n_in(), 1);
        if (wanted)
            for (int i = 0; i < h->op.n_in() && i < n_in; i++)
                want[i] = wanted[i] ? 1 : 0;
        for (int i = 0; i < h->op.n_in(); i++)
            if (i >= n_in || !dx[i].data)
                want[i] = 0;
        auto res = h->op.adjoint_all(o, in_arr(*dy), want);
        for (int i = 0; i < n_in && i < int(res.size()); i++)
            if (want[i])
                out_arr(res[i], dx[i]);
        sync_and_check();
    });
}

mdnn_nlop* mdnn_nlop_combine(const mdnn_nlop* f, const mdnn_nlop* g)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(combine(f->op, g->op)); });
}
mdnn_nlop* mdnn_nlop_link(const mdnn_nlop* h, int o, int i)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(link(h->op, o, i)); });
}
mdnn_nlop* mdnn_nlop_duplicate(const mdnn_nlop* h, int i, int j)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(duplicate(h->op, i, j)); });
}
mdnn_nlop* mdnn_nlop_chain(const mdnn_nlop* f, const mdnn_nlop* g)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(chain(f->op, g->op)); });
}

mdnn_nlop* mdnn_nlop_dft(int rank, const long* dims, unsigned long flags, int inverse)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(Nlop(node_dft(mk(rank, dims), flags, inverse != 0))); });
}
mdnn_nlop* mdnn_nlop_tenmul(int rank, const long* iter, const long* od, const long* so, const long* i1,
                            const long* s1, const long* i2, const long* s2)
{
    return guard_ptr<mdnn_nlop>([&] {
        return wrap(Nlop(node_tenmul("tenmul", mk(rank, iter), mk(rank, od), mk(rank, so), mk(rank, i1),
                                     mk(rank, s1), mk(rank, i2), mk(rank, s2))));
    });
}
mdnn_nlop* mdnn_nlop_add(int rank, const long* dims, int subtract)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(Nlop(node_add(mk(rank, dims), subtract != 0))); });
}
mdnn_nlop* mdnn_nlop_bcast_add(int rank, const long* x, const long* b)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(Nlop(node_bcast_add(mk(rank, x), mk(rank, b)))); });
}
mdnn_nlop* mdnn_nlop_fork(int rank, const long* dims, int n)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(Nlop(node_fork(mk(rank, dims), n))); });
}
mdnn_nlop* mdnn_nlop_zconj(int rank, const long* dims)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(Nlop(node_zconj(mk(rank, dims)))); });
}
mdnn_nlop* mdnn_nlop_zreal(int rank, const long* dims)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(Nlop(node_zreal(mk(rank, dims)))); });
}
mdnn_nlop* mdnn_nlop_real_chan(int rank, const long* dims, int cd)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(Nlop(node_real_chan(mk(rank, dims), cd))); });
}
mdnn_nlop* mdnn_nlop_chan_cplx(int rank, const long* dims, int cd)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(Nlop(node_chan_cplx(mk(rank, dims), cd))); });
}
mdnn_nlop* mdnn_nlop_crelu(int rank, const long* dims)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(Nlop(node_crelu(mk(rank, dims)))); });
}
mdnn_nlop* mdnn_nlop_exp_real(int rank, const long* dims)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(Nlop(node_exp_real(mk(rank, dims)))); });
}
mdnn_nlop* mdnn_nlop_mse(int rank, const long* dims)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(Nlop(node_mse(mk(rank, dims)))); });
}
mdnn_nlop* mdnn_nlop_batchnorm(int rank, const long* dims, unsigned long flags, int train, double eps, double mom)
{
    return guard_ptr<mdnn_nlop>(
        [&] { return wrap(Nlop(node_batchnorm(mk(rank, dims), flags, train != 0, eps, mom))); });
}
mdnn_nlop* mdnn_nlop_rbf(int rank, const long* z, int fd, int n, const float* centers, float sigma)
{
    return guard_ptr<mdnn_nlop>([&] {
        std::vector<float> c(centers, centers + n);
        return wrap(Nlop(node_rbf(mk(rank, z), fd, c, sigma)));
    });
}
mdnn_nlop* mdnn_nlop_pad(int rank, const long* in, const long* out, const long* corner)
{
    return guard_ptr<mdnn_nlop>(
        [&] { return wrap(Nlop(node_pad(mk(rank, in), mk(rank, out), mk(rank, corner), false))); });
}
mdnn_nlop* mdnn_nlop_inverse(const mdnn_nlop* s, long max_iter, double tol)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(Nlop(node_inverse(s->op, max_iter, tol))); });
}

mdnn_nlop* mdnn_nlop_checkpoint(const mdnn_nlop* f)
{
    return guard_ptr<mdnn_nlop>([&] { return wrap(Nlop(node_checkpoint(f->op))); });
}

long mdnn_nlop_checkpoint_reexecutions(const mdnn_nlop* h)
{
    long r = -1;
    guard([&] { r = checkpoint_reexecutions(h->op); });
    return r;
}

int mdnn_nlop_cg_status(const mdnn_nlop* h, long* iterations, double* rel_residual, int* converged)
{
    return guard([&] {
        if (!inverse_status(h->op, iterations, rel_residual, converged))
            throw ConfigError("cg_status: no inverse node in graph");
    });
}

int mdnn_sense_forward(const mdnn_array* coils, const mdnn_array* pattern, const mdnn_array* x, mdnn_array* y)
{
    return guard([&] {
        DArray C = in_arr(*coils), P = in_arr(*pattern), X = in_arr(*x);
        check_binary(P);
        SenseGeom g = geom_from(C, P);
        if (X.dims != img_dims(g))
            throw ShapeError("linop forward: expected " + dims_to_string(img_dims(g)) + ", got "
                             + dims_to_string(X.dims));
        DArray out(kspace_dims(g), false);
        sense_forward(out.data(), X.data(), C.data(), P.data(), g);
        out_arr(out, *y);
        sync_and_check();
    });
}

int mdnn_sense_adjoint(const mdnn_array* coils, const mdnn_array* pattern, const mdnn_array* y, mdnn_array* x)
{
    return guard([&] {
        DArray C = in_arr(*coils), P = in_arr(*pattern), Y = in_arr(*y);
        check_binary(P);
        SenseGeom g = geom_from(C, P);
        if (Y.dims != kspace_dims(g))
            throw ShapeError("linop adjoint: expected " + dims_to_string(kspace_dims(g)) + ", got "
                             + dims_to_string(Y.dims));
        DArray out(img_dims(g), false);
        sense_adjoint(out.data(), Y.data(), C.data(), P.data(), g);
        out_arr(out, *x);
        sync_and_check();
    });
}

int mdnn_sense_normal(const mdnn_array* coils, const mdnn_array* pattern, float lambda, const mdnn_array* x,
                      mdnn_array* y)
{
    return guard([&] {
        DArray C = in_view(*coils), P = in_view(*pattern), X = in_view(*x);
        SenseGeom g = geom_from(C, P);
        if (X.dims != img_dims(g))
            throw ShapeError("linop normal: expected " + dims_to_string(img_dims(g)));
        DArray out = out_target(*y, img_dims(g));
        if (out.data() == X.data())
            out = DArray(img_dims(g), false); // in-place call: keep x intact until the kernel is done
        // the binary-pattern check (check_binary) rides in the A^H A plan pass
        sense_normal_value(out.data(), X.data(), C.data(), P.data(), lambda, g, true);
        out_arr_if_needed(out, *y);
        sync_and_check();
    });
}

int mdnn_cg_normal_solve(const mdnn_array* coils, const mdnn_array* pattern, float lambda, const mdnn_array* b,
                         long max_iter, double tol, mdnn_array* x, long* iterations, double* rel_residual)
{
    return guard([&] {
        if (lambda < 0)
            throw ConfigError("cg_normal_solve: lambda must be nonnegative");
        DArray C = in_view(*coils), P = in_view(*pattern), B = in_view(*b);
        check_binary(P);
        SenseGeom g = geom_from(C, P);
        if (B.dims != img_dims(g))
            throw ShapeError("cg: rhs dims mismatch");
        DArray lam = DArray::scalar(lambda);
        DArray out(img_dims(g), false);
        DArray st(Dims{3}, true); // 3 doubles
        cg_normal_device(out.data(), B.data(), C.data(), P.data(), lam.data(), g, max_iter, tol,
                         reinterpret_cast<double*>(st.data()));
        auto res = read_cg_status(reinterpret_cast<double*>(st.data()));
        out_arr(out, *x);
        sync_and_check();
        if (iterations)
            *iterations = res.iterations;
        if (rel_residual)
            *rel_residual = res.rel_residual;
    });
}

int mdnn_dft(const mdnn_array* in, unsigned long flags, int inverse, mdnn_array* out)
{
    return guard([&] {
        DArray a = in_arr(*in);
        DArray o(a.dims, false);
        fft_flags(o.data(), a.data(), a.dims, flags, inverse != 0);
        out_arr(o, *out);
        sync_and_check();
    });
}

// ---- Model -----------------------------------------------------------------
void mdnn_model_free(mdnn_model* m) { delete m; }
mdnn_nlop* mdnn_model_nlop(const mdnn_model* m) { return new mdnn_nlop{m->m.op}; }
int mdnn_model_n_args(const mdnn_model* m) { return int(m->m.args.size()); }
const char* mdnn_model_arg_name(const mdnn_model* m, int i) { return m->m.args.at(i).name.c_str(); }
int mdnn_model_arg_kind(const mdnn_model* m, int i) { return int(m->m.args.at(i).kind); }
int mdnn_model_arg_real(const mdnn_model* m, int i) { return m->m.args.at(i).real_weights ? 1 : 0; }
int mdnn_model_n_outs(const mdnn_model* m) { return int(m->m.out_names.size()); }
const char* mdnn_model_out_name(const mdnn_model* m, int o) { return m->m.out_names.at(o).c_str(); }
int mdnn_model_arg_index(const mdnn_model* m, const char* name)
{
    int r = -1;
    if (guard([&] { r = m->m.arg_index(name); }) != MDNN_OK)
        return -1;
    return r;
}
int mdnn_model_output_index(const mdnn_model* m, const char* name)
{
    int r = -1;
    if (guard([&] { r = m->m.output_index(name); }) != MDNN_OK)
        return -1;
    return r;
}
long mdnn_model_num_real_params(const mdnn_model* m) { return m->m.num_real_params(); }

int mdnn_model_init_weight(const mdnn_model* m, uint64_t seed, const char* name, mdnn_array* out)
{
    return guard([&] {
        int i = m->m.arg_index(name);
        if (m->m.args[i].kind == ArgKind::Data)
            throw ConfigError(std::string("init_weight: no weights argument ") + name);
        auto h = m->m.init_weight(seed, i);
        out_arr(from_host(m->m.op.in_dims(i), h.data()), *out);
        sync_and_check();
    });
}

mdnn_model* mdnn_model_chain(const mdnn_model* a, const mdnn_model* b, const char* b_in, int a_out)
{
    return guard_ptr<mdnn_model>([&] { return wrapm(model_chain(a->m, b->m, b_in, a_out)); });
}
mdnn_model* mdnn_model_link(const mdnn_model* m, int out_idx, const char* arg)
{
    return guard_ptr<mdnn_model>([&] { return wrapm(model_link(m->m, out_idx, arg)); });
}
mdnn_model* mdnn_model_combine(const mdnn_model* a, const mdnn_model* b)
{
    return guard_ptr<mdnn_model>([&] { return wrapm(model_combine(a->m, b->m)); });
}
mdnn_model* mdnn_model_dedupe(const mdnn_model* m)
{
    return guard_ptr<mdnn_model>([&] { return wrapm(model_dedupe(m->m)); });
}

mdnn_model* mdnn_conv_layer(const char* name, const mdnn_conv_spec* s, int bias)
{
    return guard_ptr<mdnn_model>([&] {
        ConvSpec spec;
        spec.in_dims = mk(s->rank, s->in_dims);
        spec.axes.assign(s->axes, s->axes + s->n_axes);
        spec.kernel.assign(s->kernel, s->kernel + s->n_axes);
        spec.chan_dim = s->chan_dim;
        spec.out_channels = s->out_channels;
        spec.pad_same = s->pad_same != 0;
        spec.transposed = s->transposed != 0;
        return wrapm(conv_layer(name, spec, bias != 0));
    });
}
mdnn_model* mdnn_batchnorm_layer(const char* name, int rank, const long* dims, unsigned long flags, int train,
                                 double eps, double mom)
{
    return guard_ptr<mdnn_model>(
        [&] { return wrapm(batchnorm_layer(name, mk(rank, dims), flags, train != 0, eps, mom)); });
}

void mdnn_modl_cfg_default(mdnn_modl_cfg* c)
{
    ModlConfig d;
    c->iterations = d.iterations;
    c->layers = d.layers;
    c->filters = d.filters;
    c->kernel = d.kernel;
    c->cg_iter = d.cg_iter;
    c->cg_tol = d.cg_tol;
    c->lambda_init = d.lambda_init;
    c->im_x = d.im_x;
    c->im_y = d.im_y;
    c->coils = d.coils;
    c->maps = d.maps;
    c->batch = d.batch;
    c->train_mode = d.train_mode ? 1 : 0;
}
void mdnn_varnet_cfg_default(mdnn_varnet_cfg* c)
{
    VarNetConfig d;
    c->iterations = d.iterations;
    c->filters = d.filters;
    c->kernel = d.kernel;
    c->rbf = d.rbf;
    c->im_x = d.im_x;
    c->im_y = d.im_y;
    c->coils = d.coils;
    c->maps = d.maps;
    c->batch = d.batch;
}
static ModlConfig to_modl(const mdnn_modl_cfg* c)
{
    ModlConfig m;
    m.iterations = c->iterations;
    m.layers = c->layers;
    m.filters = c->filters;
    m.kernel = c->kernel;
    m.cg_iter = c->cg_iter;
    m.cg_tol = c->cg_tol;
    m.lambda_init = c->lambda_init;
    m.im_x = c->im_x;
    m.im_y = c->im_y;
    m.coils = c->coils;
    m.maps = c->maps;
    m.batch = c->batch;
    m.train_mode = c->train_mode != 0;
    return m;
}
static VarNetConfig to_varnet(const mdnn_varnet_cfg* c)
{
    VarNetConfig v;
    v.iterations = c->iterations;
    v.filters = c->filters;
    v.kernel = c->kernel;
    v.rbf = c->rbf;
    v.im_x = c->im_x;
    v.im_y = c->im_y;
    v.coils = c->coils;
    v.maps = c->maps;
    v.batch = c->batch;
    return v;
}
mdnn_model* mdnn_bn_block(const char* name, int rank, const long* dims)
{
    return guard_ptr<mdnn_model>([&] {
        Dims d(dims, dims + rank);
        return wrapm(bn_block_fragment(name, d));
    });
}
mdnn_model* mdnn_modl_denoiser(const mdnn_modl_cfg* c)
{
    return guard_ptr<mdnn_model>([&] { return wrapm(modl_denoiser(to_modl(c), "")); });
}
mdnn_model* mdnn_varnet_reg(const mdnn_varnet_cfg* c)
{
    return guard_ptr<mdnn_model>([&] { return wrapm(varnet_reg(to_varnet(c), "it0")); });
}
mdnn_model* mdnn_model_rebatch(const mdnn_model* m, long batch)
{
    return guard_ptr<mdnn_model>([&] {
        if (!m->m.rebatch)
            throw ConfigError("model has no rebatch");
        if (batch < 1)
            throw ConfigError("rebatch: batch " + std::to_string(batch));
        return wrapm(m->m.rebatch(batch));
    });
}
mdnn_model* mdnn_build_modl(const mdnn_modl_cfg* c)
{
    return guard_ptr<mdnn_model>([&] {
        ModlConfig m;
        m.iterations = c->iterations;
        m.layers = c->layers;
        m.filters = c->filters;
        m.kernel = c->kernel;
        m.cg_iter = c->cg_iter;
        m.cg_tol = c->cg_tol;
        m.lambda_init = c->lambda_init;
        m.im_x = c->im_x;
        m.im_y = c->im_y;
        m.coils = c->coils;
        m.maps = c->maps;
        m.batch = c->batch;
        m.train_mode = c->train_mode != 0;
        return wrapm(build_modl(m));
    });
}
mdnn_model* mdnn_build_varnet(const mdnn_varnet_cfg* c)
{
    return guard_ptr<mdnn_model>([&] {
        VarNetConfig v;
        v.iterations = c->iterations;
        v.filters = c->filters;
        v.kernel = c->kernel;
        v.rbf = c->rbf;
        v.im_x = c->im_x;
        v.im_y = c->im_y;
        v.coils = c->coils;
        v.maps = c->maps;
        v.batch = c->batch;
        return wrapm(build_varnet(v));
    });
}
mdnn_model* mdnn_sense_normal_fragment(const mdnn_sense_dims* sd)
{
    return guard_ptr<mdnn_model>([&] { return wrapm(sense_normal_fragment(to_sd(sd))); });
}
mdnn_model* mdnn_sense_adjoint_fragment(const mdnn_sense_dims* sd)
{
    return guard_ptr<mdnn_model>([&] { return wrapm(sense_adjoint_fragment(to_sd(sd))); });
}
mdnn_model* mdnn_modl_normal_plus_lambda(const mdnn_sense_dims* sd)
{
    return guard_ptr<mdnn_model>([&] { return wrapm(modl_normal_plus_lambda(to_sd(sd))); });
}
mdnn_model* mdnn_loss_model_mse(int rank, const long* dims)
{
    return guard_ptr<mdnn_model>([&] { return wrapm(loss_model_mse(mk(rank, dims))); });
}

int mdnn_sim_item(uint64_t seed, long item, long x, long y, long coils, float* phantom, float* coil_maps)
{
    return guard([&] {
        Rng prng(hash_rand(seed, 2 * uint64_t(item)));
        Rng crng(hash_rand(seed, 2 * uint64_t(item) + 1));
        sim_phantom(reinterpret_cast<std::complex<float>*>(phantom), x, y, prng);
        sim_coils(reinterpret_cast<std::complex<float>*>(coil_maps), x, y, coils, crng);
    });
}

int mdnn_sim_pattern(long y, long accel, long acl, float* pattern)
{
    return guard([&] { sim_pattern(reinterpret_cast<std::complex<float>*>(pattern), y, accel, acl); });
}

// ---- training --------------------------------------------------------------
void mdnn_train_cfg_default(mdnn_train_cfg* c)
{
    TrainConfig d;
    c->lr = d.lr;
    c->beta1 = d.beta1;
    c->beta2 = d.beta2;
    c->eps = d.eps;
    c->clip = d.clip;
    c->algo = int(d.algo);
    c->ipalm_alpha = d.ipalm_alpha;
    c->ipalm_beta = d.ipalm_beta;
}

mdnn_trainer* mdnn_trainer_create(const mdnn_model* model, const mdnn_train_cfg* c, uint64_t seed)
{
    return guard_ptr<mdnn_trainer>([&] {
        TrainConfig cfg;
        cfg.lr = c->lr;
        cfg.beta1 = c->beta1;
        cfg.beta2 = c->beta2;
        cfg.eps = c->eps;
        cfg.clip = c->clip;
        if (c->algo < 0 || c->algo > 2)
            throw ConfigError("unknown optimizer id " + std::to_string(c->algo));
        cfg.algo = OptAlgo(c->algo);
        cfg.ipalm_alpha = c->ipalm_alpha;
        cfg.ipalm_beta = c->ipalm_beta;
        auto t = new mdnn_trainer{std::make_unique<Trainer>(model->m, cfg, seed)};
        sync_and_check();
        return t;
    });
}
void mdnn_trainer_free(mdnn_trainer* t) { delete t; }
int mdnn_trainer_set_data(mdnn_trainer* t, const char* name, const mdnn_array* a)
{
    return guard([&] { t->t->set_data(name, in_arr(*a)); });
}
int mdnn_trainer_stage_data(mdnn_trainer* t, const char* name, const mdnn_array* a)
{
    return guard([&] { t->t->stage_data(name, hv(*a)); });
}
int mdnn_trainer_set_weight(mdnn_trainer* t, const char* name, const mdnn_array* a)
{
    return guard([&] { t->t->set_weight(name, in_arr(*a)); });
}
int mdnn_trainer_get_weight(mdnn_trainer* t, const char* name, mdnn_array* out)
{
    return guard([&] {
        out_arr(t->t->weight(name), *out);
        sync_and_check();
    });
}
int mdnn_trainer_get_grad(mdnn_trainer* t, const char* name, mdnn_array* out)
{
    return guard([&] {
        out_arr(t->t->grad(name), *out);
        sync_and_check();
    });
}
int mdnn_trainer_forward_backward(mdnn_trainer* t, double* loss)
{
    return guard([&] {
        double l = t->t->forward_backward();
        if (loss)
            *loss = l;
    });
}
int mdnn_trainer_grad_buffer(mdnn_trainer* t, float** ptr, long* n)
{
    return guard([&] {
        *ptr = t->t->grad_buffer();
        *n = t->t->grad_floats();
    });
}
int mdnn_trainer_update(mdnn_trainer* t, float s)
{
    return guard([&] { t->t->update(s); });
}
int mdnn_trainer_step(mdnn_trainer* t, double* loss)
{
    return guard([&] {
        double l = t->t->step();
        if (loss)
            *loss = l;
    });
}
int mdnn_trainer_sync_buffer(mdnn_trainer* t, float** ptr, long* n)
{
    return guard([&] {
        *ptr = t->t->sync_buffer();
        *n = t->t->sync_floats();
    });
}
int mdnn_trainer_update_dp(mdnn_trainer* t, int world)
{
    return guard([&] { t->t->update_dp(world); });
}
int mdnn_nccl_unique_id(uint8_t* id128)
{
    return guard([&] { nccl_unique_id(id128); });
}
int mdnn_trainer_set_comm(mdnn_trainer* t, const uint8_t* id128, int nranks, int rank)
{
    return guard([&] { t->t->set_comm(std::make_unique<Comm>(id128, nranks, rank)); });
}
int mdnn_trainer_n_weights(const mdnn_trainer* t) { return int(t->t->weight_names().size()); }
const char* mdnn_trainer_weight_name(const mdnn_trainer* t, int k) { return t->t->weight_names().at(k).c_str(); }

} // extern "C"

// ---- cfl files and weight bundles -------------------------------------------
extern "C" {

int mdnn_cfl_dims(const char* base, long* dims16)
{
    return guard([&] {
        const Dims d = cfl_read_dims(base);
        for (int k = 0; k < max_rank; k++)
            dims16[k] = d[k];
    });
}

int mdnn_cfl_read(const char* base, mdnn_array* out)
{
    return guard([&] {
        DArray a = cfl_read(base);
        HostView v = hv(*out);
        Dims vd = v.dims;
        vd.resize(max_rank, 1);
        if (vd != a.dims)
            throw ShapeError(std::string("cfl_read: ") + base + " has dims " + dims_to_string(a.dims)
                             + ", output buffer " + dims_to_string(vd));
        DArray r = a; // same buffer, the caller's (possibly shorter) rank
        r.dims = v.dims;
        out_arr(r, *out);
        sync_and_check();
    });
}

int mdnn_cfl_write(const char* base, const mdnn_array* a)
{
    return guard([&] {
        cfl_write(base, in_arr(*a));
        sync_and_check();
    });
}

int mdnn_weights_save(mdnn_trainer* t, const char* dir, int n_meta, const char* const* keys,
                      const char* const* vals)
{
    return guard([&] {
        WeightsBundle b;
        for (int i = 0; i < n_meta; i++)
            b.meta[keys[i]] = vals[i];
        for (const auto& [name, arr] : t->t->all_weights()) // weights + moving statistics (cli.hpp:219-224)
            b.arrays.emplace(name, arr);
        b.save(dir);
        sync_and_check();
    });
}

int mdnn_weights_load(mdnn_trainer* t, const char* dir)
{
    return guard([&] {
        WeightsBundle b = WeightsBundle::load(dir);
        for (auto& [name, arr] : b.arrays) {
            // cfl arrays come back with 16 dims: keep the argument's own rank
            const auto& all = t->t->all_weights();
            auto it = all.find(name);
            if (it == all.end())
                throw ConfigError("trainer: no weight named '" + name + "'");
            Dims want = it->second.dims, wp = want;
            wp.resize(max_rank, 1);
            if (wp != arr.dims)
                throw ShapeError("weights bundle: array '" + name + "' has the wrong shape");
            DArray r = arr;
            r.dims = want;
            t->t->set_weight(name, r);
        }
        sync_and_check();
    });
}

int mdnn_weights_meta(const char* dir, const char* key, const char* fallback, char* buf, long buflen)
{
    return guard([&] {
        // manifest only (arrays are not read)
        std::ifstream mf(std::string(dir) + "/manifest.txt");
        if (!mf)
            throw IoError(std::string("missing weights manifest in ") + dir);
        std::string line, val = fallback ? fallback : "";
        while (std::getline(mf, line)) {
            const auto sp = line.find(' ');
            if (line.substr(0, sp) == key && std::string(key) != "array")
                val = sp == std::string::npos ? "" : line.substr(sp + 1);
        }
        if (long(val.size()) + 1 > buflen)
            throw BoundsError("mdnn_weights_meta: buffer too small");
        std::memcpy(buf, val.c_str(), val.size() + 1);
    });
}

} // extern "C"

// ---- reconet driver -----------------------------------------------------------
extern "C" {

void mdnn_reconet_opts_default(mdnn_reconet_opts* o)
{
    std::memset(o, 0, sizeof(*o));
    o->network = "varnet";
    o->iterations = o->filters = o->kernel = o->rbf = o->layers = o->cg_iter = -1;
    o->epochs = 10;
    o->batch_size = 10;
    o->lr = -1;
    o->seed = 42;
    o->verbose = 1;
}

int mdnn_reconet(const mdnn_reconet_opts* c)
{
    return guard([&] {
        auto str = [](const char* p) { return std::string(p ? p : ""); };
        ReconetOptions o;
        o.network = str(c->network);
        o.do_train = c->do_train != 0;
        o.do_apply = c->do_apply != 0;
        o.normalize = c->normalize != 0;
        o.pattern_file = str(c->pattern_file);
        o.init_weights = str(c->init_weights);
        o.iterations = c->iterations;
        o.filters = c->filters;
        o.kernel = c->kernel;
        o.rbf = c->rbf;
        o.layers = c->layers;
        o.cg_iter = c->cg_iter;
        o.epochs = c->epochs;
        o.batch_size = c->batch_size;
        o.lr = c->lr;
        o.optimizer = str(c->optimizer);
        o.seed = c->seed;
        o.verbose = c->verbose != 0;
        o.kspace_file = str(c->kspace_file);
        o.coils_file = str(c->coils_file);
        o.weights_dir = str(c->weights_dir);
        o.target_file = str(c->target_file);
        run_reconet(o);
    });
}

int mdnn_estimate_pattern(const mdnn_array* kspace, mdnn_array* pattern)
{
    return guard([&] {
        out_arr(estimate_pattern(in_arr(*kspace)), *pattern);
        sync_and_check();
    });
}

} // extern "C"
