#include "model.h"

#include "kernels.h"

#include <algorithm>

namespace mdnn {

int Model::arg_index(const std::string& name) const
{
    for (size_t i = 0; i < args.size(); i++)
        if (args[i].name == name)
            return int(i);
    throw ConfigError("model: no argument named '" + name + "'");
}

int Model::output_index(const std::string& name) const
{
    for (size_t i = 0; i < out_names.size(); i++)
        if (out_names[i] == name)
            return int(i);
    throw ConfigError("model: no output named '" + name + "'");
}

long Model::num_real_params() const
{
    long n = 0;
    for (size_t i = 0; i < args.size(); i++)
        if (args[i].kind == ArgKind::Weights)
            n += md_size(op.in_dims(int(i))) * (args[i].real_weights ? 1 : 2);
    return n;
}

// nn.hpp:117-145: Glorot uniform from Rng(derive_seed(seed, name)), canonical order
std::vector<std::complex<float>> Model::init_weight(uint64_t seed, int i) const
{
    const Arg& a = args.at(i);
    if (a.kind == ArgKind::Data)
        throw ConfigError("init_weight: '" + a.name + "' is a data argument");
    std::vector<std::complex<float>> v(size_t(md_size(op.in_dims(i))), {0.f, 0.f});
    switch (a.init.kind) {
    case Initializer::None:
        break;
    case Initializer::Constant:
        std::fill(v.begin(), v.end(), std::complex<float>(float(a.init.value), 0.f));
        break;
    case Initializer::GlorotUniform: {
        Rng rng(derive_seed(seed, a.name));
        double bound = std::sqrt(6.0 / double(a.init.fan_in + a.init.fan_out));
        for (auto& e : v) {
            double re = rng.uniform(-bound, bound);
            double im = a.real_weights ? 0.0 : rng.uniform(-bound, bound);
            e = {float(re), float(im)};
        }
        break;
    }
    }
    return v;
}

Model model_chain(const Model& a, const Model& b, const std::string& b_in, int a_out)
{
    if (a_out < 0)
        a_out = a.output_index("out");
    int bi = b.arg_index(b_in);
    Model m;
    m.op = link(combine(a.op, b.op), a_out, a.op.n_in() + bi);
    m.args = a.args;
    for (size_t i = 0; i < b.args.size(); i++)
        if (int(i) != bi)
            m.args.push_back(b.args[i]);
    m.out_names = a.out_names;
    m.out_names.erase(m.out_names.begin() + a_out);
    m.out_names.insert(m.out_names.end(), b.out_names.begin(), b.out_names.end());
    return m;
}

Model model_link(Model m, int out_idx, const std::string& arg)
{
    int ai = m.arg_index(arg);
    m.op = link(m.op, out_idx, ai);
    m.args.erase(m.args.begin() + ai);
    m.out_names.erase(m.out_names.begin() + out_idx);
    return m;
}

Model model_combine(const Model& a, const Model& b)
{
    Model m;
    m.op = combine(a.op, b.op);
    m.args = a.args;
    m.args.insert(m.args.end(), b.args.begin(), b.args.end());
    m.out_names = a.out_names;
    m.out_names.insert(m.out_names.end(), b.out_names.begin(), b.out_names.end());
    return m;
}

Model model_dedupe(Model m)
{
    for (size_t i = 0; i < m.args.size(); i++)
        for (size_t j = i + 1; j < m.args.size();) {
            if (m.args[j].name == m.args[i].name) {
                m.op = duplicate(m.op, int(i), int(j));
                m.args.erase(m.args.begin() + j);
            } else {
                j++;
            }
        }
    return m;
}

static Model plain(Nlop op, std::vector<Arg> args, std::vector<std::string> outs)
{
    Model m;
    m.op = std::move(op);
    m.args = std::move(args);
    m.out_names = std::move(outs);
    return m;
}

// nn.hpp:344-426
Model conv_layer(const std::string& name, const ConvSpec& spec, bool bias)
{
    if (spec.axes.size() != spec.kernel.size())
        throw ConfigError("conv: one kernel extent per axis required");
    for (size_t a = 0; a < spec.axes.size(); a++)
        if (!spec.pad_same && spec.kernel[a] > spec.in_dims.at(spec.axes[a]))
            throw ShapeError("conv: kernel larger than padded input");
    long fan_k = 1;
    for (long k : spec.kernel)
        fan_k *= k;
    auto w_init = Initializer::glorot(fan_k * spec.in_dims[spec.chan_dim], fan_k * spec.out_channels);
    Arg w{name + "_w", ArgKind::Weights, w_init, ProxKind::None, false};
    Model m;
    m.op = conv_core(name, spec);
    m.args = spec.transposed ? std::vector<Arg>{w, data_arg("x")} : std::vector<Arg>{data_arg("x"), w};
    m.out_names = {"out"};
    if (bias) {
        Dims final_out = spec.transposed ? spec.in_dims : spec.out_dims();
        Dims b_dims(final_out.size(), 1);
        b_dims[spec.chan_dim] = final_out[spec.chan_dim];
        Model bm = plain(Nlop(node_bcast_add(final_out, b_dims)),
                         {data_arg("x"),
                          Arg{name + "_b", ArgKind::Weights, Initializer::constant(0), ProxKind::None, false}},
                         {"out"});
        m = model_chain(m, bm, "x");
    }
    return m;
}

// nn.hpp:441-453
Model batchnorm_layer(const std::string& name, const Dims& dims, unsigned long flags, bool train, double eps,
                      double momentum)
{
    Model m;
    m.op = Nlop(node_batchnorm(dims, flags, train, eps, momentum));
    m.args = {data_arg("x"), Arg{name + "_mean", ArgKind::MovingStats, Initializer::constant(0), ProxKind::None, false},
              Arg{name + "_var", ArgKind::MovingStats, Initializer::constant(1), ProxKind::None, false}};
    m.out_names = train ? std::vector<std::string>{"out", name + "_mean", name + "_var"}
                        : std::vector<std::string>{"out"};
    return m;
}

Model loss_model_mse(const Dims& dims)
{
    return plain(Nlop(node_mse(dims)), {data_arg("prediction"), data_arg("reference")}, {"loss"});
}

// recon.hpp:412-418 — one fused node; args (x, coils, pattern, coils) as the reference's chained fragment
Model sense_normal_fragment(const SenseDims& sd)
{
    return plain(Nlop(node_sense_normal(sd)), {data_arg("x"), data_arg("coils"), data_arg("pattern"), data_arg("coils")},
                 {"out"});
}

// recon.hpp:402-408 — args (x, pattern, coils)
Model sense_adjoint_fragment(const SenseDims& sd)
{
    return plain(Nlop(node_sense_adjoint(sd)), {data_arg("x"), data_arg("pattern"), data_arg("coils")}, {"out"});
}

// recon.hpp:807-820 — args after dedupe: (x, coils, pattern, lambda)
Model modl_normal_plus_lambda(const SenseDims& sd)
{
    return plain(Nlop(node_sense_normal_lambda(sd)),
                 {data_arg("x"), data_arg("coils"), data_arg("pattern"), data_arg("lambda")}, {"out"});
}

// builder fragments (recon.hpp:421-680)

Model scalar_mul_fragment(const SenseDims& sd, const std::string& scalar_name, ArgKind kind)
{
    // recon.hpp:421-431
    Dims sdims(max_rank, 1);
    Dims iter = sd.image();
    Dims s_img = default_strides(iter);
    Dims s_sc(max_rank, 0);
    return plain(Nlop(node_tenmul("scale_" + scalar_name, iter, iter, s_img, iter, s_img, sdims, s_sc)),
                 {data_arg("x"), Arg{scalar_name, kind, {}, ProxKind::None, false}}, {"out"});
}

Model add_fragment(const Dims& dims, bool sub)
{
    return plain(Nlop(node_add(dims, sub)), {data_arg("a"), data_arg("b")}, {"out"});
}

Model first_map_slice(const SenseDims& sd)
{
    Dims out = sd.image();
    out[dim_maps] = 1;
    Dims corner(max_rank, 0);
    // linop_slice (linop.hpp:172-183) = crop of the first map set
    return plain(Nlop(node_pad(out, sd.image(), corner, true)), {data_arg("x")}, {"out"});
}

Model embed_first_map(const SenseDims& sd)
{
    Dims small = sd.image();
    small[dim_maps] = 1;
    Dims corner(max_rank, 0);
    return plain(Nlop(node_pad(small, sd.image(), corner, false)), {data_arg("x")}, {"out"});
}

// one layer's train-mode BN -> gamma -> beta -> CReLU (recon.hpp:748-776) as
// the fused channels-last node, standalone (no TF32 rounding of its output or
// input cotangent: no tensor-core conv neighbours)
Model bn_block_fragment(const std::string& ln, const Dims& cur)
{
    return plain(Nlop(node_bnblock(cur, false, false)),
                 {data_arg("x"),
                  Arg{ln + "_bn_mean", ArgKind::MovingStats, Initializer::constant(0), ProxKind::None, false},
                  Arg{ln + "_bn_var", ArgKind::MovingStats, Initializer::constant(1), ProxKind::None, false},
                  Arg{ln + "_g", ArgKind::Weights, Initializer::constant(1), ProxKind::None, false},
                  Arg{ln + "_beta", ArgKind::Weights, Initializer::constant(0), ProxKind::None, false}},
                 {ln + "_bn_mean", ln + "_bn_var", "out"});
}

// recon.hpp:714-803, CNN output resolved by name (the shipped builder's
// hard-coded index 1 is a BN statistic in train mode)
Model modl_denoiser(const ModlConfig& cfg, const std::string& stat_suffix)
{
    SenseDims sd = cfg.sense();
    SenseDims sd1 = sd;
    sd1.maps = 1;
    Model cnn;
    if (sd.maps > 1)
        cnn = first_map_slice(sd);
    Dims cur = sd1.image();
    const unsigned long bn_flags = (1UL << dim_x) | (1UL << dim_y) | (1UL << dim_batch);
    // train mode with a supported width: the BN / gamma / beta / CReLU chain runs
    // as one fused channels-last node, and every conv of the chain keeps its
    // feature maps channels-last (no layout conversions inside the denoiser)
    const bool fused = cfg.train_mode && bnblock_supported(cfg.filters) && cfg.layers >= 2;
    auto is_tc = [&](long cin, long cout) { return conv_tc_supported(cin, cout, cfg.kernel, cfg.kernel); };
    for (long l = 0; l < cfg.layers; l++) {
        const bool last = l + 1 == cfg.layers;
        const std::string ln = "dw" + std::to_string(l);
        ConvSpec spec;
        spec.in_dims = cur;
        spec.axes = {dim_x, dim_y};
        spec.kernel = {cfg.kernel, cfg.kernel};
        spec.chan_dim = dim_chan;
        spec.out_channels = last ? 1 : cfg.filters;
        spec.pad_same = true;
        spec.chlast_hint = fused ? 1 : 0;
        Model conv = conv_layer(ln, spec, last);
        cnn = cnn.valid() ? model_chain(cnn, conv, "x") : conv;
        const long cin = cur[dim_chan];
        cur = spec.out_dims();
        if (last)
            break;
        if (fused) {
            const bool next_tc = is_tc(cfg.filters, l + 2 == cfg.layers ? 1 : cfg.filters);
            const bool this_tc = is_tc(cin, cfg.filters);
            Model blk = plain(Nlop(node_bnblock(cur, next_tc, this_tc)),
                              {data_arg("x"),
                               Arg{ln + "_bn_mean", ArgKind::MovingStats, Initializer::constant(0), ProxKind::None, false},
                               Arg{ln + "_bn_var", ArgKind::MovingStats, Initializer::constant(1), ProxKind::None, false},
                               Arg{ln + "_g", ArgKind::Weights, Initializer::constant(1), ProxKind::None, false},
                               Arg{ln + "_beta", ArgKind::Weights, Initializer::constant(0), ProxKind::None, false}},
                              {ln + "_bn_mean" + stat_suffix, ln + "_bn_var" + stat_suffix, "out"});
            cnn = model_chain(cnn, blk, "x");
            continue;
        }
        Model bn = batchnorm_layer(ln + "_bn", cur, bn_flags, cfg.train_mode);
        if (!stat_suffix.empty() && cfg.train_mode)
            for (auto& n : bn.out_names)
                if (n != "out")
                    n += stat_suffix;
        cnn = model_chain(cnn, bn, "x");
        Dims gdims(max_rank, 1);
        gdims[dim_chan] = cur[dim_chan];
        Dims sc = default_strides(cur);
        Dims sg(max_rank, 0);
        sg[dim_chan] = 1;
        Model gamma = plain(Nlop(node_tenmul("bn_scale" + std::to_string(l), cur, cur, sc, cur, sc, gdims, sg)),
                            {data_arg("x"), Arg{ln + "_g", ArgKind::Weights, Initializer::constant(1), ProxKind::None,
                                                false}},
                            {"out"});
        cnn = model_chain(cnn, gamma, "x");
        Model beta = plain(Nlop(node_bcast_add(cur, gdims)),
                           {data_arg("x"), Arg{ln + "_beta", ArgKind::Weights, Initializer::constant(0),
                                               ProxKind::None, false}},
                           {"out"});
        cnn = model_chain(cnn, beta, "x");
        Model act = plain(Nlop(node_crelu(cur)), {data_arg("x")}, {"out"});
        cnn = model_chain(cnn, act, "x");
    }
    if (sd.maps > 1)
        cnn = model_chain(cnn, embed_first_map(sd), "x");
    Model fork = plain(Nlop(node_fork(sd.image(), 2)), {data_arg("x")}, {"cnn_in", "skip"});
    Model f = model_chain(fork, cnn, "x", 0);
    f = model_chain(f, add_fragment(sd.image(), false), "a", f.output_index("out"));
    return model_link(f, f.output_index("skip"), "b");
}

// recon.hpp:826-869
Model modl_step(const ModlConfig& cfg, const std::string& stat_suffix)
{
    SenseDims sd = cfg.sense();
    Dims img = sd.image();
    Dims sdims(max_rank, 1);
    Model dw = modl_denoiser(cfg, stat_suffix);
    Model lam = plain(Nlop(node_exp_real(sdims)),
                      {Arg{"lam_log", ArgKind::Weights, Initializer::constant(std::log(cfg.lambda_init)),
                           ProxKind::None, true}},
                      {"out"});
    Model lam_fork = plain(Nlop(node_fork(sdims, 2)), {data_arg("x")}, {"lam_rhs", "lam_inv"});
    lam = model_chain(lam, lam_fork, "x");
    Model rhs = model_chain(dw, scalar_mul_fragment(sd, "lam_mul", ArgKind::Data), "x");
    rhs = model_chain(rhs, add_fragment(img, false), "a");
    rhs.out_names[rhs.output_index("out")] = "rhs";
    Model s_model = modl_normal_plus_lambda(sd);
    Model inv;
    inv.op = Nlop(node_inverse(s_model.op, cfg.cg_iter, cfg.cg_tol));
    inv.args = s_model.args;
    inv.args[0] = data_arg("y");
    inv.out_names = {"out"};
    Model m = model_combine(lam, model_combine(rhs, inv));
    m = model_link(m, m.output_index("lam_rhs"), "lam_mul");
    m = model_link(m, m.output_index("lam_inv"), "lambda");
    m = model_link(m, m.output_index("rhs"), "y");
    for (auto& a : m.args)
        if (a.name == "b")
            a.name = "x0";
    return model_dedupe(std::move(m));
}

// recon.hpp:522-609
Model varnet_reg(const VarNetConfig& cfg, const std::string& prefix)
{
    SenseDims sd = cfg.sense();
    SenseDims sd1 = sd;
    sd1.maps = 1;
    Dims img1 = sd1.image();
    Model m;
    if (sd.maps > 1)
        m = first_map_slice(sd);
    Model rc = plain(Nlop(node_real_chan(img1, dim_chan)), {data_arg("x")}, {"out"});
    m = m.valid() ? model_chain(m, rc, "x") : rc;
    Dims chan_img = img1;
    chan_img[dim_chan] = 2;
    ConvSpec spec;
    spec.in_dims = chan_img;
    spec.axes = {dim_x, dim_y};
    spec.kernel = {cfg.kernel, cfg.kernel};
    spec.chan_dim = dim_chan;
    spec.out_channels = cfg.filters;
    spec.pad_same = true;
    Model conv = conv_layer(prefix + "_k", spec, false);
    conv.args[conv.arg_index(prefix + "_k_w")].real_weights = true;
    m = model_chain(m, conv, "x");
    Dims feat = spec.out_dims();
    m = model_chain(m, plain(Nlop(node_zreal(feat)), {data_arg("x")}, {"out"}), "x");
    std::vector<float> centers(cfg.rbf);
    float spacing = float(2.0 / double(cfg.rbf - 1));
    for (long j = 0; j < cfg.rbf; j++)
        centers[j] = -1.f + float(j) * spacing;
    Model act = plain(Nlop(node_rbf(feat, dim_chan, centers, spacing)),
                      {data_arg("x"),
                       Arg{prefix + "_rbf_w", ArgKind::Weights, Initializer::constant(0), ProxKind::None, true}},
                      {"out"});
    m = model_chain(m, act, "x");
    ConvSpec tspec = spec;
    tspec.transposed = true;
    Model convt = conv_layer(prefix + "_k", tspec, false);
    convt.args[convt.arg_index(prefix + "_k_w")].real_weights = true;
    m = model_chain(m, convt, "x");
    m = model_chain(m, plain(Nlop(node_chan_cplx(chan_img, dim_chan)), {data_arg("x")}, {"out"}), "x");
    if (sd.maps > 1)
        m = model_chain(m, embed_first_map(sd), "x");
    return model_dedupe(std::move(m));
}

// recon.hpp:618-645, with the x0 link into the add's own "b"
Model varnet_step(const VarNetConfig& cfg, const std::string& prefix)
{
    SenseDims sd = cfg.sense();
    Dims img = sd.image();
    Model reg = varnet_reg(cfg, prefix);
    Model dc = sense_normal_fragment(sd);
    dc = model_chain(dc, add_fragment(img, true), "a");
    dc = model_chain(dc, scalar_mul_fragment(sd, prefix + "_lam", ArgKind::Weights), "x");
    auto& lam = dc.args[dc.arg_index(prefix + "_lam")];
    lam.init = Initializer::constant(1.0);
    lam.real_weights = true;
    lam.prox = ProxKind::NonNeg;
    Model m = model_combine(reg, dc);
    m = model_chain(m, add_fragment(img, false), "a", 0);
    {
        const int last = int(m.args.size()) - 1;
        m.op = link(m.op, 0, last);
        m.args.erase(m.args.begin() + last);
        m.out_names.erase(m.out_names.begin());
    }
    m = model_chain(m, add_fragment(img, true), "b", 0);
    for (auto& a : m.args) {
        if (a.name == "a")
            a.name = "x";
        else if (a.name == "b")
            a.name = "x0";
    }
    return model_dedupe(std::move(m));
}



void ModlConfig::validate() const
{
    if (iterations < 1 || layers < 1 || filters < 1 || cg_iter < 1)
        throw ConfigError("modl: invalid hyperparameters");
    if (im_x < 1 || im_y < 1)
        throw ConfigError("modl: image size not set");
}

void VarNetConfig::validate() const
{
    if (iterations < 1 || filters < 1 || kernel < 1 || rbf < 2)
        throw ConfigError("varnet: invalid hyperparameters");
    if (im_x < 1 || im_y < 1)
        throw ConfigError("varnet: image size not set");
}

// recon.hpp:875-904
Model build_modl(const ModlConfig& cfg)
{
    cfg.validate();
    SenseDims sd = cfg.sense();
    Model adj = sense_adjoint_fragment(sd);
    adj.args[adj.arg_index("x")].name = "kspace";
    Model fork = plain(Nlop(node_fork(sd.image(), 2)), {data_arg("x")}, {"out", "x0src"});
    Model net = model_chain(adj, fork, "x");
    for (long t = 0; t < cfg.iterations; t++) {
        const bool last = t + 1 == cfg.iterations;
        Model step = modl_step(cfg, last ? "" : "@" + std::to_string(t));
        net = model_chain(net, step, "x", net.output_index("out"));
        net = model_dedupe(std::move(net));
    }
    net = model_link(net, net.output_index("x0src"), "x0");
    net.rebatch = [cfg](long b) {
        ModlConfig c = cfg;
        c.batch = b;
        return build_modl(c);
    };
    return net;
}

// recon.hpp:652-680
Model build_varnet(const VarNetConfig& cfg)
{
    cfg.validate();
    SenseDims sd = cfg.sense();
    Model adj = sense_adjoint_fragment(sd);
    adj.args[adj.arg_index("x")].name = "kspace";
    Model fork = plain(Nlop(node_fork(sd.image(), 2)), {data_arg("x")}, {"out", "x0src"});
    Model net = model_chain(adj, fork, "x");
    for (long t = 0; t < cfg.iterations; t++) {
        Model step = varnet_step(cfg, "it" + std::to_string(t));
        net = model_chain(net, step, "x", net.output_index("out"));
        net = model_dedupe(std::move(net));
    }
    net = model_link(net, net.output_index("x0src"), "x0");
    net.rebatch = [cfg](long b) {
        VarNetConfig c = cfg;
        c.batch = b;
        return build_varnet(c);
    };
    return net;
}

// ---- simulate.hpp:40-133 ------------------------------------------------------
void sim_phantom(std::complex<float>* v, long nx, long ny, Rng& rng)
{
    const int n_ell = 4 + int(rng.below(5));
    struct Ell {
        double cx, cy, ax, ay, cs, sn, amp;
    };
    std::vector<Ell> ells;
    for (int e = 0; e < n_ell; e++) {
        double th = rng.uniform(0, 2 * M_PI);
        Ell el;
        el.cx = rng.uniform(-0.55, 0.55);
        el.cy = rng.uniform(-0.55, 0.55);
        el.ax = rng.uniform(0.12, 0.5);
        el.ay = rng.uniform(0.12, 0.5);
        el.cs = std::cos(th);
        el.sn = std::sin(th);
        el.amp = rng.uniform(0.25, 1.0);
        ells.push_back(el);
    }
    double p1 = rng.uniform(-2, 2), p2 = rng.uniform(-2, 2), p3 = rng.uniform(-1, 1);
    for (long j = 0; j < ny; j++) {
        double y = 2.0 * double(j) / double(ny - 1) - 1.0;
        for (long i = 0; i < nx; i++) {
            double x = 2.0 * double(i) / double(nx - 1) - 1.0;
            double mag = 0;
            for (const auto& e : ells) {
                double dx = x - e.cx, dy = y - e.cy;
                double u = (dx * e.cs + dy * e.sn) / e.ax;
                double w = (-dx * e.sn + dy * e.cs) / e.ay;
                double r2 = u * u + w * w;
                if (r2 < 1.0)
                    mag += e.amp * (1.0 - r2);
            }
            double ph = p1 * x + p2 * y + p3 * x * y;
            v[i + nx * j] = {float(mag * std::cos(ph)), float(mag * std::sin(ph))};
        }
    }
}

void sim_coils(std::complex<float>* v, long nx, long ny, long nc, Rng& rng)
{
    const long cstride = nx * ny;
    for (long c = 0; c < nc; c++) {
        double ang = 2 * M_PI * (double(c) + rng.uniform(-0.15, 0.15)) / double(nc);
        double cx = 1.3 * std::cos(ang), cy = 1.3 * std::sin(ang);
        double w = rng.uniform(0.9, 1.3);
        double px = rng.uniform(-0.8, 0.8), py = rng.uniform(-0.8, 0.8);
        for (long j = 0; j < ny; j++) {
            double y = 2.0 * double(j) / double(ny - 1) - 1.0;
            for (long i = 0; i < nx; i++) {
                double x = 2.0 * double(i) / double(nx - 1) - 1.0;
                double d2 = (x - cx) * (x - cx) + (y - cy) * (y - cy);
                double mag = std::exp(-d2 / (2 * w * w));
                double ph = px * x + py * y;
                v[i + nx * j + c * cstride] = {float(mag * std::cos(ph)), float(mag * std::sin(ph))};
            }
        }
    }
    for (long j = 0; j < ny; j++)
        for (long i = 0; i < nx; i++) {
            double ss = 0;
            for (long c = 0; c < nc; c++) {
                auto z = v[i + nx * j + c * cstride];
                ss += double(z.real()) * z.real() + double(z.imag()) * z.imag();
            }
            float f = float(1.0 / std::sqrt(ss));
            for (long c = 0; c < nc; c++)
                v[i + nx * j + c * cstride] *= f;
        }
}

void sim_pattern(std::complex<float>* v, long size, long accel, long acl)
{
    for (long k = 0; k < size; k++) {
        bool regular = (k % accel) == 0;
        long dist = std::min(k, size - k);
        bool in_acl = 2 * dist < acl;
        v[k] = (regular || in_acl) ? std::complex<float>(1.f, 0.f) : std::complex<float>(0.f, 0.f);
    }
}

} // namespace mdnn
