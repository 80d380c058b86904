// `reconet` driver (cli.hpp:94-265): the train / apply loop either side of
// the training step, on device arrays.
//
//   cfl inputs -> (estimate_pattern, cli.hpp:28-50) -> (normalize: per-item
//   1 / max |A^H y|, recon.hpp:464-482) -> train: seeded epoch shuffle, batch
//   gather, run_step per batch (optim.hpp:218-310), weights bundle out;
//   apply: chunked batched inference (MoDL with inference-mode BN), inverse
//   scaling (recon.hpp:484-493), cfl out.
//
// Same option semantics and error taxonomy as the reference command; the CLI
// parsing itself (CLI11) stays out of scope — callers fill mdnn_reconet_opts.
#include "reconet.h"

#include "cfl.h"
#include "kernels.h"
#include "model.h"
#include "train.h"

#include <algorithm>
#include <cmath>
#include <cstdio>

namespace mdnn {

void launch_estimate_pattern(cfloat* pattern, const cfloat* kspace, long X, long Y, long rest);
void launch_item_maxabs(double* out, const cfloat* x, long per_item, long items);
void launch_scale_items(cfloat* out, const cfloat* in, const cfloat* scale, long per_item, long items, bool invert);

namespace {

void check_dim_match(const std::string& fa, const DArray& a, const std::string& fb, const DArray& b, int dim)
{
    if (a.dims[dim] != b.dims[dim])
        throw ShapeError("file '" + fa + "' dimension " + std::to_string(dim) + " (=" + std::to_string(a.dims[dim])
                         + ") does not match file '" + fb + "' dimension " + std::to_string(dim) + " (="
                         + std::to_string(b.dims[dim]) + ")");
}

void check_pattern_binary(const DArray& p)
{
    // recon.hpp:67-77
    for (auto& v : to_host(p))
        if (v.imag() != 0 || (v.real() != 0 && v.real() != 1))
            throw ConfigError("sense: sampling pattern must be binary");
}

long meta_long(const WeightsBundle& b, const std::string& key, long fallback)
{
    auto it = b.meta.find(key);
    return it == b.meta.end() ? fallback : std::stol(it->second);
}

// items [pos, pos + cnt) of a batch-stacked array (dim 15 outermost: contiguous)
DArray slice_items(const DArray& a, long pos, long cnt)
{
    Dims d = a.dims;
    const long per = md_size(d) / d[dim_batch];
    d[dim_batch] = cnt;
    DArray o(d, false);
    CUDA_CHECK(cudaMemcpyAsync(o.data(), a.data() + pos * per, sizeof(cfloat) * per * cnt, cudaMemcpyDeviceToDevice,
                               ctx().stream));
    return o;
}

// detail::gather_batch (optim.hpp): items in shuffled order
DArray gather_items(const DArray& a, const long* items, long cnt)
{
    Dims d = a.dims;
    const long per = md_size(d) / d[dim_batch];
    d[dim_batch] = cnt;
    DArray o(d, false);
    for (long k = 0; k < cnt; k++)
        CUDA_CHECK(cudaMemcpyAsync(o.data() + k * per, a.data() + items[k] * per, sizeof(cfloat) * per,
                                   cudaMemcpyDeviceToDevice, ctx().stream));
    return o;
}

SenseGeom geom_of_data(const DArray& coils, const DArray& pattern)
{
    SenseGeom g{};
    g.X = coils.dims[dim_x];
    g.Y = coils.dims[dim_y];
    g.C = coils.dims[dim_coil];
    g.M = coils.dims[dim_maps];
    g.B = coils.dims[dim_batch];
    g.pat_x = pattern.dims[dim_x];
    g.pat_y = pattern.dims[dim_y];
    g.pat_c = pattern.dims[dim_coil];
    g.pat_b = pattern.dims[dim_batch];
    return g;
}

std::vector<DArray> gather_model_inputs(const Model& m, const std::map<std::string, DArray>& weights,
                                        const std::map<std::string, DArray>& data)
{
    std::vector<DArray> in;
    for (size_t i = 0; i < m.args.size(); i++) {
        const auto& a = m.args[i];
        const auto& src = a.kind == ArgKind::Data ? data : weights;
        auto it = src.find(a.name);
        if (it == src.end())
            throw ConfigError("model: missing array for argument '" + a.name + "'");
        DArray v = it->second;
        const Dims& want = m.op.in_dims(int(i));
        if (v.dims != want) { // bundle arrays come back with 16 dims
            Dims p = want, q = v.dims;
            p.resize(max_rank, 1);
            q.resize(max_rank, 1);
            if (p != q)
                throw ShapeError("model: argument '" + a.name + "' expected " + dims_to_string(want) + ", got "
                                 + dims_to_string(v.dims));
            v.dims = want;
        }
        in.push_back(v);
    }
    return in;
}

} // namespace

DArray estimate_pattern(const DArray& kspace)
{
    Dims pd(max_rank, 1);
    pd[dim_y] = kspace.dims[dim_y];
    DArray p(pd, false);
    const long X = kspace.dims[dim_x], Y = kspace.dims[dim_y];
    launch_estimate_pattern(p.data(), kspace.data(), X, Y, md_size(kspace.dims) / (X * Y));
    return p;
}

int run_reconet(ReconetOptions o)
{
    if (o.do_train == o.do_apply)
        throw ConfigError("reconet: exactly one of --train / --apply is required");
    if (o.network != "varnet" && o.network != "modl")
        throw ConfigError("reconet: --network must be varnet or modl");

    DArray kspace = cfl_read(o.kspace_file);
    DArray coils = cfl_read(o.coils_file);
    for (int d : {dim_x, dim_y, dim_coil, dim_batch})
        check_dim_match(o.coils_file, coils, o.kspace_file, kspace, d);
    DArray pattern = o.pattern_file.empty() ? estimate_pattern(kspace) : cfl_read(o.pattern_file);
    check_dim_match(o.pattern_file.empty() ? "<estimated pattern>" : o.pattern_file, pattern, o.kspace_file, kspace,
                    dim_y);
    check_pattern_binary(pattern);

    const long n = kspace.dims[dim_batch];
    const long maps = coils.dims[dim_maps];
    VarNetConfig vn;
    ModlConfig md;
    vn.im_x = md.im_x = kspace.dims[dim_x];
    vn.im_y = md.im_y = kspace.dims[dim_y];
    vn.coils = md.coils = kspace.dims[dim_coil];
    vn.maps = md.maps = maps;

    WeightsBundle bundle;
    if (o.do_apply || !o.init_weights.empty()) {
        bundle = WeightsBundle::load(o.do_apply ? o.weights_dir : o.init_weights);
        if (bundle.meta_or("network", o.network) != o.network)
            throw ConfigError("weights bundle was trained for network '" + bundle.meta_or("network", "?") + "', not '"
                              + o.network + "'");
        auto take = [&](const std::string& key, long& dst) { dst = meta_long(bundle, key, dst); };
        if (o.network == "varnet") {
            take("iterations", vn.iterations);
            take("filters", vn.filters);
            take("kernel", vn.kernel);
            take("rbf", vn.rbf);
        } else {
            take("iterations", md.iterations);
            take("layers", md.layers);
            take("filters", md.filters);
            take("kernel", md.kernel);
            take("cg_iter", md.cg_iter);
        }
        if (o.do_apply)
            o.normalize = bundle.meta_or("normalize", "0") == "1";
    }
    auto override_long = [](long flag, long& dst, const char* what, bool frozen) {
        if (flag < 0)
            return;
        if (frozen && flag != dst)
            throw ConfigError(std::string("flag --") + what + " conflicts with the weights bundle");
        dst = flag;
    };
    const bool frozen = o.do_apply;
    if (o.network == "varnet") {
        override_long(o.iterations, vn.iterations, "iterations", frozen);
        override_long(o.filters, vn.filters, "filters", frozen);
        override_long(o.kernel, vn.kernel, "kernel", frozen);
        override_long(o.rbf, vn.rbf, "rbf", frozen);
    } else {
        override_long(o.iterations, md.iterations, "iterations", frozen);
        override_long(o.layers, md.layers, "layers", frozen);
        override_long(o.filters, md.filters, "filters", frozen);
        override_long(o.cg_iter, md.cg_iter, "cg-iter", frozen);
    }

    // per-item scaling from the adjoint reconstruction (recon.hpp:464-482)
    DArray scale;
    if (o.normalize) {
        const SenseGeom g = geom_of_data(coils, pattern);
        Dims xd(max_rank, 1);
        xd[dim_x] = g.X;
        xd[dim_y] = g.Y;
        xd[dim_maps] = g.M;
        xd[dim_batch] = n;
        DArray x0(xd, false);
        sense_adjoint(x0.data(), kspace.data(), coils.data(), pattern.data(), g);
        DArray mx(Dims{n}, false); // doubles, n of them fit in n complex slots
        launch_item_maxabs(reinterpret_cast<double*>(mx.data()), x0.data(), md_size(xd) / n, n);
        std::vector<double> h(static_cast<size_t>(n));
        CUDA_CHECK(cudaMemcpyAsync(h.data(), mx.data(), sizeof(double) * n, cudaMemcpyDeviceToHost, ctx().stream));
        sync_and_check();
        std::vector<std::complex<float>> s(static_cast<size_t>(n));
        for (long k = 0; k < n; k++) {
            if (h[k] == 0)
                throw SolverError("normalize: adjoint reconstruction is zero for item " + std::to_string(k));
            s[k] = {float(1.0 / h[k]), 0.f};
        }
        Dims sd(max_rank, 1);
        sd[dim_batch] = n;
        scale = from_host(sd, s.data());
        DArray ks(kspace.dims, false);
        launch_scale_items(ks.data(), kspace.data(), scale.data(), md_size(kspace.dims) / n, n, false);
        kspace = ks;
    }

    if (o.do_train) {
        DArray reference = cfl_read(o.target_file);
        for (int d : {dim_x, dim_y, dim_batch})
            check_dim_match(o.target_file, reference, o.kspace_file, kspace, d);
        if (o.normalize) {
            DArray r(reference.dims, false);
            launch_scale_items(r.data(), reference.data(), scale.data(), md_size(reference.dims) / n, n, false);
            reference = r;
        }
        TrainConfig tc;
        if (!o.optimizer.empty()) {
            if (o.optimizer == "sgd")
                tc.algo = OptAlgo::Sgd;
            else if (o.optimizer == "adam")
                tc.algo = OptAlgo::Adam;
            else if (o.optimizer == "ipalm")
                tc.algo = OptAlgo::Ipalm;
            else
                throw ConfigError("unknown optimizer: " + o.optimizer);
        } else {
            tc.algo = o.network == "varnet" ? OptAlgo::Ipalm : OptAlgo::Adam;
        }
        tc.lr = o.lr > 0 ? o.lr : (o.network == "varnet" ? 1e-2 : 1e-3);
        if (o.batch_size < 1) // TrainConfig::validate (optim.hpp:44-58)
            throw ConfigError("train: batch size must be >= 1");
        if (o.epochs < 0)
            throw ConfigError("train: epochs must be >= 0");
        if (n < o.batch_size)
            throw ConfigError("train: dataset smaller than one batch (" + std::to_string(n) + " < "
                              + std::to_string(o.batch_size) + ")");
        Model net;
        if (o.network == "varnet") {
            vn.batch = o.batch_size;
            net = build_varnet(vn);
        } else {
            md.batch = o.batch_size;
            md.train_mode = true;
            net = build_modl(md);
        }
        Trainer tr(net, tc, o.seed);
        for (auto& [name, arr] : bundle.arrays) { // warm start (--init)
            DArray v = arr;
            v.dims = tr.all_weights().at(name).dims;
            tr.set_weight(name, v);
        }
        const long nb = o.batch_size;
        for (long epoch = 0; epoch < o.epochs; epoch++) {
            // reproducible shuffle keyed by (seed, epoch) (optim.hpp:256-261)
            std::vector<long> order(static_cast<size_t>(n));
            for (long k = 0; k < n; k++)
                order[size_t(k)] = k;
            Rng rng(hash_rand(o.seed, uint64_t(epoch) + 0x517cc1b7u));
            for (long k = n - 1; k > 0; k--)
                std::swap(order[size_t(k)], order[size_t(rng.below(uint64_t(k + 1)))]);
            double loss_sum = 0;
            long steps = 0;
            for (long pos = 0; pos + nb <= n; pos += nb) { // drop_last
                tr.set_data("kspace", gather_items(kspace, order.data() + pos, nb));
                tr.set_data("coils", gather_items(coils, order.data() + pos, nb));
                tr.set_data("reference", gather_items(reference, order.data() + pos, nb));
                tr.set_data("pattern", pattern);
                loss_sum += tr.step();
                steps++;
            }
            if (o.verbose)
                std::printf("epoch %ld loss %.8g\n", epoch + 1, steps ? loss_sum / double(steps) : 0.0);
        }
        WeightsBundle out;
        out.meta["network"] = o.network;
        out.meta["normalize"] = o.normalize ? "1" : "0";
        out.meta["seed"] = std::to_string(o.seed);
        if (o.network == "varnet") {
            out.meta["iterations"] = std::to_string(vn.iterations);
            out.meta["filters"] = std::to_string(vn.filters);
            out.meta["kernel"] = std::to_string(vn.kernel);
            out.meta["rbf"] = std::to_string(vn.rbf);
        } else {
            out.meta["iterations"] = std::to_string(md.iterations);
            out.meta["layers"] = std::to_string(md.layers);
            out.meta["filters"] = std::to_string(md.filters);
            out.meta["kernel"] = std::to_string(md.kernel);
            out.meta["cg_iter"] = std::to_string(md.cg_iter);
        }
        out.meta["epochs"] = std::to_string(o.epochs);
        for (const auto& [name, arr] : tr.all_weights())
            out.arrays.emplace(name, arr);
        out.save(o.weights_dir);
        sync_and_check();
        return 0;
    }

    // apply: chunked batched inference (cli.hpp:228-262)
    std::map<std::string, DArray> weights;
    for (const auto& [name, arr] : bundle.arrays)
        weights.emplace(name, arr);
    Dims od(max_rank, 1);
    od[dim_x] = kspace.dims[dim_x];
    od[dim_y] = kspace.dims[dim_y];
    od[dim_maps] = maps;
    od[dim_batch] = n;
    DArray output(od, false);
    const long per_out = md_size(od) / n;
    const long chunk = std::min(n, o.batch_size);
    Model net;
    long built = -1;
    for (long pos = 0; pos < n; pos += chunk) {
        const long cnt = std::min(chunk, n - pos);
        if (built != cnt) {
            if (o.network == "varnet") {
                vn.batch = cnt;
                net = build_varnet(vn);
            } else {
                md.batch = cnt;
                md.train_mode = false;
                net = build_modl(md);
            }
            built = cnt;
        }
        std::map<std::string, DArray> dmap;
        dmap["kspace"] = slice_items(kspace, pos, cnt);
        dmap["coils"] = slice_items(coils, pos, cnt);
        dmap["pattern"] = pattern;
        auto outs = net.op.apply(gather_model_inputs(net, weights, dmap));
        DArray res = to_layout(outs[net.output_index("out")], Layout::CANON);
        CUDA_CHECK(cudaMemcpyAsync(output.data() + pos * per_out, res.data(), sizeof(cfloat) * per_out * cnt,
                                   cudaMemcpyDeviceToDevice, ctx().stream));
    }
    if (o.normalize) {
        DArray r(od, false);
        launch_scale_items(r.data(), output.data(), scale.data(), per_out, n, true);
        output = r;
    }
    cfl_write(o.target_file, output);
    sync_and_check();
    return 0;
}

} // namespace mdnn
