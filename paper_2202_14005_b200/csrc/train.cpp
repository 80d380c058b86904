#include "train.h"

#include "kernels.h"

#include <cmath>

namespace mdnn {

Trainer::Trainer(const Model& model, const TrainConfig& cfg, uint64_t seed) : cfg_(cfg)
{
    const int oi = model.output_index("out");
    joint_ = model_chain(model, loss_model_mse(model.op.out_dims(oi)), "prediction", oi);
    loss_idx_ = joint_.output_index("loss");
    long off = 0;
    for (size_t i = 0; i < joint_.args.size(); i++) {
        const Arg& a = joint_.args[i];
        if (a.kind == ArgKind::Data)
            continue;
        auto h = joint_.init_weight(seed, int(i));
        weights_[a.name] = from_host(joint_.op.in_dims(int(i)), h.data());
        if (a.kind == ArgKind::Weights) {
            wargs_.push_back(int(i));
            wnames_.push_back(a.name);
            woff_.push_back(off);
            off += long(h.size());
        }
    }
    flat_n_ = off;
    flat_ = DArray(Dims{std::max(1L, flat_n_)}, true);
    float* v;
    CUDA_CHECK(cudaMalloc(&v, sizeof(float) * std::max(1L, flat_n_)));
    CUDA_CHECK(cudaMemset(v, 0, sizeof(float) * std::max(1L, flat_n_)));
    vbuf_.reset(v, [](float* p) { cudaFree(p); });
    adam_.resize(wargs_.size());
    for (size_t k = 0; k < wargs_.size(); k++) {
        adam_[k].m = DArray(joint_.op.in_dims(wargs_[k]), true);
        adam_[k].v = v + woff_[k];
    }
}

void Trainer::set_data(const std::string& name, DArray a)
{
    int i = joint_.arg_index(name);
    if (joint_.args[i].kind != ArgKind::Data)
        throw ConfigError("trainer: '" + name + "' is not a data argument");
    if (a.dims != joint_.op.in_dims(i))
        throw ShapeError("trainer: data '" + name + "' expected " + dims_to_string(joint_.op.in_dims(i)) + ", got "
                         + dims_to_string(a.dims));
    data_[name] = std::move(a);
}

void Trainer::set_weight(const std::string& name, DArray a)
{
    auto it = weights_.find(name);
    if (it == weights_.end())
        throw ConfigError("trainer: no weight named '" + name + "'");
    if (a.dims != it->second.dims)
        throw ShapeError("trainer: weight '" + name + "' shape mismatch");
    it->second = std::move(a);
}

const DArray& Trainer::weight(const std::string& name) const
{
    auto it = weights_.find(name);
    if (it == weights_.end())
        throw ConfigError("trainer: no weight named '" + name + "'");
    return it->second;
}

DArray Trainer::grad(const std::string& name) const
{
    for (size_t k = 0; k < wnames_.size(); k++)
        if (wnames_[k] == name) {
            Dims d = joint_.op.in_dims(wargs_[k]);
            DArray g(d, false);
            launch_copy(g.data(), flat_.data() + woff_[k], g.size());
            return g;
        }
    throw ConfigError("trainer: no weight named '" + name + "'");
}

std::vector<DArray> Trainer::gather_inputs() const
{
    std::vector<DArray> in;
    for (const auto& a : joint_.args) {
        const auto& src = a.kind == ArgKind::Data ? data_ : weights_;
        auto it = src.find(a.name);
        if (it == src.end())
            throw ConfigError("model: missing array for argument '" + a.name + "'");
        in.push_back(it->second);
    }
    return in;
}

double Trainer::forward_backward()
{
    last_outs_ = joint_.op.apply(gather_inputs());
    std::vector<char> want(joint_.args.size(), 0);
    for (int i : wargs_)
        want[i] = 1;
    DArray one = DArray::scalar(1.f);
    auto grads = joint_.op.adjoint_all(loss_idx_, one, want);
    for (size_t k = 0; k < wargs_.size(); k++) {
        const DArray& g = grads[wargs_[k]];
        launch_copy(flat_.data() + woff_[k], g.data(), g.size());
    }
    launch_check_finite(flat_.data(), flat_n_);
    cfloat lv;
    CUDA_CHECK(cudaMemcpyAsync(&lv, last_outs_[loss_idx_].data(), sizeof(cfloat), cudaMemcpyDeviceToHost,
                               ctx().stream));
    sync_and_check();
    if (!std::isfinite(lv.x))
        throw SolverError("training aborted: non-finite loss");
    return double(lv.x);
}

void Trainer::update(float grad_scale)
{
    // optim.hpp:383-399 per weight: clip, realify, Adam, realify, prox
    for (size_t k = 0; k < wargs_.size(); k++) {
        const Arg& a = joint_.args[wargs_[k]];
        DArray& w = weights_[a.name];
        // weights are immutable values shared with the graph: update a fresh copy
        DArray nw = w.clone();
        float scale = grad_scale;
        cfloat* g = flat_.data() + woff_[k];
        if (cfg_.clip > 0) {
            double nrm = host_znorm(g, w.size()) * grad_scale;
            if (nrm > cfg_.clip)
                scale *= float(cfg_.clip / nrm);
        }
        auto& st = adam_[k];
        st.t++;
        const float c1 = 1.f / float(1.0 - std::pow(cfg_.beta1, double(st.t)));
        const float c2 = 1.f / float(1.0 - std::pow(cfg_.beta2, double(st.t)));
        adam_update(nw.data(), st.m.data(), st.v, g, w.size(), float(cfg_.lr), float(cfg_.beta1),
                    float(cfg_.beta2), float(cfg_.eps), c1, c2, scale, a.real_weights, a.prox == ProxKind::NonNeg);
        w = nw;
    }
    // update_stats: moving-statistics outputs feed their same-named inputs
    for (const auto& a : joint_.args) {
        if (a.kind != ArgKind::MovingStats)
            continue;
        for (size_t o = 0; o < joint_.out_names.size(); o++)
            if (joint_.out_names[o] == a.name) {
                weights_[a.name] = last_outs_[o];
                break;
            }
    }
}

} // namespace mdnn
