#include "train.h"

#include "kernels.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace mdnn {

Trainer::Trainer(const Model& model, const TrainConfig& cfg, uint64_t seed) : cfg_(cfg)
{
    // pre-map the allocator pool (MDNN_POOL_RESERVE_GB overrides; default half
    // of the free device memory, at most 96 GB)
    if (!std::getenv("MDNN_POOL_RESERVE_GB")) {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess)
            reserve_pool(std::min<size_t>(free_b / 2, size_t(96) << 30));
    }
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
    // moving statistics (BN means / variances): the tail of the sync buffer
    for (const auto& a : joint_.args) {
        if (a.kind != ArgKind::MovingStats)
            continue;
        StatSlot s;
        s.name = a.name;
        for (size_t o = 0; o < joint_.out_names.size(); o++)
            if (joint_.out_names[o] == a.name)
                s.out = int(o);
        s.off = flat_n_ + stats_n_;
        s.n = md_size(joint_.op.in_dims(joint_.arg_index(a.name)));
        stats_n_ += s.n;
        stats_.push_back(s);
    }
    flat_ = DArray(Dims{std::max(1L, flat_n_ + stats_n_)}, true);
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

Trainer::~Trainer()
{
    // a staged batch's H2D copy may still be running on the copy stream: order
    // its release (stream-ordered free on the compute stream) after the copy
    auto& c = ctx();
    for (auto& [name, q] : staged_)
        for (auto& s : q) {
            cudaStreamWaitEvent(c.stream, s.ev, 0);
            cudaEventDestroy(s.ev);
        }
    staged_.clear();
    if (comm_)
        cudaStreamSynchronize(comm_->stream());
    if (ev_sync_)
        cudaEventDestroy(ev_sync_);
    if (ev_done_)
        cudaEventDestroy(ev_done_);
}

void Trainer::allreduce_range(long off, long n)
{
    if (!ev_sync_) {
        CUDA_CHECK(cudaEventCreateWithFlags(&ev_sync_, cudaEventDisableTiming));
        CUDA_CHECK(cudaEventCreateWithFlags(&ev_done_, cudaEventDisableTiming));
    }
    // the producers of this range were enqueued on the compute stream
    CUDA_CHECK(cudaEventRecord(ev_sync_, ctx().stream));
    CUDA_CHECK(cudaStreamWaitEvent(comm_->stream(), ev_sync_, 0));
    comm_->allreduce_sum(flat_.fdata() + 2 * off, 2 * n);
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

void Trainer::stage_data(const std::string& name, const HostView& v)
{
    int i = joint_.arg_index(name);
    if (joint_.args[i].kind != ArgKind::Data)
        throw ConfigError("trainer: '" + name + "' is not a data argument");
    if (v.dims != joint_.op.in_dims(i))
        throw ShapeError("trainer: data '" + name + "' expected " + dims_to_string(joint_.op.in_dims(i)) + ", got "
                         + dims_to_string(v.dims));
    cudaEvent_t ev;
    CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    staged_[name].push_back(Staged{import_array_async(v, ev), ev});
}

int Trainer::staged(const std::string& name) const
{
    auto it = staged_.find(name);
    return it == staged_.end() ? 0 : int(it->second.size());
}

void Trainer::take_staged()
{
    auto& c = ctx();
    for (auto& [name, q] : staged_) {
        if (q.empty())
            continue;
        Staged s = std::move(q.front());
        q.pop_front();
        CUDA_CHECK(cudaStreamWaitEvent(c.stream, s.ev, 0));
        CUDA_CHECK(cudaEventDestroy(s.ev));
        data_[name] = std::move(s.a);
    }
}

void Trainer::set_weight(const std::string& name, DArray a)
{
    auto it = weights_.find(name);
    if (it == weights_.end())
        throw ConfigError("trainer: no weight named '" + name + "'");
    if (a.dims != it->second.dims)
        throw ShapeError("trainer: weight '" + name + "' shape mismatch");
    // a caller-provided value of a real-weight argument is only tagged real
    // (known_real in gather_inputs) when it is (weights are small: host check)
    bool real = true;
    for (const auto& v : to_host(a))
        if (v.imag() != 0.f) {
            real = false;
            break;
        }
    not_real_[name] = !real;
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
        // real-valued weights stay real under the realified updates (optim.hpp:382-399)
        if (a.kind != ArgKind::Data && a.real_weights) {
            auto nr = not_real_.find(a.name);
            in.back().known_real = nr == not_real_.end() || !nr->second;
        }
    }
    return in;
}

double Trainer::forward_backward()
{
    static const bool trace = std::getenv("MDNN_TRACE_HOST") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    take_staged();
    last_outs_ = joint_.op.apply(gather_inputs());
    // this shard's new moving statistics -> tail of the sync buffer; with a
    // communicator their all-reduce runs under the whole backward pass
    for (const auto& s : stats_)
        if (s.out >= 0)
            launch_copy(flat_.data() + s.off, last_outs_[s.out].data(), s.n);
    if (comm_ && stats_n_ > 0)
        allreduce_range(flat_n_, stats_n_);
    std::vector<char> want(joint_.args.size(), 0);
    std::vector<int> slot(joint_.args.size(), -1);
    for (size_t k = 0; k < wargs_.size(); k++) {
        want[wargs_[k]] = 1;
        slot[wargs_[k]] = int(k);
    }
    // gradient buckets: a maximal run of consecutive finalised, not yet reduced
    // weights is all-reduced once it holds bucket_min_floats_ (or nothing is
    // left); the sweep's finalisation order is deterministic, so every rank
    // issues the same collectives in the same order
    const int nw = int(wargs_.size());
    std::vector<char> fin(nw, 0), sent(nw, 0);
    int n_fin = 0;
    auto flush = [&](bool all) {
        for (int k = 0; k < nw;) {
            if (!fin[k] || sent[k]) {
                k++;
                continue;
            }
            int e = k;
            long n = 0;
            while (e < nw && fin[e] && !sent[e])
                n += md_size(joint_.op.in_dims(wargs_[e++]));
            if (all || 2 * n >= bucket_min_floats_) {
                allreduce_range(woff_[k], n);
                for (int q = k; q < e; q++)
                    sent[q] = 1;
            }
            k = e;
        }
    };
    DArray one = DArray::scalar(1.f);
    joint_.op.adjoint_all(loss_idx_, one, want, [&](int i, const DArray& g) {
        const int k = slot[i];
        if (k < 0)
            return;
        launch_copy(flat_.data() + woff_[k], g.data(), g.size());
        fin[k] = 1;
        if (comm_)
            flush(++n_fin == nw);
    });
    if (comm_) {
        CUDA_CHECK(cudaEventRecord(ev_done_, comm_->stream()));
        CUDA_CHECK(cudaStreamWaitEvent(ctx().stream, ev_done_, 0));
    }
    launch_check_finite(flat_.data(), flat_n_);
    cfloat lv;
    CUDA_CHECK(cudaMemcpyAsync(&lv, last_outs_[loss_idx_].data(), sizeof(cfloat), cudaMemcpyDeviceToHost,
                               ctx().stream));
    const auto t1 = std::chrono::steady_clock::now();
    sync_and_check();
    if (trace) {
        const auto t2 = std::chrono::steady_clock::now();
        cudaMemPool_t pool;
        uint64_t res = 0, used = 0, hi = 0;
        cudaDeviceGetDefaultMemPool(&pool, ctx().device);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &hi);
        std::fprintf(stderr, "[mdnn] forward_backward host enqueue %.2f ms, wait %.2f ms; pool reserved %.2f GB "
                     "(high %.2f) used %.2f GB\n",
                     std::chrono::duration<double, std::milli>(t1 - t0).count(),
                     std::chrono::duration<double, std::milli>(t2 - t1).count(), res / 1e9, hi / 1e9, used / 1e9);
    }
    if (!std::isfinite(lv.x))
        throw SolverError("training aborted: non-finite loss");
    return double(lv.x);
}

void Trainer::update(float grad_scale)
{
    if (cfg_.algo == OptAlgo::Ipalm)
        throw ConfigError("trainer: ipalm updates per block inside step(); use mdnn_trainer_step");
    // optim.hpp:383-399 per weight: clip, realify, Adam / SGD, realify, prox
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
        if (cfg_.algo == OptAlgo::Sgd) {
            // sgd_step (optim.hpp:66-71) on the clipped, realified gradient, then realify / prox
            sgd_update(nw.data(), g, w.size(), float(cfg_.lr), scale, a.real_weights, a.prox == ProxKind::NonNeg);
            w = nw;
            continue;
        }
        auto& st = adam_[k];
        st.t++;
        const float c1 = 1.f / float(1.0 - std::pow(cfg_.beta1, double(st.t)));
        const float c2 = 1.f / float(1.0 - std::pow(cfg_.beta2, double(st.t)));
        adam_update(nw.data(), st.m.data(), st.v, g, w.size(), float(cfg_.lr), float(cfg_.beta1),
                    float(cfg_.beta2), float(cfg_.eps), c1, c2, scale, a.real_weights, a.prox == ProxKind::NonNeg);
        w = nw;
    }
    update_stats(last_outs_);
}

void Trainer::update_dp(int world)
{
    if (world < 1)
        throw ConfigError("trainer: world size " + std::to_string(world));
    update(1.f / float(world));
    // replica mean of the moving statistics (summed in the sync buffer)
    for (const auto& s : stats_) {
        DArray v(joint_.op.in_dims(joint_.arg_index(s.name)), false);
        launch_scale(v.data(), flat_.data() + s.off, cfloat{1.f / float(world), 0.f}, s.n);
        weights_[s.name] = v;
    }
}

// update_stats: moving-statistics outputs feed their same-named inputs (optim.hpp:403-415)
void Trainer::update_stats(const std::vector<DArray>& outs)
{
    for (const auto& a : joint_.args) {
        if (a.kind != ArgKind::MovingStats)
            continue;
        for (size_t o = 0; o < joint_.out_names.size(); o++)
            if (joint_.out_names[o] == a.name) {
                weights_[a.name] = outs[o];
                break;
            }
    }
}

// clip_gradient (optim.hpp:201-208) and realify, in place
void Trainer::finish_grad(DArray& g, const Arg& a, float grad_scale) const
{
    if (cfg_.clip > 0) {
        const double nrm = host_znorm(g.data(), g.size());
        if (nrm > cfg_.clip)
            launch_scale(g.data(), g.data(), cfloat{float(cfg_.clip / nrm), 0.f}, g.size());
    }
    if (grad_scale != 1.f)
        launch_scale(g.data(), g.data(), cfloat{grad_scale, 0.f}, g.size());
    if (a.real_weights)
        launch_real(g.data(), g.data(), g.size());
}

double Trainer::ipalm_step()
{
    const int nb = int(wargs_.size());
    if (ipalm_prev_.size() != size_t(nb))
        ipalm_prev_.resize(nb);
    const float lr = float(cfg_.lr), al = float(cfg_.ipalm_alpha), be = float(cfg_.ipalm_beta);
    // cur: the iterate the gradient oracle sees (blocks < j updated, j at z, > j old)
    take_staged();
    std::vector<DArray> in = gather_inputs();
    double loss = 0;
    for (int j = 0; j < nb; j++) {
        const Arg& a = joint_.args[wargs_[j]];
        DArray& theta = weights_[a.name];
        if (!ipalm_prev_[j].valid())
            ipalm_prev_[j] = theta.clone();
        const long n = theta.size();
        DArray d(theta.dims, false), y(theta.dims, false), z(theta.dims, false);
        launch_add(d.data(), theta.data(), ipalm_prev_[j].data(), -1.f, n); // theta - prev
        launch_add(y.data(), theta.data(), d.data(), al, n);                // prox extrapolation
        launch_add(z.data(), theta.data(), d.data(), be, n);                // gradient extrapolation
        in[wargs_[j]] = z;
        auto outs = joint_.op.apply(in);
        cfloat lv;
        CUDA_CHECK(cudaMemcpyAsync(&lv, outs[loss_idx_].data(), sizeof(cfloat), cudaMemcpyDeviceToHost,
                                   ctx().stream));
        sync_and_check();
        loss = double(lv.x);
        if (!std::isfinite(loss))
            throw SolverError("training aborted: non-finite loss");
        DArray g = joint_.op.adjoint_derivative(loss_idx_, wargs_[j], DArray::scalar(1.f)).clone();
        launch_check_finite(g.data(), n); // check_gradient_finite (optim.hpp:143)
        finish_grad(g, a, 1.f);
        launch_add(y.data(), y.data(), g.data(), -lr, n);
        if (a.prox == ProxKind::NonNeg)
            launch_prox_nonneg(y.data(), n);
        ipalm_prev_[j] = theta;
        theta = y;
        in[wargs_[j]] = y;
        // the flat buffer mirrors the last block gradients (inspection / tests)
        launch_copy(flat_.data() + woff_[j], g.data(), n);
    }
    bool has_stats = false;
    for (const auto& a : joint_.args)
        has_stats |= a.kind == ArgKind::MovingStats;
    if (has_stats)
        update_stats(joint_.op.apply(gather_inputs()));
    sync_and_check();
    return loss;
}

} // namespace mdnn
