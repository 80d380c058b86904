// Training step (optim.hpp:218-415): joint model + MSE loss, forward, reverse
// sweep restricted to the weights, flat fp32 gradient buffer (the all-reduce
// payload for data parallelism), complex Adam, realify / prox, and the
// moving-statistics carry-over (update_stats, optim.hpp:403-415).
#pragma once

#include "comm.h"
#include "model.h"

#include <deque>

namespace mdnn {

// OptAlgo (optim.hpp:10) and the TrainConfig fields the step uses (optim.hpp:20-56)
enum class OptAlgo { Sgd = 0, Adam = 1, Ipalm = 2 };
struct TrainConfig {
    double lr = 1e-3, beta1 = 0.9, beta2 = 0.999, eps = 1e-8, clip = 0;
    OptAlgo algo = OptAlgo::Adam;
    double ipalm_alpha = 0.5, ipalm_beta = 0.5;
};

class Trainer {
public:
    Trainer(const Model& model, const TrainConfig& cfg, uint64_t seed);
    ~Trainer(); // drains staged batches (their H2D copies) before the buffers go back to the pool

    void set_data(const std::string& name, DArray a);
    // prefetch: queue a host batch for `name`, copied asynchronously on the
    // copy stream; each forward pass takes the oldest queued batch of every
    // name (the host buffer must stay valid until that pass has been issued)
    void stage_data(const std::string& name, const HostView& v);
    int staged(const std::string& name) const;
    void set_weight(const std::string& name, DArray a);
    const DArray& weight(const std::string& name) const;
    DArray grad(const std::string& name) const;

    double forward_backward();           // returns loss (synchronises once)
    void update(float grad_scale);       // Adam on the flat buffer
    // data parallel: the sync buffer after forward_backward holds this shard's
    // gradients and new moving statistics; after it has been summed over `world`
    // replicas, update_dp applies Adam to gradient / world and sets every moving
    // statistic to the replica mean, so replicas stay bitwise identical
    void update_dp(int world);
    double step()
    {
        if (cfg_.algo == OptAlgo::Ipalm)
            return ipalm_step();
        double l = forward_backward();
        if (comm_)
            update_dp(comm_->nranks());
        else
            update(1.f);
        return l;
    }
    // attach an NCCL communicator: forward_backward then all-reduces the sync
    // buffer in buckets on the comm stream while the reverse sweep runs
    void set_comm(std::unique_ptr<Comm> c) { comm_ = std::move(c); }
    const Comm* comm() const { return comm_.get(); }
    float* sync_buffer() const { return flat_.fdata(); }
    long sync_floats() const { return 2 * (flat_n_ + stats_n_); }
    // one iPALM sweep over the weight blocks in Gauss-Seidel order
    // (ipalm_step + run_step's iPALM branch, optim.hpp:118-153, 331-370)
    double ipalm_step();
    float* grad_buffer() const { return flat_.fdata(); }
    long grad_floats() const { return 2 * flat_n_; }
    const std::vector<std::string>& weight_names() const { return wnames_; }
    // every non-data argument (trainable weights and moving statistics), by name
    const std::map<std::string, DArray>& all_weights() const { return weights_; }
    int kernel_launch_estimate() const { return 0; }

private:
    std::vector<DArray> gather_inputs() const;
    void take_staged(); // commit the oldest staged batch of every name (stream wait, no host sync)
    struct Staged {
        DArray a;
        cudaEvent_t ev;
    };
    std::map<std::string, std::deque<Staged>> staged_;

    Model joint_;
    TrainConfig cfg_;
    int loss_idx_ = 0;
    std::map<std::string, DArray> weights_, data_;
    std::map<std::string, bool> not_real_; // set_weight values of real-weight args with imaginary parts
    std::vector<int> wargs_;
    std::vector<std::string> wnames_;
    std::vector<long> woff_;
    // flat sync buffer: [weight gradients (flat_n_ complex) | moving statistics (stats_n_ complex)]
    DArray flat_;
    long flat_n_ = 0;
    struct StatSlot {
        std::string name;
        int out = -1; // joint output carrying the new value
        long off = 0, n = 0;
    };
    std::vector<StatSlot> stats_;
    long stats_n_ = 0;
    std::unique_ptr<Comm> comm_;
    cudaEvent_t ev_sync_ = nullptr; // compute -> comm stream hand-offs
    cudaEvent_t ev_done_ = nullptr; // comm -> compute stream (all buckets reduced)
    long bucket_min_floats_ = 1 << 16;
    void allreduce_range(long off, long n); // complex offsets into flat_
    struct Adam {
        DArray m;
        float* v = nullptr;
        long t = 0;
    };
    std::vector<Adam> adam_;
    std::vector<DArray> ipalm_prev_; // IpalmState::prev per weight block
    void update_stats(const std::vector<DArray>& outs);
    void finish_grad(DArray& g, const Arg& a, float grad_scale) const; // clip + realify
    std::shared_ptr<float> vbuf_;
    std::vector<DArray> last_outs_;
};

} // namespace mdnn
