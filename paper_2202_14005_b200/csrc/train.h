// Training step (optim.hpp:218-415): joint model + MSE loss, forward, reverse
// sweep restricted to the weights, flat fp32 gradient buffer (the all-reduce
// payload for data parallelism), complex Adam, realify / prox, and the
// moving-statistics carry-over (update_stats, optim.hpp:403-415).
#pragma once

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
    double step()
    {
        if (cfg_.algo == OptAlgo::Ipalm)
            return ipalm_step();
        double l = forward_backward();
        update(1.f);
        return l;
    }
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
    DArray flat_;
    long flat_n_ = 0;
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
