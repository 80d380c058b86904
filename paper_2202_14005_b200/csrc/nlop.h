// Nlop graph engine over device arrays.
//
// Mirrors the reference's NlopNode / Nlop (nlop.hpp:18-437): a flattened DAG
// of atomic nodes, Kahn topological order (smallest index first), forward
// sweep storing derivative state, tangent sweep with fan-in accumulation,
// reverse sweep with fan-out accumulation, generation-counter staleness and
// the combine / link / duplicate / chain algebra.  Differences by design:
//   * values are immutable device arrays shared by reference (no clones);
//   * adjoint_all takes a `wanted` mask and prunes every node whose
//     cotangent cannot reach a wanted input (training asks for weights only);
//   * each node may request a storage layout per port (core.h Layout); the
//     engine converts on edges whose producer and consumer layouts differ.
#pragma once

#include "core.h"

#include <functional>
#include <memory>
#include <string>
#include <vector>

namespace mdnn {

class Node {
public:
    Node(std::string name, std::vector<Dims> in, std::vector<Dims> out)
        : name_(std::move(name)), ins_(std::move(in)), outs_(std::move(out))
    {
    }
    virtual ~Node() = default;

    const std::string& name() const { return name_; }
    int n_in() const { return int(ins_.size()); }
    int n_out() const { return int(outs_.size()); }
    const Dims& in_dims(int i) const { return ins_.at(i); }
    const Dims& out_dims(int o) const { return outs_.at(o); }

    // Compute outputs (out is resized to n_out by the caller) and refresh the
    // evaluation state.
    virtual void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool store) = 0;
    // dy = D_i F_o dx
    virtual DArray deriv(int o, int i, const DArray& dx) = 0;
    // dx = (D_i F_o)^H dy
    virtual DArray adjoint(int o, int i, const DArray& dy) = 0;
    virtual bool zero_deriv(int o, int i) const
    {
        (void)o;
        (void)i;
        return false;
    }
    virtual bool holomorphic() const { return false; }
    // cotangent of output o to every wanted input (containers override)
    virtual void adjoint_all(int o, const DArray& dy, std::vector<DArray>& dx, const std::vector<char>& want);
    // storage layout the node wants for input i / produces on output o (the
    // engine hands cotangents of output o to adjoint_all in out_layout(o))
    virtual Layout in_layout(int i) const
    {
        (void)i;
        return Layout::CANON;
    }
    virtual Layout out_layout(int o) const
    {
        (void)o;
        return Layout::CANON;
    }

    uint64_t generation() const { return gen_; }

    // Producer-side hint for the cotangent of output o: state of this node
    // that the kernel computing that cotangent may fold work for (the
    // batch-norm block's backward reduction into the convolution that
    // produces its output cotangent); nullptr = none.
    virtual const void* cotangent_hint(int o) const
    {
        (void)o;
        return nullptr;
    }
    // set by the engine around adjoint calls: the producers' hints per input
    void set_input_hints(std::vector<const void*> h) { in_hints_ = std::move(h); }

protected:
    void bump_generation() { ++gen_; }
    void require_forward() const;
    const void* input_hint(int i) const { return size_t(i) < in_hints_.size() ? in_hints_[size_t(i)] : nullptr; }

    std::string name_;
    std::vector<Dims> ins_, outs_;

private:
    uint64_t gen_ = 0;
    std::vector<const void*> in_hints_;
};

using NodePtr = std::shared_ptr<Node>;

class Nlop {
public:
    struct Src {
        int node; // -1: graph input slot `port`
        int port;
        bool operator==(const Src& o) const { return node == o.node && port == o.port; }
    };

    Nlop() = default;
    explicit Nlop(NodePtr node);

    bool valid() const { return !nodes_.empty(); }
    int n_in() const { return n_in_; }
    int n_out() const { return int(outputs_.size()); }
    const Dims& in_dims(int i) const { return in_dims_.at(i); }
    const Dims& out_dims(int o) const;

    std::vector<DArray> apply(const std::vector<DArray>& in);
    // forward sweep without the derivative bookkeeping (containers: store =
    // false evaluates without retaining state, nlop.hpp:363-386)
    std::vector<DArray> run_forward(const std::vector<DArray>& in, bool store);
    DArray derivative(int o, int i, const DArray& dx);
    // on_final(i, g): called during the reverse sweep as soon as wanted input
    // i's cotangent g is complete (its last consumer has been processed), in
    // the order the sweep finalises them -- lets a trainer start the gradient
    // all-reduce of early buckets under the rest of the backward pass
    using FinalFn = std::function<void(int, const DArray&)>;
    std::vector<DArray> adjoint_all(int o, const DArray& dy, const std::vector<char>& want = {},
                                    const FinalFn& on_final = nullptr);
    DArray adjoint_derivative(int o, int i, const DArray& dy);

    const std::vector<NodePtr>& nodes() const { return nodes_; }

    friend Nlop combine(const Nlop& f, const Nlop& g);
    friend Nlop link(const Nlop& h, int o, int i);
    friend Nlop duplicate(const Nlop& h, int i, int j);
    friend Nlop chain(const Nlop& f, const Nlop& g);

private:
    void check_state() const;
    void finalize();

    std::vector<NodePtr> nodes_;
    std::vector<std::vector<Src>> in_srcs_;
    std::vector<Src> outputs_;
    std::vector<Dims> in_dims_;
    int n_in_ = 0;

    std::vector<uint64_t> last_gens_;
    std::vector<int> topo_;
    bool has_forward_ = false;
};

Nlop combine(const Nlop& f, const Nlop& g);
Nlop link(const Nlop& h, int o, int i);
Nlop duplicate(const Nlop& h, int i, int j);
Nlop chain(const Nlop& f, const Nlop& g);

// sum of two cotangents (reuses a uniquely owned buffer when possible)
DArray accumulate(DArray acc, const DArray& add);

} // namespace mdnn
