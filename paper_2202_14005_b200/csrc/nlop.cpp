#include "nlop.h"

#include "kernels.h"

#include <algorithm>

namespace mdnn {

void Node::require_forward() const
{
    if (gen_ == 0)
        throw StaleDerivativeError(name_ + ": derivative requested before any forward call");
}

void Node::adjoint_all(int o, const DArray& dy, std::vector<DArray>& dx, const std::vector<char>& want)
{
    dx.assign(n_in(), DArray{});
    for (int i = 0; i < n_in(); i++) {
        if (!want[i] || zero_deriv(o, i))
            continue;
        dx[i] = adjoint(o, i, dy);
    }
}

DArray accumulate(DArray acc, const DArray& add)
{
    if (!acc.valid())
        return add;
    DArray b = add.layout == acc.layout ? add : to_layout(add, acc.layout);
    if (acc.buf.use_count() == 1) {
        launch_axpy(acc.data(), cfloat{1.f, 0.f}, b.data(), acc.size());
        acc.drop_chstats(); // producer statistics no longer describe the values
        acc.known_real = acc.known_real && b.known_real;
        return acc;
    }
    DArray out(acc.dims, false, acc.layout);
    launch_add(out.data(), acc.data(), b.data(), 1.f, acc.size());
    out.known_real = acc.known_real && b.known_real;
    return out;
}

Nlop::Nlop(NodePtr node)
{
    nodes_.push_back(node);
    in_srcs_.push_back({});
    n_in_ = node->n_in();
    for (int i = 0; i < n_in_; i++) {
        in_srcs_[0].push_back({-1, i});
        in_dims_.push_back(node->in_dims(i));
    }
    for (int o = 0; o < node->n_out(); o++)
        outputs_.push_back({0, o});
    finalize();
}

const Dims& Nlop::out_dims(int o) const
{
    auto s = outputs_.at(o);
    return nodes_[s.node]->out_dims(s.port);
}

static DArray as_layout(const DArray& a, Layout l) { return a.layout == l ? a : to_layout(a, l); }

std::vector<DArray> Nlop::apply(const std::vector<DArray>& in)
{
    if (long(in.size()) != n_in_)
        throw ShapeError("nlop apply: expected " + std::to_string(n_in_) + " inputs, got "
                         + std::to_string(in.size()));
    for (int i = 0; i < n_in_; i++) {
        if (!in[i].valid())
            throw ShapeError("nlop apply: input " + std::to_string(i) + " is uninitialized");
        if (in[i].dims != in_dims_[i])
            throw ShapeError("nlop apply: input " + std::to_string(i) + " expected " + dims_to_string(in_dims_[i])
                             + ", got " + dims_to_string(in[i].dims));
    }
    auto out = run_forward(in, true);
    last_gens_.resize(nodes_.size());
    for (size_t n = 0; n < nodes_.size(); n++)
        last_gens_[n] = nodes_[n]->generation();
    has_forward_ = true;
    return out;
}

std::vector<DArray> Nlop::run_forward(const std::vector<DArray>& in, bool store)
{
    std::vector<std::vector<DArray>> vals(nodes_.size());
    std::vector<DArray> args;
    for (int ni : topo_) {
        auto& node = *nodes_[ni];
        args.clear();
        for (int k = 0; k < node.n_in(); k++) {
            auto s = in_srcs_[ni][k];
            const DArray& v = s.node < 0 ? in[s.port] : vals[s.node][s.port];
            args.push_back(as_layout(v, node.in_layout(k)));
        }
        std::vector<DArray> outs(node.n_out());
        node.forward(args, outs, store);
        vals[ni] = std::move(outs);
        // release values no longer needed by later consumers is left to refcounts
    }
    std::vector<DArray> out;
    for (auto s : outputs_)
        out.push_back(as_layout(vals[s.node][s.port], Layout::CANON));
    return out;
}

void Nlop::check_state() const
{
    if (!has_forward_)
        throw StaleDerivativeError("nlop derivative requested before any forward call");
    for (size_t n = 0; n < nodes_.size(); n++)
        if (nodes_[n]->generation() != last_gens_[n])
            throw StaleDerivativeError("nlop derivative state is stale: '" + nodes_[n]->name()
                                       + "' was re-applied after this operator's forward pass");
}

DArray Nlop::derivative(int o, int i, const DArray& dx)
{
    check_state();
    if (dx.dims != in_dims(i))
        throw ShapeError("nlop derivative: probe shape mismatch");
    std::vector<std::vector<DArray>> tan(nodes_.size());
    for (size_t n = 0; n < nodes_.size(); n++)
        tan[n].resize(nodes_[n]->n_out());
    for (int ni : topo_) {
        auto& node = *nodes_[ni];
        for (int p = 0; p < node.n_out(); p++) {
            DArray acc;
            for (int k = 0; k < node.n_in(); k++) {
                auto s = in_srcs_[ni][k];
                const DArray* t = nullptr;
                if (s.node < 0) {
                    if (s.port != i)
                        continue;
                    t = &dx;
                } else {
                    if (!tan[s.node][s.port].valid())
                        continue;
                    t = &tan[s.node][s.port];
                }
                if (node.zero_deriv(p, k))
                    continue;
                DArray dy = node.deriv(p, k, as_layout(*t, node.in_layout(k)));
                acc = accumulate(std::move(acc), dy);
            }
            if (acc.valid())
                tan[ni][p] = std::move(acc);
        }
    }
    auto s = outputs_.at(o);
    if (tan[s.node][s.port].valid())
        return as_layout(tan[s.node][s.port], Layout::CANON);
    return DArray(out_dims(o)); // structurally zero
}

std::vector<DArray> Nlop::adjoint_all(int o, const DArray& dy, const std::vector<char>& want_in,
                                      const FinalFn& on_final)
{
    check_state();
    if (dy.dims != out_dims(o))
        throw ShapeError("nlop adjoint: probe shape mismatch");
    std::vector<char> want = want_in.empty() ? std::vector<char>(n_in_, 1) : want_in;

    // needs[n]: some input of node n transitively reaches a wanted graph input
    std::vector<char> needs(nodes_.size(), 0);
    for (int ni : topo_) {
        for (auto s : in_srcs_[ni])
            if ((s.node < 0 && want[s.port]) || (s.node >= 0 && needs[s.node]))
                needs[ni] = 1;
    }

    std::vector<std::vector<DArray>> cot(nodes_.size());
    for (size_t n = 0; n < nodes_.size(); n++)
        cot[n].resize(nodes_[n]->n_out());
    std::vector<DArray> in_cot(n_in_);
    auto os = outputs_.at(o);
    cot[os.node][os.port] = dy;

    // last_use[i]: position in the reverse sweep after which no node adds to
    // input i's cotangent (-1: no needed node consumes it)
    std::vector<int> last_use(n_in_, -1);
    {
        int pos = 0;
        for (auto it = topo_.rbegin(); it != topo_.rend(); ++it, ++pos)
            if (needs[*it])
                for (auto s : in_srcs_[*it])
                    if (s.node < 0)
                        last_use[s.port] = pos;
    }
    auto finish = [&](int i) {
        if (!in_cot[i].valid())
            in_cot[i] = DArray(in_dims_[i]);
        else
            in_cot[i] = as_layout(in_cot[i], Layout::CANON);
        if (on_final)
            on_final(i, in_cot[i]);
    };
    for (int i = 0; i < n_in_; i++)
        if (want[i] && last_use[i] < 0)
            finish(i);

    std::vector<DArray> contrib;
    std::vector<char> wk;
    std::vector<const void*> hints;
    int pos = -1;
    for (auto it = topo_.rbegin(); it != topo_.rend(); ++it) {
        int ni = *it;
        ++pos;
        if (!needs[ni])
            continue;
        auto& node = *nodes_[ni];
        wk.assign(node.n_in(), 0);
        for (int k = 0; k < node.n_in(); k++) {
            auto s = in_srcs_[ni][k];
            wk[k] = s.node < 0 ? want[s.port] : needs[s.node];
        }
        for (int p = 0; p < node.n_out(); p++) {
            if (!cot[ni][p].valid())
                continue;
            DArray g = as_layout(std::move(cot[ni][p]), node.out_layout(p));
            // producers' hints for the cotangents this node is about to emit
            hints.assign(node.n_in(), nullptr);
            for (int k = 0; k < node.n_in(); k++) {
                auto s = in_srcs_[ni][k];
                if (s.node >= 0)
                    hints[k] = nodes_[s.node]->cotangent_hint(s.port);
            }
            node.set_input_hints(hints);
            node.adjoint_all(p, g, contrib, wk);
            node.set_input_hints({});
            for (int k = 0; k < node.n_in(); k++) {
                if (k >= int(contrib.size()) || !contrib[k].valid())
                    continue;
                auto s = in_srcs_[ni][k];
                DArray& dst = (s.node < 0) ? in_cot[s.port] : cot[s.node][s.port];
                dst = accumulate(std::move(dst), contrib[k]);
            }
            contrib.clear();
        }
        for (auto s : in_srcs_[ni])
            if (s.node < 0 && want[s.port] && last_use[s.port] == pos) {
                last_use[s.port] = -2; // a node may read the same input twice
                finish(s.port);
            }
    }
    return in_cot;
}

DArray Nlop::adjoint_derivative(int o, int i, const DArray& dy)
{
    std::vector<char> want(n_in_, 0);
    want.at(i) = 1;
    return adjoint_all(o, dy, want)[i];
}

Nlop combine(const Nlop& f, const Nlop& g)
{
    Nlop h;
    h.nodes_ = f.nodes_;
    h.in_srcs_ = f.in_srcs_;
    h.n_in_ = f.n_in_ + g.n_in_;
    h.in_dims_ = f.in_dims_;
    h.in_dims_.insert(h.in_dims_.end(), g.in_dims_.begin(), g.in_dims_.end());
    h.outputs_ = f.outputs_;
    const int nshift = int(f.nodes_.size());
    for (size_t n = 0; n < g.nodes_.size(); n++) {
        h.nodes_.push_back(g.nodes_[n]);
        auto srcs = g.in_srcs_[n];
        for (auto& s : srcs) {
            if (s.node < 0)
                s.port += f.n_in_;
            else
                s.node += nshift;
        }
        h.in_srcs_.push_back(std::move(srcs));
    }
    for (auto s : g.outputs_)
        h.outputs_.push_back({s.node + nshift, s.port});
    h.finalize();
    return h;
}

Nlop link(const Nlop& h, int o, int i)
{
    if (o < 0 || o >= h.n_out() || i < 0 || i >= h.n_in())
        throw ShapeError("link: index out of range");
    if (h.out_dims(o) != h.in_dims(i))
        throw ShapeError("link: output " + dims_to_string(h.out_dims(o)) + " does not match input "
                         + dims_to_string(h.in_dims(i)));
    Nlop r = h;
    auto src = h.outputs_[o];
    for (auto& srcs : r.in_srcs_)
        for (auto& s : srcs) {
            if (s.node < 0 && s.port == i)
                s = src;
            else if (s.node < 0 && s.port > i)
                s.port--;
        }
    r.outputs_.erase(r.outputs_.begin() + o);
    r.in_dims_.erase(r.in_dims_.begin() + i);
    r.n_in_--;
    r.finalize();
    return r;
}

Nlop duplicate(const Nlop& h, int i, int j)
{
    if (i < 0 || j < 0 || i >= h.n_in() || j >= h.n_in() || i == j)
        throw ShapeError("duplicate: index out of range");
    if (h.in_dims(i) != h.in_dims(j))
        throw ShapeError("duplicate: input shapes differ");
    Nlop r = h;
    for (auto& srcs : r.in_srcs_)
        for (auto& s : srcs) {
            if (s.node < 0 && s.port == j)
                s.port = i < j ? i : i - 1;
            else if (s.node < 0 && s.port > j)
                s.port--;
        }
    r.in_dims_.erase(r.in_dims_.begin() + j);
    r.n_in_--;
    r.finalize();
    return r;
}

Nlop chain(const Nlop& f, const Nlop& g)
{
    if (f.n_out() != 1)
        throw ShapeError("chain: first operator must have a single output");
    if (g.n_in() != 1)
        throw ShapeError("chain: second operator must have a single input");
    return link(combine(f, g), 0, f.n_in());
}

void Nlop::finalize()
{
    for (size_t n = 0; n < nodes_.size(); n++) {
        if (int(in_srcs_[n].size()) != nodes_[n]->n_in())
            throw ShapeError("nlop wiring: port count mismatch");
        for (int k = 0; k < nodes_[n]->n_in(); k++) {
            auto s = in_srcs_[n][k];
            const Dims& have = s.node < 0 ? in_dims_.at(s.port) : nodes_.at(s.node)->out_dims(s.port);
            if (have != nodes_[n]->in_dims(k))
                throw ShapeError("nlop wiring: shape mismatch into '" + nodes_[n]->name() + "'");
        }
    }
    // Kahn, smallest index first (nlop.hpp:410-415)
    std::vector<int> indeg(nodes_.size(), 0);
    std::vector<std::vector<int>> consumers(nodes_.size());
    for (size_t n = 0; n < nodes_.size(); n++)
        for (auto s : in_srcs_[n])
            if (s.node >= 0) {
                indeg[n]++;
                consumers[s.node].push_back(int(n));
            }
    topo_.clear();
    std::vector<int> ready;
    for (size_t n = 0; n < nodes_.size(); n++)
        if (indeg[n] == 0)
            ready.push_back(int(n));
    while (!ready.empty()) {
        auto it = std::min_element(ready.begin(), ready.end());
        int n = *it;
        ready.erase(it);
        topo_.push_back(n);
        for (int m : consumers[n])
            if (--indeg[m] == 0)
                ready.push_back(m);
    }
    if (topo_.size() != nodes_.size())
        throw ShapeError("nlop wiring: graph contains a cycle");
    has_forward_ = false;
}

} // namespace mdnn
