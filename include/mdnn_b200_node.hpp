// mdnn_b200_node.hpp — reference-side adapter over the C ABI (include/mdnn.h).
//
// A maintainer of the reference (/root/reference/proj/include/mdnn) adds this
// header to splice B200 operators into reference graphs unchanged: B200Node is
// an NlopNode<float> (nlop.hpp:18-83) whose forward / deriv / adjoint /
// adjoint_all forward to mdnn_nlop_apply / _derivative / _adjoint /
// _adjoint_all (mdnn.h:104-111) on host buffers (the library stages H2D / D2H).
// Reference exceptions are re-raised from the MDNN_ERR_* codes
// (common.hpp:15-26).  Compiled and exercised by tests/adapter/splice_main.cpp
// (built by oracle/Makefile, run by tests/test_gpu_adapter.py).
//
//   auto s = mdnn::Nlop<float>(std::make_shared<mdnn::B200Node>(
//                mdnn_model_nlop(mdnn_modl_normal_plus_lambda(&sd))));
//   auto inv = mdnn::make_inverse_nlop<float>(s, 10, 1e-7);   // reference CG over the B200 S
#pragma once

#include <mdnn/nlop.hpp>

#include <complex>
#include <span>
#include <string>
#include <vector>

#include "mdnn.h"

namespace mdnn {

inline mdnn_array b200_view(const MdArray<float>& a)
{
    mdnn_array v{};
    v.data = reinterpret_cast<float*>(const_cast<std::complex<float>*>(a.data()));
    v.rank = a.rank();
    v.device = -1; // host buffers
    for (int d = 0; d < a.rank(); d++) {
        v.dims[d] = a.dims()[d];
        v.strides[d] = a.strides()[d];
    }
    v.has_strides = 1;
    return v;
}

inline void b200_check(int rc)
{
    if (rc == MDNN_OK)
        return;
    const std::string m = mdnn_last_error();
    switch (rc) {
    case MDNN_ERR_SHAPE: throw ShapeError(m);
    case MDNN_ERR_IO: throw IoError(m);
    case MDNN_ERR_CONFIG: throw ConfigError(m);
    case MDNN_ERR_SOLVER: throw SolverError(m);
    case MDNN_ERR_BOUNDS: throw BoundsError(m);
    case MDNN_ERR_ALIAS: throw AliasError(m);
    case MDNN_ERR_STALE: throw StaleDerivativeError(m);
    default: throw Error(m);
    }
}

class B200Node : public NlopNode<float> {
public:
    // takes ownership of the handle
    explicit B200Node(mdnn_nlop* h, std::string name = "b200") : h_(h), name_(std::move(name))
    {
        if (!h_)
            throw Error(std::string("b200: null operator handle: ") + mdnn_last_error());
        for (int i = 0; i < mdnn_nlop_n_in(h_); i++)
            ins_.push_back(query(i, false));
        for (int o = 0; o < mdnn_nlop_n_out(h_); o++)
            outs_.push_back(query(o, true));
    }
    ~B200Node() override { mdnn_nlop_free(h_); }
    B200Node(const B200Node&) = delete;
    B200Node& operator=(const B200Node&) = delete;

    std::string name() const override { return name_; }
    int n_in() const override { return int(ins_.size()); }
    int n_out() const override { return int(outs_.size()); }
    const Dims& in_dims(int i) const override { return ins_.at(i); }
    const Dims& out_dims(int o) const override { return outs_.at(o); }
    bool holomorphic() const override { return false; } // adjoint is the real-Jacobian transpose either way

    void forward(std::span<const MdArray<float>> in, std::span<MdArray<float>> out, bool) override
    {
        std::vector<mdnn_array> a, b;
        for (const auto& x : in)
            a.push_back(b200_view(x));
        for (auto& y : out) {
            if (!y.valid())
                y = MdArray<float>(outs_[b.size()]);
            b.push_back(b200_view(y));
        }
        b200_check(mdnn_nlop_apply(h_, int(a.size()), a.data(), int(b.size()), b.data()));
        bump_generation();
    }
    void deriv(int o, int i, const MdArray<float>& dx, MdArray<float>& dy) override
    {
        require_forward();
        auto a = b200_view(dx), b = b200_view(dy);
        b200_check(mdnn_nlop_derivative(h_, o, i, &a, &b));
    }
    void adjoint(int o, int i, const MdArray<float>& dy, MdArray<float>& dx) override
    {
        require_forward();
        auto a = b200_view(dy), b = b200_view(dx);
        b200_check(mdnn_nlop_adjoint(h_, o, i, &a, &b));
    }
    // one backward sweep of the library graph for every input (nlop.hpp:53-63)
    void adjoint_all(int o, const MdArray<float>& dy, std::vector<MdArray<float>>& dx) override
    {
        require_forward();
        dx.assign(n_in(), MdArray<float>{});
        std::vector<mdnn_array> v;
        for (int i = 0; i < n_in(); i++) {
            dx[i] = MdArray<float>(ins_[i]);
            v.push_back(b200_view(dx[i]));
        }
        auto a = b200_view(dy);
        b200_check(mdnn_nlop_adjoint_all(h_, o, &a, n_in(), v.data(), nullptr));
    }

private:
    Dims query(int k, bool out) const
    {
        int r = 0;
        long d[MDNN_MAX_RANK];
        b200_check(out ? mdnn_nlop_out_dims(h_, k, &r, d) : mdnn_nlop_in_dims(h_, k, &r, d));
        return Dims(d, d + r);
    }
    mdnn_nlop* h_;
    std::string name_;
    std::vector<Dims> ins_, outs_;
};

} // namespace mdnn
