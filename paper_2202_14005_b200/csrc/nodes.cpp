// Node implementations.  Each class cites the reference node whose forward /
// deriv / adjoint semantics it reproduces.  Inputs are never modified; outputs
// are fresh device arrays; derivative state is held by reference (arrays are
// immutable once produced), replacing the reference's defensive clones.
#include "nodes.h"

#include "kernels.h"

#include <algorithm>
#include <cmath>

namespace mdnn {

namespace {

Dims stride_for(const Dims& adims, const Dims& iter)
{
    // recon.hpp:59-66: default strides, 0 on broadcast dims
    Dims s = default_strides(adims);
    for (size_t d = 0; d < adims.size(); d++)
        if (adims[d] == 1 && iter[d] != 1)
            s[d] = 0;
    return s;
}

struct Iso {
    bool ok = false;
    long inner = 1, nstat = 1, outer = 1;
    IsoGeom geom() const { return IsoGeom{inner, nstat, outer}; }
};

// `sub` broadcasts into `full` (each dim 1 or equal).  ISO when the kept
// (non-broadcast, >1) dims form one contiguous block.
Iso iso_of(const Dims& full, const Dims& sub)
{
    Iso r;
    if (full.size() != sub.size())
        return r;
    int first = -1, last = -1;
    for (size_t d = 0; d < full.size(); d++) {
        if (sub[d] != 1 && sub[d] != full[d])
            return r;
        if (full[d] > 1 && sub[d] == full[d]) {
            if (first < 0)
                first = int(d);
            last = int(d);
        }
    }
    for (size_t d = 0; d < full.size(); d++) {
        bool kept = full[d] > 1 && sub[d] == full[d];
        bool inside = first >= 0 && int(d) >= first && int(d) <= last;
        if (inside && !kept && full[d] > 1)
            return r;
        if (first < 0 || int(d) < first)
            r.inner *= full[d];
        else if (int(d) <= last)
            r.nstat *= full[d];
        else
            r.outer *= full[d];
    }
    r.ok = true;
    return r;
}

class Atom : public Node {
public:
    using Node::Node;
};

// ---------------------------------------------------------------------------
// LinopNode(linop_dft) — fft.hpp:180, linop.hpp:132
class DftNode : public Atom {
public:
    DftNode(const Dims& d, unsigned long flags, bool inv)
        : Atom(inv ? "ifft" : "fft", {d}, {d}), flags_(flags), inv_(inv)
    {
        for (size_t k = 0; k < d.size(); k++)
            if ((flags & (1UL << k)) && d[k] > 1 && !fft_supported(d[k]))
                throw ConfigError("dft: unsupported length " + std::to_string(d[k]));
    }
    bool holomorphic() const override { return true; }
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool) override
    {
        out[0] = run(in[0], inv_);
        bump_generation();
    }
    DArray deriv(int, int, const DArray& dx) override
    {
        require_forward();
        return run(dx, inv_);
    }
    DArray adjoint(int, int, const DArray& dy) override
    {
        require_forward();
        return run(dy, !inv_);
    }

private:
    DArray run(const DArray& x, bool inv) const
    {
        DArray o(x.dims, false);
        fft_flags(o.data(), x.data(), x.dims, flags_, inv);
        return o;
    }
    unsigned long flags_;
    bool inv_;
};

// LinopNode(linop_pad) and its adjoint (crop) — linop.hpp:142-169
class PadNode : public Atom {
public:
    PadNode(const Dims& in, const Dims& out, const Dims& corner, bool crop)
        : Atom(crop ? "crop" : "pad", {crop ? out : in}, {crop ? in : out}), small_(in), big_(out), corner_(corner),
          crop_(crop)
    {
        if (in.size() != out.size() || corner.size() != in.size())
            throw ShapeError("linop_pad: rank mismatch");
        for (size_t d = 0; d < in.size(); d++)
            if (corner[d] < 0 || corner[d] + in[d] > out[d])
                throw ShapeError("linop_pad: window outside output");
    }
    bool holomorphic() const override { return true; }
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool) override
    {
        out[0] = crop_ ? do_crop(in[0]) : do_pad(in[0]);
        bump_generation();
    }
    DArray deriv(int, int, const DArray& dx) override
    {
        require_forward();
        return crop_ ? do_crop(dx) : do_pad(dx);
    }
    DArray adjoint(int, int, const DArray& dy) override
    {
        require_forward();
        return crop_ ? do_pad(dy) : do_crop(dy);
    }

private:
    long window_off(const Dims& s) const
    {
        long off = 0;
        for (size_t d = 0; d < corner_.size(); d++)
            off += corner_[d] * s[d];
        return off;
    }
    DArray do_pad(const DArray& x) const
    {
        DArray y(big_, true);
        Dims sb = default_strides(big_);
        launch_strided_copy(small_, y.data() + window_off(sb), sb, x.data(), default_strides(small_));
        return y;
    }
    DArray do_crop(const DArray& y) const
    {
        DArray x(small_, false);
        Dims sb = default_strides(big_);
        launch_strided_copy(small_, x.data(), default_strides(small_), y.data() + window_off(sb), sb);
        return x;
    }
    Dims small_, big_, corner_;
    bool crop_;
};

// ---------------------------------------------------------------------------
// TenMulNode — ops.hpp:69-118.  Broadcast-elementwise instances (per-channel
// scale, scalar multiply) run on the ISO stat kernels; everything else on the
// generic md_fmac2 kernel.
class TenMulNode : public Atom {
public:
    TenMulNode(const std::string& name, Dims iter, Dims od, Dims so, Dims i1, Dims s1, Dims i2, Dims s2)
        : Atom(name, {i1, i2}, {od}), iter_(std::move(iter)), so_(std::move(so)), s1_(std::move(s1)),
          s2_(std::move(s2))
    {
        const Dims& o = outs_[0];
        // strides on extent-1 iteration dims never move the pointer: ignore them
        auto same = [&](const Dims& a, const Dims& b) {
            for (size_t d = 0; d < iter_.size(); d++)
                if (iter_[d] > 1 && a[d] != b[d])
                    return false;
            return true;
        };
        if (iter_ == o && ins_[0] == o && same(so_, default_strides(o)) && same(s1_, default_strides(o))
            && same(s2_, stride_for(ins_[1], iter_))) {
            iso_ = iso_of(o, ins_[1]);
        }
    }
    bool holomorphic() const override { return true; }

    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool store) override
    {
        out[0] = mul(in[0], in[1]);
        if (store) {
            x1_ = in[0];
            x2_ = in[1];
        } else {
            x1_ = {};
            x2_ = {};
        }
        bump_generation();
    }
    DArray deriv(int, int i, const DArray& dx) override
    {
        require_forward();
        return i == 0 ? mul(dx, x2_) : mul(x1_, dx);
    }
    DArray adjoint(int, int i, const DArray& dy) override
    {
        require_forward();
        if (iso_.ok) {
            if (i == 0) {
                DArray dx(ins_[0], false);
                launch_stat_mul(dx.data(), dy.data(), x2_.data(), iso_.geom(), true);
                return dx;
            }
            DArray dx(ins_[1], false);
            launch_iso_reduce(dx.data(), dy.data(), x1_.data(), iso_.inner, iso_.nstat, iso_.outer, 1, 1.f);
            return dx;
        }
        if (i == 0) {
            DArray dx(ins_[0], true);
            launch_fmac_generic(iter_, dx.data(), s1_, dy.data(), so_, x2_.data(), s2_, true);
            return dx;
        }
        DArray dx(ins_[1], true);
        launch_fmac_generic(iter_, dx.data(), s2_, dy.data(), so_, x1_.data(), s1_, true);
        return dx;
    }

private:
    DArray mul(const DArray& a, const DArray& b) const
    {
        if (iso_.ok) {
            DArray o(outs_[0], false);
            launch_stat_mul(o.data(), a.data(), b.data(), iso_.geom(), false);
            return o;
        }
        DArray o(outs_[0], true);
        launch_fmac_generic(iter_, o.data(), so_, a.data(), s1_, b.data(), s2_, false);
        return o;
    }
    Dims iter_, so_, s1_, s2_;
    Iso iso_;
    DArray x1_, x2_;
};

// AddNode — ops.hpp:122-149
class AddNode : public Atom {
public:
    AddNode(const Dims& d, bool sub) : Atom(sub ? "sub" : "add", {d, d}, {d}), sub_(sub) {}
    bool holomorphic() const override { return true; }
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool) override
    {
        DArray o(outs_[0], false);
        launch_add(o.data(), in[0].data(), in[1].data(), sub_ ? -1.f : 1.f, o.size());
        out[0] = o;
        bump_generation();
    }
    DArray deriv(int, int i, const DArray& dx) override
    {
        require_forward();
        if (sub_ && i == 1) {
            DArray o(dx.dims, false);
            launch_neg(o.data(), dx.data(), o.size());
            return o;
        }
        return dx;
    }
    DArray adjoint(int o, int i, const DArray& dy) override { return deriv(o, i, dy); }

private:
    bool sub_;
};

// BroadcastAddNode — ops.hpp:153-209
class BcastAddNode : public Atom {
public:
    BcastAddNode(const Dims& x, const Dims& b) : Atom("add_bcast", {x, b}, {x})
    {
        if (x.size() != b.size())
            throw ShapeError("add_bcast: rank mismatch");
        for (size_t d = 0; d < x.size(); d++)
            if (b[d] != 1 && b[d] != x[d])
                throw ShapeError("add_bcast: dim " + std::to_string(d) + " not broadcastable");
        iso_ = iso_of(x, b);
        sb_ = stride_for(b, x);
    }
    bool holomorphic() const override { return true; }
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool) override
    {
        out[0] = add(in[0], in[1]);
        bump_generation();
    }
    DArray deriv(int, int i, const DArray& dx) override
    {
        require_forward();
        if (i == 0)
            return dx;
        DArray z(outs_[0], true);
        return add(z, dx);
    }
    DArray adjoint(int, int i, const DArray& dy) override
    {
        require_forward();
        if (i == 0)
            return dy;
        DArray db(ins_[1], false);
        if (iso_.ok) {
            launch_iso_reduce(db.data(), dy.data(), nullptr, iso_.inner, iso_.nstat, iso_.outer, 0, 1.f);
        } else {
            db.zero();
            DArray one = DArray::scalar(1.f);
            launch_fmac_generic(outs_[0], db.data(), sb_, dy.data(), default_strides(outs_[0]), one.data(),
                                Dims(outs_[0].size(), 0), false);
        }
        return db;
    }

private:
    DArray add(const DArray& x, const DArray& b) const
    {
        DArray o(outs_[0], false);
        if (iso_.ok)
            launch_stat_add(o.data(), x.data(), b.data(), iso_.geom());
        else
            launch_bcast_binary(outs_[0], o.data(), x.data(), default_strides(outs_[0]), b.data(), sb_, 0);
        return o;
    }
    Iso iso_;
    Dims sb_;
};

// ForkNode — ops.hpp:214-238 (outputs share the immutable input)
class ForkNode : public Atom {
public:
    ForkNode(const Dims& d, int n) : Atom("fork", {d}, std::vector<Dims>(size_t(n), d)) {}
    bool holomorphic() const override { return true; }
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool) override
    {
        for (auto& o : out)
            o = in[0];
        bump_generation();
    }
    DArray deriv(int, int, const DArray& dx) override
    {
        require_forward();
        return dx;
    }
    DArray adjoint(int, int, const DArray& dy) override
    {
        require_forward();
        return dy;
    }
};

// elementwise R-linear maps: Zconj (ops.hpp:246), Zreal (ops.hpp:266)
class MapNode : public Atom {
public:
    enum Kind { Conj, Real };
    MapNode(const Dims& d, Kind k) : Atom(k == Conj ? "zconj" : "zreal", {d}, {d}), k_(k) {}
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool) override
    {
        out[0] = run(in[0]);
        bump_generation();
    }
    DArray deriv(int, int, const DArray& dx) override
    {
        require_forward();
        return run(dx);
    }
    DArray adjoint(int, int, const DArray& dy) override
    {
        require_forward();
        return run(dy);
    }

private:
    DArray run(const DArray& x) const
    {
        if (x.known_real) // Re(x) = conj(x) = x (values are immutable: share the array)
            return x;
        DArray o(x.dims, false);
        if (k_ == Conj) {
            launch_conj(o.data(), x.data(), o.size());
            o.known_real = x.known_real;
        } else {
            launch_real(o.data(), x.data(), o.size());
            o.known_real = true;
        }
        return o;
    }
    Kind k_;
};

// RealChanNode / ChanCplxNode — ops.hpp:318-411
class ChanSplitNode : public Atom {
public:
    ChanSplitNode(const Dims& d, int cd, bool join)
        : Atom(join ? "chan_cplx" : "real_chan", {d}, {chan(d, cd, join)}), join_(join)
    {
        const Dims& small = join ? outs_[0] : ins_[0];
        for (int k = 0; k < cd; k++)
            inner_ *= small[k];
        for (size_t k = cd + 1; k < small.size(); k++)
            outer_ *= small[k];
    }
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool) override
    {
        out[0] = join_ ? do_join(in[0]) : do_split(in[0]);
        bump_generation();
    }
    DArray deriv(int, int, const DArray& dx) override
    {
        require_forward();
        return join_ ? do_join(dx) : do_split(dx);
    }
    DArray adjoint(int, int, const DArray& dy) override
    {
        require_forward();
        return join_ ? do_split(dy) : do_join(dy);
    }

private:
    static Dims chan(Dims d, int cd, bool join)
    {
        if (d.at(cd) != (join ? 2 : 1))
            throw ShapeError(join ? "chan_cplx: channel dim must have size 2" : "real_chan: channel dim must have size 1");
        d[cd] = join ? 1 : 2;
        return d;
    }
    DArray do_split(const DArray& x) const
    {
        Dims big = join_ ? ins_[0] : outs_[0];
        DArray o(big, false);
        launch_real_chan_split(o.data(), x.data(), inner_, outer_);
        o.known_real = true;
        return o;
    }
    DArray do_join(const DArray& x) const
    {
        Dims small = join_ ? outs_[0] : ins_[0];
        DArray o(small, false);
        launch_real_chan_join(o.data(), x.data(), inner_, outer_);
        return o;
    }
    bool join_;
    long inner_ = 1, outer_ = 1;
};

// CReluNode — ops.hpp:451-475
class CReluNode : public Atom {
public:
    explicit CReluNode(const Dims& d) : Atom("crelu", {d}, {d}) {}
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool store) override
    {
        DArray o(outs_[0], false);
        launch_crelu(o.data(), in[0].data(), o.size());
        out[0] = o;
        x_ = store ? in[0] : DArray{};
        bump_generation();
    }
    DArray deriv(int, int, const DArray& dx) override
    {
        require_forward();
        DArray o(dx.dims, false);
        launch_crelu_mask(o.data(), dx.data(), x_.data(), o.size());
        return o;
    }
    DArray adjoint(int o, int i, const DArray& dy) override { return deriv(o, i, dy); }

private:
    DArray x_;
};

// ExpRealNode — ops.hpp:672-697
class ExpRealNode : public Atom {
public:
    explicit ExpRealNode(const Dims& d) : Atom("exp_real", {d}, {d}) {}
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool store) override
    {
        DArray o(outs_[0], false);
        launch_exp_real(o.data(), in[0].data(), o.size());
        out[0] = o;
        y_ = store ? o : DArray{};
        bump_generation();
    }
    DArray deriv(int, int, const DArray& dx) override
    {
        require_forward();
        DArray o(dx.dims, false);
        launch_mul_real_real(o.data(), y_.data(), dx.data(), o.size());
        return o;
    }
    DArray adjoint(int o, int i, const DArray& dy) override { return deriv(o, i, dy); }

private:
    DArray y_;
};

// MseNode — ops.hpp:874-906
class MseNode : public Atom {
public:
    explicit MseNode(const Dims& d) : Atom("mse", {d, d}, {Dims{1}}) {}
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool store) override
    {
        DArray diff(ins_[0], false), loss(Dims{1}, false);
        mse_forward(loss.data(), diff.data(), in[0].data(), in[1].data(), diff.size());
        out[0] = loss;
        diff_ = store ? diff : DArray{};
        bump_generation();
    }
    DArray deriv(int, int i, const DArray& dx) override
    {
        require_forward();
        const long n = md_size(ins_[0]);
        DArray z(Dims{1}, false), o(Dims{1}, false);
        launch_iso_reduce(z.data(), dx.data(), diff_.data(), n, 1, 1, 1, 1.f);
        launch_real_scalar(o.data(), z.data(), float((i == 0 ? 2.0 : -2.0) / double(n)));
        return o;
    }
    DArray adjoint(int, int i, const DArray& dy) override
    {
        require_forward();
        const long n = md_size(ins_[0]);
        DArray o(ins_[0], false);
        launch_scale_dev_real(o.data(), diff_.data(), dy.data(), float((i == 0 ? 2.0 : -2.0) / double(n)), n);
        return o;
    }

private:
    DArray diff_;
};

// BatchNormNode — ops.hpp:1070-1298
class BatchNormNode : public Atom {
public:
    BatchNormNode(const Dims& d, unsigned long flags, bool train, double eps, double mom)
        : Atom("batchnorm", {d, stat_dims(d, flags), stat_dims(d, flags)},
               train ? std::vector<Dims>{d, stat_dims(d, flags), stat_dims(d, flags)} : std::vector<Dims>{d}),
          train_(train), eps_(float(eps)), mom_(float(mom))
    {
        iso_ = iso_of(d, stat_dims(d, flags));
        if (!iso_.ok)
            throw ConfigError("batchnorm: statistics axes must form inner/outer blocks around the feature axes");
        m_ = double(iso_.inner * iso_.outer);
    }
    bool zero_deriv(int o, int i) const override
    {
        if (!train_)
            return false;
        if (o == 0)
            return i != 0;
        if (o == 1)
            return i == 2;
        return i == 1;
    }
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool store) override
    {
        const Dims& sd = ins_[1];
        DArray y(ins_[0], false), u(ins_[0], false), istd(sd, false);
        if (train_) {
            DArray mo(sd, false), vo(sd, false);
            bn_train_forward(y.data(), u.data(), istd.data(), mo.data(), vo.data(), in[0].data(), in[1].data(),
                             in[2].data(), iso_.geom(), eps_, mom_);
            out[1] = mo;
            out[2] = vo;
        } else {
            bn_infer_forward(y.data(), u.data(), istd.data(), in[0].data(), in[1].data(), in[2].data(), iso_.geom(),
                             eps_);
        }
        out[0] = y;
        if (store) {
            u_ = u;
            istd_ = istd;
        } else {
            u_ = {};
            istd_ = {};
        }
        bump_generation();
    }
    DArray deriv(int o, int i, const DArray& dx) override
    {
        require_forward();
        const Dims& xd = ins_[0];
        const Dims& sd = ins_[1];
        if (!train_) {
            DArray dy(xd, false);
            if (i == 0) {
                launch_stat_mul(dy.data(), dx.data(), istd_.data(), iso_.geom(), false);
            } else if (i == 1) {
                DArray z(xd, true), t(xd, false);
                launch_stat_add(t.data(), z.data(), dx.data(), iso_.geom());
                DArray ni = neg(istd_);
                launch_stat_mul(dy.data(), t.data(), ni.data(), iso_.geom(), false);
            } else {
                DArray f = small_f(dx, istd_, -0.5f); // -Re(dvar)/2 istd^3
                launch_stat_mul(dy.data(), u_.data(), f.data(), iso_.geom(), false);
            }
            return dy;
        }
        if (o == 0) {
            DArray dy(xd, false);
            bn_train_deriv_x(dy.data(), dx.data(), u_.data(), istd_.data(), iso_.geom());
            return dy;
        }
        DArray dy(sd, false);
        if (i != 0) {
            launch_scale(dy.data(), dx.data(), cfloat{1.f - mom_, 0.f}, dy.size());
            return dy;
        }
        if (o == 1) {
            launch_iso_reduce(dy.data(), dx.data(), nullptr, iso_.inner, iso_.nstat, iso_.outer, 0,
                              float(mom_ / m_));
        } else {
            DArray p(sd, false);
            launch_iso_reduce(p.data(), dx.data(), u_.data(), iso_.inner, iso_.nstat, iso_.outer, 1, 1.f);
            // dy = (mom * 2 * Re(p) / m, 0)
            DArray q(sd, false);
            launch_real(q.data(), p.data(), q.size());
            launch_scale(dy.data(), q.data(), cfloat{float(mom_ * 2.0 / m_), 0.f}, dy.size());
        }
        return dy;
    }
    DArray adjoint(int o, int i, const DArray& g) override
    {
        require_forward();
        const Dims& xd = ins_[0];
        const Dims& sd = ins_[1];
        if (!train_) {
            if (i == 0) {
                DArray dx(xd, false);
                launch_stat_mul(dx.data(), g.data(), istd_.data(), iso_.geom(), false);
                return dx;
            }
            DArray dx(sd, false);
            if (i == 1) {
                // -sum(g) * istd
                DArray s(sd, false);
                launch_iso_reduce(s.data(), g.data(), nullptr, iso_.inner, iso_.nstat, iso_.outer, 0, 1.f);
                DArray ni = neg(istd_);
                launch_stat_mul(dx.data(), s.data(), ni.data(), IsoGeom{1, iso_.nstat, 1}, false);
            } else {
                // -Re(sum g conj(u)) istd^3 / 2
                DArray p(sd, false);
                launch_iso_reduce(p.data(), g.data(), u_.data(), iso_.inner, iso_.nstat, iso_.outer, 1, 1.f);
                dx = small_f(p, istd_, -0.5f);
            }
            return dx;
        }
        if (o == 0) {
            if (i != 0)
                throw StaleDerivativeError("batchnorm: structurally zero adjoint requested");
            DArray dx(xd, false);
            bn_train_adjoint_x(dx.data(), g.data(), u_.data(), istd_.data(), iso_.geom());
            return dx;
        }
        if (i != 0) {
            DArray dx(sd, false);
            launch_scale(dx.data(), g.data(), cfloat{1.f - mom_, 0.f}, dx.size());
            return dx;
        }
        DArray dx(xd, false);
        if (o == 1) {
            DArray z(xd, true), t(xd, false);
            launch_stat_add(t.data(), z.data(), g.data(), iso_.geom());
            launch_scale(dx.data(), t.data(), cfloat{float(mom_ / m_), 0.f}, dx.size());
        } else {
            DArray q(sd, false), f(sd, false);
            launch_real(q.data(), g.data(), q.size());
            launch_scale(f.data(), q.data(), cfloat{float(mom_ * 2.0 / m_), 0.f}, f.size());
            launch_stat_mul(dx.data(), u_.data(), f.data(), iso_.geom(), false);
        }
        return dx;
    }

    static Dims stat_dims(Dims d, unsigned long flags)
    {
        for (size_t k = 0; k < d.size(); k++)
            if (flags & (1UL << k))
                d[k] = 1;
        return d;
    }

private:
    static DArray neg(const DArray& a)
    {
        DArray o(a.dims, false);
        launch_neg(o.data(), a.data(), o.size());
        return o;
    }
    // (c * Re(p) * istd^3, 0) per stat
    static DArray small_f(const DArray& p, const DArray& istd, float c)
    {
        DArray r(p.dims, false), i3(p.dims, false), t(p.dims, false);
        launch_real(r.data(), p.data(), r.size());
        DArray i2(p.dims, false);
        launch_bcast_binary(Dims{p.size()}, i2.data(), istd.data(), Dims{1}, istd.data(), Dims{1}, 1);
        launch_bcast_binary(Dims{p.size()}, i3.data(), i2.data(), Dims{1}, istd.data(), Dims{1}, 1);
        launch_bcast_binary(Dims{p.size()}, t.data(), r.data(), Dims{1}, i3.data(), Dims{1}, 1);
        DArray o(p.dims, false);
        launch_scale(o.data(), t.data(), cfloat{c, 0.f}, o.size());
        return o;
    }
    bool train_;
    float eps_, mom_;
    double m_ = 1;
    Iso iso_;
    DArray u_, istd_;
};

// RbfNode — ops.hpp:1308-1427
class RbfNode : public Atom {
public:
    RbfNode(const Dims& z, int fd, const std::vector<float>& mu, float sigma)
        : Atom("rbf", {z, Dims{z.at(fd), long(mu.size())}}, {z}), sigma_(sigma)
    {
        if (!(sigma > 0))
            throw ConfigError("rbf: width must be positive");
        for (size_t j = 1; j < mu.size(); j++)
            if (!(mu[j] > mu[j - 1]))
                throw ConfigError("rbf: centers must be strictly increasing");
        g_.inner = 1;
        g_.outer = 1;
        for (int k = 0; k < fd; k++)
            g_.inner *= z[k];
        for (size_t k = fd + 1; k < z.size(); k++)
            g_.outer *= z[k];
        g_.nf = z[fd];
        g_.nw = int(mu.size());
        g_.sigma = sigma;
        mu_host_ = mu;
        rbf_set_window(g_, mu);
    }
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool store) override
    {
        if (!mu_) { // centres uploaded on first use: graph construction stays host-only
            float* d;
            CUDA_CHECK(cudaMalloc(&d, mu_host_.size() * sizeof(float)));
            CUDA_CHECK(cudaMemcpy(d, mu_host_.data(), mu_host_.size() * sizeof(float), cudaMemcpyHostToDevice));
            mu_.reset(d, [](float* p) { cudaFree(p); });
        }
        DArray y(outs_[0], false);
        rbf_forward(y.data(), in[0].data(), in[1].data(), mu_.get(), g_);
        y.known_real = true; // phi acts on Re z and writes zero imaginary parts
        out[0] = y;
        if (store) {
            z_ = in[0];
            w_ = in[1];
        } else {
            z_ = {};
            w_ = {};
        }
        bump_generation();
    }
    DArray deriv(int, int i, const DArray& dx) override
    {
        require_forward();
        DArray dy(outs_[0], false);
        if (i == 0)
            rbf_deriv_z(dy.data(), dx.data(), z_.data(), w_.data(), mu_.get(), g_);
        else
            rbf_deriv_w(dy.data(), dx.data(), z_.data(), mu_.get(), g_);
        return dy;
    }
    DArray adjoint(int, int i, const DArray& dy) override
    {
        require_forward();
        if (i == 0) {
            DArray dz(ins_[0], false);
            rbf_adjoint_z(dz.data(), dy.data(), z_.data(), w_.data(), mu_.get(), g_);
            dz.known_real = true;
            return dz;
        }
        DArray dw(ins_[1], false);
        rbf_adjoint_w(dw.data(), dy.data(), z_.data(), mu_.get(), g_);
        return dw;
    }
    void adjoint_all(int o, const DArray& dy, std::vector<DArray>& dx, const std::vector<char>& want) override
    {
        if (!(want.size() > 1 && want[0] && want[1])) {
            Atom::adjoint_all(o, dy, dx, want);
            return;
        }
        require_forward();
        dx.assign(n_in(), DArray{});
        DArray dz(ins_[0], false), dw(ins_[1], false);
        rbf_adjoint_zw(dz.data(), dw.data(), dy.data(), z_.data(), w_.data(), mu_.get(), g_);
        dz.known_real = true;
        dx[0] = dz;
        dx[1] = dw;
    }

private:
    float sigma_;
    RbfGeom g_{};
    std::vector<float> mu_host_;
    std::shared_ptr<float> mu_;
    DArray z_, w_;
};

// ---------------------------------------------------------------------------
// Fused SENSE nodes.  Inputs carry the reference fragment's argument order.
SenseGeom geom_of(const SenseDims& sd)
{
    SenseGeom g{};
    g.X = sd.x;
    g.Y = sd.y;
    g.C = sd.coils;
    g.M = sd.maps;
    g.B = sd.batch;
    g.pat_x = 1;
    g.pat_y = sd.y;
    g.pat_c = 1;
    g.pat_b = 1;
    return g;
}

DArray conj_of(const DArray& a)
{
    DArray o(a.dims, false);
    launch_conj(o.data(), a.data(), o.size());
    return o;
}

// k = F2(C x) per coil (no mask)
DArray coil_fft(const SenseDims& sd, const DArray& x, const DArray& coils)
{
    SenseGeom g = geom_of(sd);
    DArray k(sd.coil_img(), false);
    launch_coil_mul(k.data(), x.data(), coils.data(), g);
    fft_flags(k.data(), k.data(), k.dims, 3UL, false);
    return k;
}

// image = sum_c conj(C) F2^H(k)
DArray coil_ifft_adj(const SenseDims& sd, const DArray& k, const DArray& coils)
{
    SenseGeom g = geom_of(sd);
    DArray t(sd.coil_img(), false), x(sd.image(), false);
    fft_flags(t.data(), k.data(), k.dims, 3UL, true);
    launch_coil_adj(x.data(), t.data(), coils.data(), g);
    return x;
}

DArray pat_mul(const SenseDims& sd, const DArray& k, const DArray& pattern)
{
    SenseGeom g = geom_of(sd);
    DArray o(k.dims, false);
    launch_pattern_mul(o.data(), k.data(), pattern.data(), g);
    return o;
}

// per-coil products: out[c] = a[c] (*) b (image broadcast over coils), op 1 = a*b, 2 = a*conj(b)
DArray coil_bcast(const SenseDims& sd, const DArray& a_coil, const DArray& b_img, int op, bool conj_a)
{
    DArray a = conj_a ? conj_of(a_coil) : a_coil;
    Dims cd = sd.coil_maps();
    DArray o(cd, false);
    Dims sa = default_strides(sd.coil_img());
    Dims sa2(max_rank, 0), sb(max_rank, 0);
    // coil image index [x,y,c,b]; image index [x,y,m,b]; out [x,y,c,m,b]
    Dims si = default_strides(sd.image());
    sa2[0] = sa[0];
    sa2[1] = sa[1];
    sa2[3] = sa[3];
    sa2[15] = sa[15];
    sb[0] = si[0];
    sb[1] = si[1];
    sb[4] = si[4];
    sb[15] = si[15];
    launch_bcast_binary(cd, o.data(), a.data(), sa2, b_img.data(), sb, op);
    return o;
}

// sum over (x, coil, batch) of a * conj(b) into the pattern dims [1,Y]
DArray pattern_reduce(const SenseDims& sd, const DArray& a, const DArray& b)
{
    Dims iter = sd.coil_img();
    DArray o(sd.pattern(), true);
    Dims so(max_rank, 0);
    so[1] = 1;
    Dims s = default_strides(iter);
    launch_fmac_generic(iter, o.data(), so, a.data(), s, b.data(), s, true);
    return o;
}

class SenseNormalNode : public Atom {
public:
    // lam_variant: inputs (x, coils, pattern, lambda); else (x, coils, pattern, coils)
    SenseNormalNode(const SenseDims& sd, bool lam_variant)
        : Atom(lam_variant ? "sense_normal_lambda" : "sense_normal",
               {sd.image(), sd.coil_maps(), sd.pattern(), lam_variant ? Dims(max_rank, 1) : sd.coil_maps()},
               {sd.image()}),
          sd_(sd), lam_(lam_variant)
    {
    }
    bool holomorphic() const override { return false; }
    const SenseDims& dims() const { return sd_; }
    bool lam_variant() const { return lam_; }

    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool store) override
    {
        out[0] = apply_S(in[0], in[1], in[2], c2(in), lam(in));
        if (store)
            st_ = in;
        else
            st_.clear();
        bump_generation();
    }
    DArray deriv(int, int i, const DArray& dx) override
    {
        require_forward();
        const DArray &x = st_[0], &C1 = st_[1], &P = st_[2];
        const DArray C2 = c2(st_);
        if (i == 0)
            return apply_S(dx, C1, P, C2, lam(st_));
        if (lam_ && i == 3) {
            DArray o(sd_.image(), false);
            launch_scale_dev(o.data(), x.data(), dx.data(), false, o.size());
            return o;
        }
        if (i == 2) // sum conj(C2) F^H (dP F(C1 x))
            return coil_ifft_adj(sd_, pat_mul(sd_, coil_fft(sd_, x, C1), dx), C2);
        // coil-multiply maps: sum conj(C2) F^H P F (dC1 x)
        auto d1 = [&] { return coil_ifft_adj(sd_, pat_mul(sd_, coil_fft(sd_, x, dx), P), C2); };
        // coil-combine maps: sum conj(dC2) F^H P F(C1 x)
        auto d2 = [&] { return coil_ifft_adj(sd_, pat_mul(sd_, coil_fft(sd_, x, C1), P), dx); };
        if (!lam_)
            return i == 1 ? d1() : d2();
        // lambda variant: the single (deduped) coils input feeds both
        return accumulate(d1(), d2());
    }
    DArray adjoint(int, int i, const DArray& g) override
    {
        require_forward();
        return param_adjoint(i, st_[0], g, st_);
    }

    // adjoint wrt input i evaluated at an explicit x (used by the fused
    // InverseNode without re-applying S at x*)
    DArray param_adjoint(int i, const DArray& x, const DArray& g, const std::vector<DArray>& in) const
    {
        const DArray &C1 = in[1], &P = in[2];
        const DArray C2 = c2(in);
        if (i == 0) { // S^H g = sum conj(C1) F^H conj(P) F (C2 g) + conj(lam) g
            DArray l = lam(in);
            DArray lc = l.valid() ? conj_of(l) : l;
            DArray Pc = conj_of(P);
            return apply_S(g, C2, Pc, C1, lc);
        }
        if (lam_ && i == 3) { // sum g conj(x)
            DArray o(ins_[3], false);
            launch_iso_reduce(o.data(), g.data(), x.data(), md_size(sd_.image()), 1, 1, 1, 1.f);
            return o;
        }
        if (i == 2) // sum F(C2 g) conj(F(C1 x))
            return pattern_reduce(sd_, coil_fft(sd_, g, C2), coil_fft(sd_, x, C1));
        // coil-multiply maps: w conj(x), w = F^H conj(P) F (C2 g)
        auto a1 = [&] {
            DArray w(sd_.coil_img(), false);
            DArray k = pat_mul(sd_, coil_fft(sd_, g, C2), conj_of(P));
            fft_flags(w.data(), k.data(), k.dims, 3UL, true);
            return coil_bcast(sd_, w, x, 2, false);
        };
        // coil-combine maps: conj(g) v, v = F^H P F (C1 x)  (= conj(conj(v) g))
        auto a2 = [&] {
            DArray v(sd_.coil_img(), false);
            DArray k = pat_mul(sd_, coil_fft(sd_, x, C1), P);
            fft_flags(v.data(), k.data(), k.dims, 3UL, true);
            return conj_of(coil_bcast(sd_, v, g, 1, true));
        };
        if (!lam_)
            return i == 1 ? a1() : a2();
        return accumulate(a1(), a2());
    }

    DArray apply_S(const DArray& x, const DArray& C1, const DArray& P, const DArray& C2, const DArray& l) const
    {
        DArray o(sd_.image(), false);
        sense_normal(o.data(), x.data(), C1.data(), P.data(), l.valid() ? l.data() : nullptr, geom_of(sd_),
                     C2.data());
        return o;
    }

private:
    DArray c2(const std::vector<DArray>& in) const { return lam_ ? in[1] : in[3]; }
    DArray lam(const std::vector<DArray>& in) const { return lam_ ? in[3] : DArray{}; }
    SenseDims sd_;
    bool lam_;
    std::vector<DArray> st_;
};

// A^H y as sense_adjoint_fragment: inputs (y, pattern, coils)
class SenseAdjointNode : public Atom {
public:
    explicit SenseAdjointNode(const SenseDims& sd)
        : Atom("sense_adjoint", {sd.coil_img(), sd.pattern(), sd.coil_maps()}, {sd.image()}), sd_(sd)
    {
    }
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool store) override
    {
        out[0] = coil_ifft_adj(sd_, pat_mul(sd_, in[0], in[1]), in[2]);
        if (store)
            st_ = in;
        bump_generation();
    }
    DArray deriv(int, int i, const DArray& dx) override
    {
        require_forward();
        const DArray &y = st_[0], &P = st_[1], &C = st_[2];
        if (i == 0)
            return coil_ifft_adj(sd_, pat_mul(sd_, dx, P), C);
        if (i == 1)
            return coil_ifft_adj(sd_, pat_mul(sd_, y, dx), C);
        return coil_ifft_adj(sd_, pat_mul(sd_, y, P), dx);
    }
    DArray adjoint(int, int i, const DArray& g) override
    {
        require_forward();
        const DArray &y = st_[0], &P = st_[1], &C = st_[2];
        if (i == 0)
            return pat_mul(sd_, coil_fft(sd_, g, C), conj_of(P));
        if (i == 1) { // sum F(C g) conj(y)
            return pattern_reduce(sd_, coil_fft(sd_, g, C), y);
        }
        // conj(g) v, v = F^H(P y)
        DArray v(sd_.coil_img(), false);
        DArray k = pat_mul(sd_, y, P);
        fft_flags(v.data(), k.data(), k.dims, 3UL, true);
        return conj_of(coil_bcast(sd_, v, g, 1, true)); // conj(conj(v) g) = conj(g) v
    }

private:
    SenseDims sd_;
    std::vector<DArray> st_;
};

// A x as sense_forward_fragment: inputs (x, coils, pattern)
class SenseForwardNode : public Atom {
public:
    explicit SenseForwardNode(const SenseDims& sd)
        : Atom("sense_forward", {sd.image(), sd.coil_maps(), sd.pattern()}, {sd.coil_img()}), sd_(sd)
    {
    }
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool store) override
    {
        out[0] = pat_mul(sd_, coil_fft(sd_, in[0], in[1]), in[2]);
        if (store)
            st_ = in;
        bump_generation();
    }
    DArray deriv(int, int i, const DArray& dx) override
    {
        require_forward();
        const DArray &x = st_[0], &C = st_[1], &P = st_[2];
        if (i == 0)
            return pat_mul(sd_, coil_fft(sd_, dx, C), P);
        if (i == 1)
            return pat_mul(sd_, coil_fft(sd_, x, dx), P);
        return pat_mul(sd_, coil_fft(sd_, x, C), dx);
    }
    DArray adjoint(int, int i, const DArray& g) override
    {
        require_forward();
        const DArray &x = st_[0], &C = st_[1], &P = st_[2];
        DArray t = pat_mul(sd_, g, conj_of(P));
        if (i == 0)
            return coil_ifft_adj(sd_, t, C);
        if (i == 1) {
            DArray w(sd_.coil_img(), false);
            fft_flags(w.data(), t.data(), t.dims, 3UL, true);
            return coil_bcast(sd_, w, x, 2, false);
        }
        return pattern_reduce(sd_, g, coil_fft(sd_, x, C));
    }

private:
    SenseDims sd_;
    std::vector<DArray> st_;
};

// ---------------------------------------------------------------------------
// InverseNode — recon.hpp:211-329 (Eq. 12 derivatives).  When S is the fused
// sense_normal_lambda node the CG runs on the fused single-pass kernel and the
// parameter cotangents are evaluated directly at x* (no settle re-apply).
class InverseNode : public Node {
public:
    InverseNode(Nlop s, long max_iter, double tol)
        : Node("inverse", in_list(s), {s.in_dims(0)}), s_(std::move(s)), max_iter_(max_iter), tol_(tol)
    {
        if (s_.nodes().size() == 1)
            fused_ = std::dynamic_pointer_cast<SenseNormalNode>(s_.nodes()[0]);
        if (fused_ && !fused_->lam_variant())
            fused_.reset();
    }
    static std::vector<Dims> in_list(const Nlop& s)
    {
        if (s.n_out() != 1)
            throw ConfigError("inverse: operator must have a single output");
        if (s.n_in() < 2)
            throw ConfigError("inverse: operator needs an x input and at least one parameter");
        if (s.out_dims(0) != s.in_dims(0))
            throw ConfigError("inverse: operator must map x to its own shape");
        std::vector<Dims> v;
        v.push_back(s.out_dims(0));
        for (int i = 1; i < s.n_in(); i++)
            v.push_back(s.in_dims(i));
        return v;
    }

    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool) override
    {
        params_.assign(in.begin() + 1, in.end());
        xstar_ = solve(in[0], true);
        out[0] = xstar_;
        settled_ = false;
        bump_generation();
    }
    DArray deriv(int, int i, const DArray& dx) override
    {
        require_forward();
        if (i == 0)
            return solve(dx, false);
        // D_p S at x*: the inner node's tangent formulas after a private forward at x*
        settle();
        DArray w = s_.derivative(0, i, dx);
        DArray z = solve(w, false);
        DArray o(z.dims, false);
        launch_neg(o.data(), z.data(), o.size());
        return o;
    }
    DArray adjoint(int o, int i, const DArray& dy) override
    {
        std::vector<char> want(n_in(), 0);
        want[i] = 1;
        std::vector<DArray> dx;
        adjoint_all(o, dy, dx, want);
        return dx[i];
    }
    void adjoint_all(int, const DArray& dy, std::vector<DArray>& dx, const std::vector<char>& want) override
    {
        require_forward();
        dx.assign(n_in(), DArray{});
        DArray z = solve(dy, false); // S^-1 is self-adjoint
        bool any = false;
        for (int i = 1; i < n_in(); i++)
            any |= want[i] != 0;
        if (any) {
            if (fused_) {
                std::vector<DArray> sin;
                sin.push_back(xstar_);
                sin.insert(sin.end(), params_.begin(), params_.end());
                for (int i = 1; i < n_in(); i++)
                    if (want[i])
                        dx[i] = negate(fused_->param_adjoint(i, xstar_, z, sin));
            } else {
                settle();
                std::vector<char> w2 = want;
                w2[0] = 0;
                auto g = s_.adjoint_all(0, z, w2);
                for (int i = 1; i < n_in(); i++)
                    if (want[i])
                        dx[i] = negate(g[i]);
            }
        }
        if (want[0])
            dx[0] = z;
    }

    CgResult status() const
    {
        if (!status_.valid())
            throw StaleDerivativeError("cg_status: inverse node has not been applied");
        return read_cg_status(reinterpret_cast<const double*>(status_.data()));
    }

private:
    static DArray negate(const DArray& a)
    {
        DArray o(a.dims, false);
        launch_neg(o.data(), a.data(), o.size());
        return o;
    }
    DArray solve(const DArray& b, bool record)
    {
        if (!status_.valid())
            status_ = DArray(Dims{3}, true); // [iterations, rel_residual, converged] as doubles
        DArray x(b.dims, false);
        double* st = record ? reinterpret_cast<double*>(status_.data()) : nullptr;
        if (fused_) {
            SenseGeom g = geom_of(fused_->dims());
            cg_normal_device(x.data(), b.data(), params_[0].data(), params_[1].data(), params_[2].data(), g,
                             max_iter_, tol_, st);
        } else {
            const Dims xd = b.dims;
            cg_generic_device(
                x.data(), b.data(), b.size(),
                [&](const cfloat* p, cfloat* ap) {
                    std::vector<DArray> in;
                    in.push_back(DArray::view(const_cast<cfloat*>(p), xd));
                    in.insert(in.end(), params_.begin(), params_.end());
                    DArray r = s_.apply(in)[0];
                    launch_copy(ap, r.data(), r.size());
                },
                max_iter_, tol_, st);
        }
        settled_ = false;
        return x;
    }
    void settle()
    {
        if (settled_)
            return;
        std::vector<DArray> in;
        in.push_back(xstar_);
        in.insert(in.end(), params_.begin(), params_.end());
        s_.apply(in);
        settled_ = true;
    }

    Nlop s_;
    long max_iter_;
    double tol_;
    std::shared_ptr<SenseNormalNode> fused_;
    std::vector<DArray> params_;
    DArray xstar_;
    DArray status_;
    bool settled_ = false;
};

// ---------------------------------------------------------------------------
// conv core nodes (canonical layout, axes {0,1}, channel dim 2, same padding)
class ConvNode : public Atom {
public:
    ConvNode(const std::string& name, const ConvSpec& s, bool transposed)
        : Atom(name, transposed ? std::vector<Dims>{s.weight_dims(), s.out_dims()}
                                : std::vector<Dims>{s.in_dims, s.weight_dims()},
               {transposed ? s.in_dims : s.out_dims()}),
          t_(transposed)
    {
        const Dims& d = s.in_dims;
        g_.X = d[0];
        g_.Y = d[1];
        g_.B = 1;
        for (size_t k = 3; k < d.size(); k++)
            g_.B *= d[k];
        g_.Cin = d[2];
        g_.Cout = s.out_channels;
        g_.KX = s.kernel[0];
        g_.KY = s.kernel[1];
        g_.px = (g_.KX - 1) / 2;
        g_.py = (g_.KY - 1) / 2;
        // channels-last storage for multi-channel activations: requested by the
        // builder (MoDL denoiser chain) or implied by the tensor-core path
        const bool tc = conv_tc_supported(g_.Cin, g_.Cout, g_.KX, g_.KY);
        const bool chl = s.chlast_hint > 0 || (s.chlast_hint == 0 && (tc || conv_chlast_forced()));
        g_.in_chlast = chl && g_.Cin > 1;
        g_.out_chlast = chl && g_.Cout > 1;
    }
    bool holomorphic() const override { return !t_; }
    Layout act_layout(bool in_side) const
    {
        return (in_side ? g_.in_chlast : g_.out_chlast) ? Layout::CHLAST : Layout::CANON;
    }
    // fwd inputs (x, w) -> y ; transposed inputs (w, y) -> x
    Layout in_layout(int i) const override
    {
        if (!t_)
            return i == 0 ? act_layout(true) : Layout::CANON;
        return i == 1 ? act_layout(false) : Layout::CANON;
    }
    Layout out_layout(int) const override { return act_layout(t_); }

    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool store) override
    {
        if (!t_)
            out[0] = fwd(in[0], in[1]);
        else
            out[0] = bwd_data(in[1], in[0]);
        if (store)
            st_ = in;
        else
            st_.clear();
        bump_generation();
    }
    DArray deriv(int, int i, const DArray& d) override
    {
        require_forward();
        if (!t_)
            return i == 0 ? fwd(d, st_[1]) : fwd(st_[0], d);
        return i == 1 ? bwd_data(d, st_[0]) : bwd_data(st_[1], d);
    }
    DArray adjoint(int, int i, const DArray& g) override
    {
        require_forward();
        if (!t_)
            return i == 0 ? bwd_data(g, st_[1], static_cast<const BnBwdHint*>(input_hint(0))) : bwd_weight(st_[0], g);
        // transposed: wrt y -> conv(g, w); wrt w -> bwd_weight(xin = g, dy = y)
        return i == 1 ? fwd(g, st_[0]) : bwd_weight(g, st_[1]);
    }

private:
    // the Cin-side tensor (x / dx) and the Cout-side tensor (y / dy) in the
    // layouts this node stores them in
    DArray as_in(const DArray& a) const { return a.layout == act_layout(true) ? a : to_layout(a, act_layout(true)); }
    DArray as_out(const DArray& a) const
    {
        return a.layout == act_layout(false) ? a : to_layout(a, act_layout(false));
    }
    DArray fwd(const DArray& x0, const DArray& w) const
    {
        DArray x = as_in(x0);
        Dims od = t_ ? ins_[1] : outs_[0];
        DArray y(od, false, act_layout(false));
        ConvGeom g = g_;
        g.in_tf32 = x.tf32;
        g.real_known = (x.known_real ? 1 : 0) | (w.known_real ? 2 : 0);
        // channel statistics from the tensor-core epilogue (consumed by a BnBlockNode)
        const long ny = 2 * g_.Cout;
        DArray st;
        int st_blocks = 0;
        const long eb = (y.layout == Layout::CHLAST && ny == 128 && conv_bn_fuse()) ? conv_epi_blocks(g_, 0) : 0;
        if (eb > 0) {
            st = DArray(Dims{eb * ny * 2}, false);
            g.stats = reinterpret_cast<double*>(st.data());
            g.stats_blocks = &st_blocks;
        }
        conv_fwd(y.data(), x.data(), w.data(), g);
        y.known_real = x.known_real && w.known_real;
        if (st_blocks > 0) {
            y.chstats = std::make_shared<DArray>(st);
            y.chstats_blocks = st_blocks;
            y.chstats_kind = 1;
        }
        return y;
    }
    // hint: forward state of the batch-norm block that produced x (it consumes
    // dx); the tensor-core epilogue then also emits that block's backward partials
    DArray bwd_data(const DArray& dy0, const DArray& w, const BnBwdHint* hint = nullptr) const
    {
        DArray dy = as_out(dy0);
        Dims xd = t_ ? outs_[0] : ins_[0];
        DArray dx(xd, false, act_layout(true));
        ConvGeom g = g_;
        g.out_tf32 = dy.tf32;
        g.real_known = (dy.known_real ? 4 : 0) | (w.known_real ? 2 : 0);
        DArray part;
        int blocks = 0;
        const long eb = (hint && dx.layout == Layout::CHLAST && 2 * g_.Cin == 128 && conv_bn_fuse())
                            ? conv_epi_blocks(g_, 1)
                            : 0;
        if (eb > 0) {
            part = DArray(Dims{eb * 128 * 3}, false);
            g.bnb = hint;
            g.bnb_part = reinterpret_cast<double*>(part.data());
            g.bnb_blocks = &blocks;
        }
        conv_bwd_data(dx.data(), dy.data(), w.data(), g);
        dx.known_real = dy.known_real && w.known_real;
        if (blocks > 0) {
            dx.chstats = std::make_shared<DArray>(part);
            dx.chstats_blocks = blocks;
            dx.chstats_kind = 2;
            dx.chstats_tag = hint;
        }
        return dx;
    }
    DArray bwd_weight(const DArray& x0, const DArray& dy0) const
    {
        DArray x = as_in(x0), dy = as_out(dy0);
        Dims wd = t_ ? ins_[0] : ins_[1];
        DArray dw(wd, false);
        ConvGeom g = g_;
        g.in_tf32 = x.tf32;
        g.out_tf32 = dy.tf32;
        g.real_known = (x.known_real ? 1 : 0) | (dy.known_real ? 4 : 0);
        conv_bwd_weight(dw.data(), x.data(), dy.data(), g);
        dw.known_real = x.known_real && dy.known_real;
        return dw;
    }
    bool t_;
    ConvGeom g_{};
    std::vector<DArray> st_;
};

// ---------------------------------------------------------------------------
// Fused BatchNorm -> bn_scale TenMul -> BroadcastAdd -> CReLU (train mode) on
// channels-last activations.  Same values and derivatives as the reference
// chain (ops.hpp:1070-1298, 69-118, 153-209, 451-475); 2 HBM passes forward,
// 2 backward.  Rare paths (tangents, statistics-output cotangents) reuse the
// reference-layout kernels.
class BnBlockNode : public Atom {
public:
    BnBlockNode(const Dims& d, bool round_out, bool round_dx, double eps, double mom)
        : Atom("bn_block", {d, sdims(d), sdims(d), sdims(d), sdims(d)}, {sdims(d), sdims(d), d}),
          round_out_(round_out), round_dx_(round_dx), eps_(float(eps)), mom_(float(mom))
    {
        C_ = d[2];
        npix_ = md_size(d) / C_;
        geo_ = IsoGeom{d[0] * d[1], C_, npix_ / (d[0] * d[1])};
        m_ = double(npix_);
    }
    static Dims sdims(Dims d)
    {
        for (size_t k = 0; k < d.size(); k++)
            if (k != size_t(dim_chan))
                d[k] = 1;
        return d;
    }
    Layout in_layout(int i) const override { return i == 0 ? Layout::CHLAST : Layout::CANON; }
    Layout out_layout(int o) const override { return o == 2 ? Layout::CHLAST : Layout::CANON; }
    bool zero_deriv(int o, int i) const override
    {
        if (o == 2)
            return !(i == 0 || i == 3 || i == 4);
        if (o == 0)
            return !(i == 0 || i == 1);
        return !(i == 0 || i == 2);
    }
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool store) override
    {
        const Dims& sd = ins_[1];
        DArray y(ins_[0], false, Layout::CHLAST), mo(sd, false), vo(sd, false);
        DArray mu(sd, false), istd(Dims{C_}, false);
        const bool pre = in[0].chstats && in[0].chstats_kind == 1 && in[0].chstats_blocks > 0;
        bnblock_forward(y.fdata(), mu.data(), istd.fdata(), mo.data(), vo.data(), in[0].fdata(), in[1].data(),
                        in[2].data(), in[3].data(), in[4].data(), npix_, int(C_), eps_, mom_, round_out_,
                        pre ? reinterpret_cast<const double*>(in[0].chstats->data()) : nullptr,
                        pre ? in[0].chstats_blocks : 0);
        y.tf32 = round_out_;
        out[0] = mo;
        out[1] = vo;
        out[2] = y;
        if (store) {
            x_ = in[0];
            g_ = in[3];
            b_ = in[4];
            mu_ = mu;
            istd_ = istd;
            hint_ = BnBwdHint{x_.fdata(), mu_.data(), istd_.fdata(), g_.data(), b_.data(), npix_, int(C_)};
        } else {
            hint_ = BnBwdHint{};
        }
        bump_generation();
    }
    // the producer of y's cotangent (a tensor-core bwd-data conv) may fold the
    // backward reduction pass into its epilogue
    const void* cotangent_hint(int o) const override { return (o == 2 && hint_.x) ? &hint_ : nullptr; }
    void adjoint_all(int o, const DArray& gin, std::vector<DArray>& dx, const std::vector<char>& want) override
    {
        require_forward();
        dx.assign(n_in(), DArray{});
        const Dims& sd = ins_[1];
        if (o == 2) {
            DArray dxx, dg, db;
            if (want[0])
                dxx = DArray(ins_[0], false, Layout::CHLAST);
            if (want[3])
                dg = DArray(sd, false);
            if (want[4])
                db = DArray(sd, false);
            if (!want[0] && !want[3] && !want[4])
                return;
            // the reduction pass always produces both sums; route them to scratch when unwanted
            DArray sg = want[3] ? dg : DArray(sd, false), sb = want[4] ? db : DArray(sd, false);
            const bool pre = gin.chstats && gin.chstats_kind == 2 && gin.chstats_tag == &hint_ && hint_.x
                             && gin.chstats_blocks > 0;
            bnblock_backward(want[0] ? dxx.fdata() : nullptr, sg.data(), sb.data(), gin.fdata(), x_.fdata(),
                             mu_.data(), istd_.fdata(), g_.data(), b_.data(), npix_, int(C_), round_dx_,
                             pre ? reinterpret_cast<const double*>(gin.chstats->data()) : nullptr,
                             pre ? gin.chstats_blocks : 0);
            if (want[0]) {
                dxx.tf32 = round_dx_;
                dx[0] = dxx;
            }
            if (want[3])
                dx[3] = dg;
            if (want[4])
                dx[4] = db;
            return;
        }
        // moving-statistics outputs (ops.hpp:1265-1282)
        const int own = o == 0 ? 1 : 2;
        if (want[own]) {
            DArray t(sd, false);
            launch_scale(t.data(), gin.data(), cfloat{1.f - mom_, 0.f}, t.size());
            dx[own] = t;
        }
        if (want[0]) {
            DArray xc = to_layout(x_, Layout::CANON);
            DArray r(ins_[0], false);
            if (o == 0) { // (mom/m) broadcast(g)
                DArray z(ins_[0], true), t(ins_[0], false);
                launch_stat_add(t.data(), z.data(), gin.data(), geo_);
                launch_scale(r.data(), t.data(), cfloat{float(mom_ / m_), 0.f}, r.size());
            } else { // u * (mom 2 Re(g) / m)
                DArray u = centred(xc), q(sd, false), f(sd, false);
                launch_real(q.data(), gin.data(), q.size());
                launch_scale(f.data(), q.data(), cfloat{float(mom_ * 2.0 / m_), 0.f}, f.size());
                launch_stat_mul(r.data(), u.data(), f.data(), geo_, false);
            }
            dx[0] = to_layout(r, Layout::CHLAST);
        }
    }
    DArray adjoint(int o, int i, const DArray& g) override
    {
        std::vector<char> want(n_in(), 0);
        want[i] = 1;
        std::vector<DArray> dx;
        adjoint_all(o, as_out(o, g), dx, want);
        return dx[i].valid() ? dx[i] : DArray(ins_[i]);
    }
    DArray deriv(int o, int i, const DArray& d0) override
    {
        require_forward();
        const Dims& sd = ins_[1];
        DArray xc = to_layout(x_, Layout::CANON);
        DArray u = centred(xc);
        if (o == 2) {
            // z = g * yhat + beta, yhat = u * istd ; tangent masked by CReLU(z)
            DArray yh(ins_[0], false), t1(ins_[0], false), z(ins_[0], false), dz(ins_[0], false);
            DArray istd_c = istd_complex();
            launch_stat_mul(yh.data(), u.data(), istd_c.data(), geo_, false);
            launch_stat_mul(t1.data(), yh.data(), g_.data(), geo_, false);
            launch_stat_add(z.data(), t1.data(), b_.data(), geo_);
            if (i == 0) {
                DArray dc = to_layout(d0, Layout::CANON), dyh(ins_[0], false);
                bn_train_deriv_x(dyh.data(), dc.data(), u.data(), istd_c.data(), geo_);
                launch_stat_mul(dz.data(), dyh.data(), g_.data(), geo_, false);
            } else if (i == 3) {
                launch_stat_mul(dz.data(), yh.data(), d0.data(), geo_, false);
            } else {
                DArray zero(ins_[0], true);
                launch_stat_add(dz.data(), zero.data(), d0.data(), geo_);
            }
            DArray r(ins_[0], false);
            launch_crelu_mask(r.data(), dz.data(), z.data(), r.size());
            return to_layout(r, Layout::CHLAST);
        }
        DArray r(sd, false);
        if (i != 0) {
            launch_scale(r.data(), d0.data(), cfloat{1.f - mom_, 0.f}, r.size());
            return r;
        }
        DArray dc = to_layout(d0, Layout::CANON);
        if (o == 0) {
            launch_iso_reduce(r.data(), dc.data(), nullptr, geo_.inner, geo_.nstat, geo_.outer, 0, float(mom_ / m_));
        } else {
            DArray p(sd, false), q(sd, false);
            launch_iso_reduce(p.data(), dc.data(), u.data(), geo_.inner, geo_.nstat, geo_.outer, 1, 1.f);
            launch_real(q.data(), p.data(), q.size());
            launch_scale(r.data(), q.data(), cfloat{float(mom_ * 2.0 / m_), 0.f}, r.size());
        }
        return r;
    }

private:
    DArray as_out(int o, const DArray& g) const { return to_layout(g, out_layout(o)); }
    // u = x - mu (reference layout)
    DArray centred(const DArray& xc) const
    {
        DArray nm(ins_[1], false), u(ins_[0], false);
        launch_neg(nm.data(), mu_.data(), nm.size());
        launch_stat_add(u.data(), xc.data(), nm.data(), geo_);
        return u;
    }
    // istd as complex (istd, 0) per channel for the reference-layout kernels
    DArray istd_complex() const
    {
        DArray r(ins_[1], false);
        launch_real_to_complex(r.data(), istd_.fdata(), C_);
        return r;
    }

    bool round_out_, round_dx_;
    float eps_, mom_;
    long C_ = 1, npix_ = 1;
    double m_ = 1;
    IsoGeom geo_{};
    DArray x_, g_, b_, mu_, istd_;
    BnBwdHint hint_{};
};

} // namespace

// ---------------------------------------------------------------------------

NodePtr node_dft(const Dims& d, unsigned long flags, bool inv) { return std::make_shared<DftNode>(d, flags, inv); }
NodePtr node_pad(const Dims& in, const Dims& out, const Dims& corner, bool crop)
{
    return std::make_shared<PadNode>(in, out, corner, crop);
}
NodePtr node_tenmul(const std::string& name, const Dims& iter, const Dims& od, const Dims& so, const Dims& i1,
                    const Dims& s1, const Dims& i2, const Dims& s2)
{
    size_t r = iter.size();
    if (od.size() != r || so.size() != r || i1.size() != r || s1.size() != r || i2.size() != r || s2.size() != r)
        throw ShapeError("tenmul: rank mismatch");
    return std::make_shared<TenMulNode>(name, iter, od, so, i1, s1, i2, s2);
}
NodePtr node_add(const Dims& d, bool sub) { return std::make_shared<AddNode>(d, sub); }
NodePtr node_bcast_add(const Dims& x, const Dims& b) { return std::make_shared<BcastAddNode>(x, b); }
NodePtr node_fork(const Dims& d, int n) { return std::make_shared<ForkNode>(d, n); }
NodePtr node_zconj(const Dims& d) { return std::make_shared<MapNode>(d, MapNode::Conj); }
NodePtr node_zreal(const Dims& d) { return std::make_shared<MapNode>(d, MapNode::Real); }
NodePtr node_real_chan(const Dims& d, int cd) { return std::make_shared<ChanSplitNode>(d, cd, false); }
NodePtr node_chan_cplx(const Dims& d, int cd) { return std::make_shared<ChanSplitNode>(d, cd, true); }
NodePtr node_crelu(const Dims& d) { return std::make_shared<CReluNode>(d); }
NodePtr node_exp_real(const Dims& d) { return std::make_shared<ExpRealNode>(d); }
NodePtr node_mse(const Dims& d) { return std::make_shared<MseNode>(d); }
NodePtr node_batchnorm(const Dims& d, unsigned long flags, bool train, double eps, double mom)
{
    return std::make_shared<BatchNormNode>(d, flags, train, eps, mom);
}
NodePtr node_rbf(const Dims& z, int fd, const std::vector<float>& mu, float sigma)
{
    return std::make_shared<RbfNode>(z, fd, mu, sigma);
}
bool bnblock_supported(long channels) { return channels >= 2 && channels <= 256 && 256 % channels == 0; }
NodePtr node_bnblock(const Dims& dims, bool round_out, bool round_dx, double eps, double mom)
{
    if (!bnblock_supported(dims.at(dim_chan)))
        throw ConfigError("bn_block: channel count must be >= 2 and divide 256");
    return std::make_shared<BnBlockNode>(dims, round_out, round_dx, eps, mom);
}
NodePtr node_sense_normal(const SenseDims& sd) { return std::make_shared<SenseNormalNode>(sd, false); }
NodePtr node_sense_normal_lambda(const SenseDims& sd) { return std::make_shared<SenseNormalNode>(sd, true); }
NodePtr node_sense_adjoint(const SenseDims& sd) { return std::make_shared<SenseAdjointNode>(sd); }
NodePtr node_sense_forward(const SenseDims& sd) { return std::make_shared<SenseForwardNode>(sd); }
NodePtr node_inverse(const Nlop& s, long max_iter, double tol)
{
    return std::make_shared<InverseNode>(s, max_iter, tol);
}

// ---------------------------------------------------------------------------
// CheckpointNode (nlop.hpp:439-513).  Recompute-for-memory: the
// inner nodes run with store = false, so only the container's inputs stay
// alive between forward and backward.  The hot path has no stochastic nodes,
// so there are no RNG counters to rewind.
class CheckpointNode : public Node {
public:
    explicit CheckpointNode(Nlop inner) : Node("checkpoint", dims_in(inner), dims_out(inner)), inner_(std::move(inner))
    {
    }
    void forward(const std::vector<DArray>& in, std::vector<DArray>& out, bool) override
    {
        saved_in_ = in;
        out = inner_.run_forward(in, false);
        bump_generation();
    }
    DArray deriv(int o, int i, const DArray& dx) override
    {
        reexecute();
        return inner_.derivative(o, i, dx);
    }
    DArray adjoint(int o, int i, const DArray& dy) override
    {
        reexecute();
        return inner_.adjoint_derivative(o, i, dy);
    }
    void adjoint_all(int o, const DArray& dy, std::vector<DArray>& dx, const std::vector<char>& want) override
    {
        reexecute();
        dx = inner_.adjoint_all(o, dy, want);
    }
    long reexecutions() const { return reexec_; }

private:
    static std::vector<Dims> dims_in(const Nlop& f)
    {
        std::vector<Dims> d;
        for (int i = 0; i < f.n_in(); i++)
            d.push_back(f.in_dims(i));
        return d;
    }
    static std::vector<Dims> dims_out(const Nlop& f)
    {
        std::vector<Dims> d;
        for (int o = 0; o < f.n_out(); o++)
            d.push_back(f.out_dims(o));
        return d;
    }
    void reexecute()
    {
        require_forward();
        inner_.apply(saved_in_);
        reexec_++;
    }

    Nlop inner_;
    std::vector<DArray> saved_in_;
    long reexec_ = 0;
};

NodePtr node_checkpoint(const Nlop& inner) { return std::make_shared<CheckpointNode>(inner); }

long checkpoint_reexecutions(const Nlop& h)
{
    for (auto& n : h.nodes())
        if (auto* p = dynamic_cast<CheckpointNode*>(n.get()))
            return p->reexecutions();
    return -1;
}

bool inverse_status(const Nlop& h, long* iterations, double* rel, int* conv)
{
    for (auto& n : h.nodes())
        if (auto* p = dynamic_cast<InverseNode*>(n.get())) {
            auto st = p->status();
            *iterations = st.iterations;
            *rel = st.rel_residual;
            *conv = st.converged ? 1 : 0;
            return true;
        }
    return false;
}

Dims ConvSpec::weight_dims() const
{
    Dims w = kernel;
    w.push_back(in_dims.at(chan_dim));
    w.push_back(out_channels);
    return w;
}

Dims ConvSpec::out_dims() const
{
    Dims out = in_dims;
    for (size_t a = 0; a < axes.size(); a++) {
        long n = in_dims[axes[a]];
        if (!pad_same) {
            if (kernel[a] > n)
                throw ShapeError("conv: kernel larger than input on axis " + std::to_string(axes[a]));
            out[axes[a]] = n - kernel[a] + 1;
        }
    }
    out[chan_dim] = out_channels;
    return out;
}

namespace {

// conv_tenmul (nn.hpp:305-337): the TenMul wiring of a valid cross-correlation
NodePtr conv_tenmul_node(const std::string& name, const ConvSpec& spec, const Dims& in_dims, const Dims& out_dims)
{
    Dims w_dims = spec.weight_dims();
    Dims si = default_strides(in_dims), so = default_strides(out_dims), sw = default_strides(w_dims);
    Dims iter, to, ti, tw;
    auto push = [&](long n, long o, long i, long w) {
        iter.push_back(n);
        to.push_back(o);
        ti.push_back(i);
        tw.push_back(w);
    };
    for (int d = 0; d < int(in_dims.size()); d++) {
        auto ax = std::find(spec.axes.begin(), spec.axes.end(), d);
        if (ax != spec.axes.end()) {
            size_t a = ax - spec.axes.begin();
            push(out_dims[d], so[d], si[d], 0);
            push(spec.kernel[a], 0, si[d], sw[a]);
        } else if (d == spec.chan_dim) {
            push(in_dims[d], 0, si[d], sw[spec.axes.size()]);
            push(spec.out_channels, so[d], 0, sw[spec.axes.size() + 1]);
        } else {
            push(in_dims[d], so[d], si[d], 0);
        }
    }
    if (spec.transposed)
        return std::make_shared<TenMulNode>(name, iter, in_dims, ti, out_dims, to, w_dims, tw);
    return std::make_shared<TenMulNode>(name, iter, out_dims, to, in_dims, ti, w_dims, tw);
}

} // namespace

Nlop conv_core(const std::string& name, const ConvSpec& spec)
{
    bool fast = spec.pad_same && spec.axes.size() == 2 && spec.axes[0] == 0 && spec.axes[1] == 1
                && spec.chan_dim == 2 && spec.kernel[0] <= 11 && spec.kernel[1] <= 11;
    if (fast)
        return Nlop(std::make_shared<ConvNode>(name + (spec.transposed ? "_convT" : "_conv"), spec,
                                               spec.transposed));
    // generic reference wiring (nn.hpp:361-413) on the generic TenMul kernel
    Dims padded = spec.in_dims;
    Dims corner(spec.in_dims.size(), 0);
    if (spec.pad_same)
        for (size_t a = 0; a < spec.axes.size(); a++) {
            padded[spec.axes[a]] += spec.kernel[a] - 1;
            corner[spec.axes[a]] = (spec.kernel[a] - 1) / 2;
        }
    Dims conv_out = spec.out_dims();
    if (spec.pad_same)
        for (size_t a = 0; a < spec.axes.size(); a++)
            conv_out[spec.axes[a]] = padded[spec.axes[a]] - spec.kernel[a] + 1;
    ConvSpec vspec = spec;
    vspec.in_dims = padded;
    if (!spec.transposed) {
        auto core = Nlop(conv_tenmul_node(name + "_conv", vspec, padded, conv_out));
        if (!spec.pad_same)
            return core;
        auto pad = Nlop(node_pad(spec.in_dims, padded, corner, false));
        return link(combine(pad, core), 0, 1);
    }
    auto scatter = Nlop(conv_tenmul_node(name + "_convT", vspec, padded, conv_out));
    auto conjw = Nlop(node_zconj(spec.weight_dims()));
    auto core = link(combine(conjw, scatter), 0, 2);
    if (spec.pad_same)
        core = chain(core, Nlop(node_pad(spec.in_dims, padded, corner, true)));
    return core;
}

} // namespace mdnn
