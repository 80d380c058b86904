// Reference-side splice test (test infrastructure; built by oracle/Makefile
// against the unmodified reference headers, run by tests/test_gpu_adapter.py).
//
// The B200 operator S = A^H A + lambda (mdnn_modl_normal_plus_lambda) is
// wrapped as a reference NlopNode (include/mdnn_b200_node.hpp) and spliced
// into reference graphs, each compared with the same graph built from the
// unmodified reference operator (recon.hpp:807-820):
//   1. S alone: apply, adjoint_all (all inputs), derivative wrt x
//   2. the reference InverseNode (make_inverse_nlop, recon.hpp:211-329) whose
//      CG runs on the host and calls the B200 S every iteration: apply and the
//      adjoint wrt y and coils
//   3. a reference chain CReLU(S(x, ...)) (nlop.hpp:343, ops.hpp:1463)
// Prints one line per check and "SPLICE OK" at the end; exit code 1 on a miss.
#include <mdnn/recon.hpp>
#include <mdnn/simulate.hpp>

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "mdnn_b200_node.hpp"

using namespace mdnn;

namespace {

void fill(MdArray<float>& a, uint64_t seed, float amp)
{
    uint64_t s = seed * 0x9E3779B97F4A7C15ULL + 1;
    auto next = [&] {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        return float((s >> 11) * (1.0 / 9007199254740992.0)) * 2.f - 1.f;
    };
    auto* v = a.data();
    for (long k = 0; k < md_size(a.dims()); k++) {
        const float re = next(), im = next();
        v[k] = std::complex<float>(amp * re, amp * im);
    }
}

double rel(const MdArray<float>& a, const MdArray<float>& b)
{
    double d = 0, n = 0;
    const auto *x = a.data(), *y = b.data();
    for (long k = 0; k < md_size(b.dims()); k++) {
        d += std::norm(std::complex<double>(x[k]) - std::complex<double>(y[k]));
        n += std::norm(std::complex<double>(y[k]));
    }
    return n > 0 ? std::sqrt(d / n) : std::sqrt(d);
}

int fails = 0;
void expect(const char* what, double err, double tol)
{
    std::printf("%-44s rel-L2 %.3e (tol %.0e)%s\n", what, err, tol, err <= tol ? "" : "  FAIL");
    fails += !(err <= tol);
}

} // namespace

int main()
{
    try {
        b200_check(mdnn_set_device(0));
        SenseDims sd;
        sd.x = 16;
        sd.y = 368; // 16 x 23: the persistent rank A^H A kernel
        sd.coils = 4;
        sd.batch = 2;
        Model<float> ref = detail::modl_normal_plus_lambda<float>(sd);
        mdnn_sense_dims csd{sd.x, sd.y, sd.coils, sd.maps, sd.batch};
        mdnn_model* bm = mdnn_modl_normal_plus_lambda(&csd);
        if (!bm)
            throw Error(mdnn_last_error());
        if (mdnn_model_n_args(bm) != int(ref.args.size()))
            throw Error("argument count differs");
        for (int i = 0; i < int(ref.args.size()); i++)
            if (ref.args[i].name != mdnn_model_arg_name(bm, i))
                throw Error("argument " + std::to_string(i) + " differs: " + ref.args[i].name);
        Nlop<float> sb(std::make_shared<B200Node>(mdnn_model_nlop(bm), "b200_normal"));
        mdnn_model_free(bm);
        Nlop<float>& sr = ref.op;

        // inputs in the reference's argument order: x, coils, pattern, lambda
        std::vector<MdArray<float>> in;
        for (int i = 0; i < sr.n_in(); i++)
            in.emplace_back(sr.in_dims(i));
        fill(in[0], 1, 1.f);
        fill(in[1], 2, 0.5f);
        {
            MdArray<float> p = make_pattern<float>(sd.y, 4, 28);
            std::copy(p.data(), p.data() + md_size(p.dims()), in[2].data());
        }
        in[3].data()[0] = std::complex<float>(0.05f, 0.f);

        // 1. S alone
        auto yr = sr.apply(in), yb = sb.apply(in);
        expect("S apply", rel(yb[0], yr[0]), 1e-5);
        MdArray<float> dy(sr.out_dims(0));
        fill(dy, 3, 1.f);
        auto ar = sr.adjoint_all(0, dy), ab = sb.adjoint_all(0, dy);
        expect("S adjoint wrt x", rel(ab[0], ar[0]), 1e-5);
        expect("S adjoint wrt coils", rel(ab[1], ar[1]), 1e-5);
        expect("S adjoint wrt lambda", rel(ab[3], ar[3]), 1e-5);
        MdArray<float> dx(sr.in_dims(0));
        fill(dx, 4, 1.f);
        expect("S derivative wrt x", rel(sb.derivative(0, 0, dx), sr.derivative(0, 0, dx)), 1e-5);

        // 2. reference InverseNode (host CG) over the B200 S
        Nlop<float> ir = make_inverse_nlop<float>(sr, 10, 1e-7), ib = make_inverse_nlop<float>(sb, 10, 1e-7);
        auto xr = ir.apply(in), xb = ib.apply(in);
        expect("inverse(S) apply (reference CG, B200 S)", rel(xb[0], xr[0]), 1e-5);
        auto gr = ir.adjoint_all(0, dy), gb = ib.adjoint_all(0, dy);
        expect("inverse(S) adjoint wrt y", rel(gb[0], gr[0]), 1e-5);
        expect("inverse(S) adjoint wrt coils", rel(gb[1], gr[1]), 1e-5);

        // 3. reference chain: CReLU after S
        Nlop<float> cr = chain(sr, nlop_activation<float>("crelu", sr.out_dims(0)));
        Nlop<float> cb = chain(sb, nlop_activation<float>("crelu", sr.out_dims(0)));
        expect("chain(S, crelu) apply", rel(cb.apply(in)[0], cr.apply(in)[0]), 1e-5);
        auto hr = cr.adjoint_all(0, dy), hb = cb.adjoint_all(0, dy);
        expect("chain(S, crelu) adjoint wrt x", rel(hb[0], hr[0]), 1e-5);

        // errors cross the boundary as reference exceptions
        bool caught = false;
        try {
            Nlop<float> fresh(std::make_shared<B200Node>(mdnn_model_nlop(mdnn_modl_normal_plus_lambda(&csd))));
            fresh.nodes()[0]->adjoint(0, 0, dy, dx);
        } catch (const StaleDerivativeError&) {
            caught = true;
        }
        std::printf("%-44s %s\n", "StaleDerivativeError before forward", caught ? "raised" : "NOT RAISED  FAIL");
        fails += !caught;
    } catch (const std::exception& e) {
        std::printf("exception: %s\n", e.what());
        return 1;
    }
    if (fails)
        return 1;
    std::printf("SPLICE OK\n");
    return 0;
}
