"""GPU parity: DFT, SENSE operator, normal operator, CG and the InverseNode
against the reference CPU implementation (oracle/_ref) on identical inputs.

Tolerance: rel-L2 <= 1e-5 for the fp32 SENSE/CG path (BASELINE.json
north_star; SURVEY §8c per-node protocol).
"""
import ctypes as C

import numpy as np
import pytest

from paper_2202_14005_b200.capi import MdnnError
from paper_2202_14005_b200.mdnn import Model, Nlop, sense_dims
from util import (coil_dims, crand, d16, image_dims, kspace_dims, pattern_dims, rel_l2, sim_data)

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.mark.parametrize("dims,flags", [
    ((12,), 1), ((5, 7), 3), ((368,), 1), ((320, 4), 1), ((8, 368, 3), 2), ((16, 23, 2), 3),
    ((64, 40, 1, 3), 3), ((30, 11, 13), 7), ((128, 128), 3), ((640, 2), 1),
])
@pytest.mark.parametrize("inverse", [False, True])
def test_dft_matches_reference(gpu, ref, dims, flags, inverse):
    rng = np.random.default_rng(len(dims) * 100 + flags)
    x = crand(rng, dims)
    outs = []
    for lib in (gpu, ref):
        y = np.zeros(dims, dtype=np.complex64, order="F")
        lib.check(lib.so.mdnn_dft(C.byref(lib.arr(x)), flags, int(inverse), C.byref(lib.arr(y))))
        outs.append(y)
    assert rel_l2(outs[0], outs[1]) <= TOL


def _sense_call(lib, name, coils, pat, inp, out_dims, lam=None):
    out = np.zeros(out_dims, dtype=np.complex64, order="F")
    fn = getattr(lib.so, name)
    if lam is None:
        lib.check(fn(C.byref(lib.arr(coils)), C.byref(lib.arr(pat)), C.byref(lib.arr(inp)), C.byref(lib.arr(out))))
    else:
        lib.check(fn(C.byref(lib.arr(coils)), C.byref(lib.arr(pat)), C.c_float(lam), C.byref(lib.arr(inp)),
                     C.byref(lib.arr(out))))
    return out


SHAPES = [(32, 40, 4, 1), (128, 128, 8, 1), (64, 46, 3, 2), (40, 368, 5, 1)]


@pytest.mark.parametrize("X,Y,NC,B", SHAPES)
def test_sense_forward_adjoint_normal(gpu, ref, X, Y, NC, B):
    ph, cm, pat = sim_data(ref, X, Y, NC, B)
    rng = np.random.default_rng(X + Y)
    k = crand(rng, kspace_dims(X, Y, NC, B))
    for name, inp, od, lam in [("mdnn_sense_forward", ph, kspace_dims(X, Y, NC, B), None),
                               ("mdnn_sense_adjoint", k, image_dims(X, Y, B), None),
                               ("mdnn_sense_normal", ph, image_dims(X, Y, B), 0.05)]:
        g = _sense_call(gpu, name, cm, pat, inp, od, lam)
        r = _sense_call(ref, name, cm, pat, inp, od, lam)
        assert rel_l2(g, r) <= TOL, name


@pytest.mark.parametrize("X,Y,NC,B", SHAPES)
def test_cg_normal_solve(gpu, ref, X, Y, NC, B):
    ph, cm, pat = sim_data(ref, X, Y, NC, B)
    b = _sense_call(ref, "mdnn_sense_adjoint", cm, pat,
                    _sense_call(ref, "mdnn_sense_forward", cm, pat, ph, kspace_dims(X, Y, NC, B)),
                    image_dims(X, Y, B))
    res = []
    for lib in (gpu, ref):
        x = np.zeros(image_dims(X, Y, B), dtype=np.complex64, order="F")
        it, rr = C.c_long(), C.c_double()
        lib.check(lib.so.mdnn_cg_normal_solve(C.byref(lib.arr(cm)), C.byref(lib.arr(pat)), C.c_float(0.05),
                                              C.byref(lib.arr(b)), 10, 0.0, C.byref(lib.arr(x)), C.byref(it),
                                              C.byref(rr)))
        res.append((x, it.value, rr.value))
    assert res[0][1] == res[1][1] == 10
    assert rel_l2(res[0][0], res[1][0]) <= TOL
    assert abs(res[0][2] - res[1][2]) <= 1e-3 * res[1][2] + 1e-9


def test_cg_converges_early_like_reference(gpu, ref):
    X, Y, NC = 24, 20, 4
    ph, cm, pat = sim_data(ref, X, Y, NC, 1, accel=1, acl=Y)  # fully sampled: A^H A = I
    res = []
    for lib in (gpu, ref):
        x = np.zeros(image_dims(X, Y), dtype=np.complex64, order="F")
        it, rr = C.c_long(), C.c_double()
        lib.check(lib.so.mdnn_cg_normal_solve(C.byref(lib.arr(cm)), C.byref(lib.arr(pat)), C.c_float(1.0),
                                              C.byref(lib.arr(ph)), 30, 1e-6, C.byref(lib.arr(x)), C.byref(it),
                                              C.byref(rr)))
        res.append((x, it.value))
    # (A^H A + 1) = 2 I: converges after one iteration, x = b / 2
    assert res[0][1] == res[1][1]
    assert rel_l2(res[0][0], ph / 2) <= TOL


def _fragment(lib, kind, sd):
    return {"normal": Model.sense_normal_fragment, "adjoint": Model.sense_adjoint_fragment,
            "normal_lambda": Model.modl_normal_plus_lambda}[kind](lib, sd)


@pytest.mark.parametrize("kind", ["normal", "adjoint", "normal_lambda"])
def test_sense_fragments_apply_derivative_adjoint(gpu, ref, kind):
    X, Y, NC, B = 32, 24, 3, 2
    ph, cm, pat = sim_data(ref, X, Y, NC, B)
    sd = sense_dims(X, Y, NC, 1, B)
    mg, mr = _fragment(gpu, kind, sd), _fragment(ref, kind, sd)
    assert mg.arg_names == mr.arg_names
    ng, nr = mg.nlop, mr.nlop
    rng = np.random.default_rng(7)
    ins = []
    for i, name in enumerate(mr.arg_names):
        dims = nr.in_dims(i)
        if name == "pattern":
            ins.append(pat)
        elif name == "coils":
            ins.append(cm)
        elif name == "lambda":
            ins.append(np.full(dims, 0.05, dtype=np.complex64, order="F"))
        else:
            ins.append(crand(rng, dims))
    og, orf = ng.apply(ins), nr.apply(ins)
    assert rel_l2(og[0], orf[0]) <= TOL
    # tangents wrt every input
    for i in range(nr.n_in):
        dx = crand(rng, nr.in_dims(i))
        assert rel_l2(ng.derivative(0, i, dx), nr.derivative(0, i, dx)) <= TOL, (kind, "deriv", i)
    dy = crand(rng, nr.out_dims(0))
    ag, ar = ng.adjoint_all(0, dy), nr.adjoint_all(0, dy)
    for i in range(nr.n_in):
        assert rel_l2(ag[i], ar[i]) <= TOL, (kind, "adjoint", i, mr.arg_names[i])


def test_inverse_node_forward_and_adjoint(gpu, ref):
    X, Y, NC, B = 32, 40, 4, 2
    ph, cm, pat = sim_data(ref, X, Y, NC, B)
    sd = sense_dims(X, Y, NC, 1, B)
    invs = [Model.modl_normal_plus_lambda(lib, sd).nlop.inverse(10, 0.0) for lib in (gpu, ref)]
    rng = np.random.default_rng(3)
    y = crand(rng, image_dims(X, Y, B))
    lam = np.full(d16(), 0.05, dtype=np.complex64, order="F")
    ins = [y, cm, pat, lam]
    outs = [n.apply(ins)[0] for n in invs]
    assert rel_l2(outs[0], outs[1]) <= TOL
    st = [n.cg_status() for n in invs]
    assert st[0][0] == st[1][0]
    dy = crand(rng, image_dims(X, Y, B))
    adj = [n.adjoint_all(0, dy) for n in invs]
    for i in (0, 1, 2, 3):
        assert rel_l2(adj[0][i], adj[1][i]) <= TOL, i
    # tangent wrt y and lambda
    for i, dx in ((0, crand(rng, image_dims(X, Y, B))), (3, np.full(d16(), 0.01, np.complex64, order="F"))):
        assert rel_l2(invs[0].derivative(0, i, dx), invs[1].derivative(0, i, dx)) <= TOL


def test_sense_normal_y_only_at_target_shape(gpu, ref):
    """C2 geometry (320 x 368 x 15 coils), fused single-pass y-only kernel."""
    X, Y, NC = 320, 368, 15
    ph, cm, pat = sim_data(ref, X, Y, NC, 1)
    g = _sense_call(gpu, "mdnn_sense_normal", cm, pat, ph, image_dims(X, Y), 0.05)
    r = _sense_call(ref, "mdnn_sense_normal", cm, pat, ph, image_dims(X, Y), 0.05)
    assert rel_l2(g, r) <= TOL


@pytest.mark.parametrize("entry", ["normal", "cg", "forward"])
def test_nonbinary_pattern_is_a_config_error(gpu, ref, entry):
    """recon.hpp:67-77: a sampling pattern with a value other than 0 or 1 is a
    ConfigError (code 4) with the reference's message, on every standalone SENSE
    entry point (the product checks it on the device and raises at the call's
    closing synchronisation); the library stays usable afterwards."""
    X, Y, NC = 16, 12, 3
    ph, cm, pat = sim_data(ref, X, Y, NC, 1)
    bad = pat.copy(order="F")
    bad.reshape(-1, order="F")[3] = 0.5
    for lib in (gpu, ref):
        for p, ok in ((bad, False), (pat, True)):
            if entry == "normal":
                out = np.zeros(image_dims(X, Y), dtype=np.complex64, order="F")
                call = lambda: lib.so.mdnn_sense_normal(C.byref(lib.arr(cm)), C.byref(lib.arr(p)), C.c_float(0.1),  # noqa: E731
                                                        C.byref(lib.arr(ph)), C.byref(lib.arr(out)))
            elif entry == "cg":
                out = np.zeros(image_dims(X, Y), dtype=np.complex64, order="F")
                it, rr = C.c_long(), C.c_double()
                call = lambda: lib.so.mdnn_cg_normal_solve(C.byref(lib.arr(cm)), C.byref(lib.arr(p)),  # noqa: E731
                                                           C.c_float(0.1), C.byref(lib.arr(ph)), 3, C.c_double(0.0),
                                                           C.byref(lib.arr(out)), C.byref(it), C.byref(rr))
            else:
                out = np.zeros(kspace_dims(X, Y, NC), dtype=np.complex64, order="F")
                call = lambda: lib.so.mdnn_sense_forward(C.byref(lib.arr(cm)), C.byref(lib.arr(p)),  # noqa: E731
                                                         C.byref(lib.arr(ph)), C.byref(lib.arr(out)))
            if ok:
                lib.check(call())
            else:
                with pytest.raises(MdnnError) as e:
                    lib.check(call())
                assert e.value.code == 4
                assert "binary" in str(e.value)
