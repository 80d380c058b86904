"""CPU-only: pin the oracles.

* the numpy restatement (oracle/restate.py) against the compiled reference
  (oracle/_ref/libmdnn_ref64.so, R = double) at 1e-9..1e-12;
* both against the committed golden vectors (tests/golden/*.npz, produced by
  tests/golden/make_golden.py from the fp32 reference);
* the reference's own known answers (test_fft.cpp:43-64 naive DFT, SPEC.md
  examples: unitary A => A^H A = I, CG on 2I gives b/2, parameter counts).
"""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import REPO
from paper_2202_14005_b200.mdnn import ARG_DATA, Model, Nlop
from util import coil_dims, crand, d16, image_dims, kspace_dims, pattern_dims, rel_l2, sim_data

import sys
sys.path.insert(0, os.path.join(REPO, "oracle"))
import restate  # noqa: E402  (test oracle)

GOLDEN = os.path.join(REPO, "tests", "golden")


def _call(lib, name, *args):
    getattr(lib.so, name)(*args)


def _sense(lib, name, coils, pat, inp, od, lam=None):
    out = np.zeros(od, dtype=np.complex64, order="F")
    fn = getattr(lib.so, name)
    if lam is None:
        lib.check(fn(C.byref(lib.arr(coils)), C.byref(lib.arr(pat)), C.byref(lib.arr(inp)), C.byref(lib.arr(out))))
    else:
        lib.check(fn(C.byref(lib.arr(coils)), C.byref(lib.arr(pat)), C.c_float(lam), C.byref(lib.arr(inp)),
                     C.byref(lib.arr(out))))
    return out


@pytest.mark.parametrize("n", [4, 6, 8, 12, 16, 5, 7, 9])
def test_restated_dft_matches_naive(n):
    # reference test_fft.cpp:43-64: naive O(N^2) unitary DFT at 1e-12 (double)
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    k = np.arange(n)
    naive = np.exp(-2j * np.pi * np.outer(k, k) / n) @ x / np.sqrt(n)
    assert np.max(np.abs(restate.dft(x, 1) - naive)) < 1e-12
    assert np.max(np.abs(restate.dft(restate.dft(x, 1), 1, inverse=True) - x)) < 1e-12


@pytest.mark.parametrize("dims,flags", [((12,), 1), ((5, 7, 2), 3), ((23, 16), 2)])
def test_restated_dft_matches_reference(ref64, dims, flags):
    x = crand(np.random.default_rng(1), dims)
    y = np.zeros(dims, dtype=np.complex64, order="F")
    ref64.check(ref64.so.mdnn_dft(C.byref(ref64.arr(x)), flags, 0, C.byref(ref64.arr(y))))
    assert rel_l2(restate.dft(x, flags), y) < 1e-6  # float output of the f64 reference


def test_restated_sense_matches_reference(ref64):
    X, Y, NC, B = 12, 10, 3, 2
    ph, cm, pat = sim_data(ref64, X, Y, NC, B, accel=2, acl=2)
    k = crand(np.random.default_rng(2), kspace_dims(X, Y, NC, B))
    assert rel_l2(restate.sense_forward(ph, cm, pat), _sense(ref64, "mdnn_sense_forward", cm, pat, ph,
                                                              kspace_dims(X, Y, NC, B))) < 1e-6
    assert rel_l2(restate.sense_adjoint(k, cm, pat), _sense(ref64, "mdnn_sense_adjoint", cm, pat, k,
                                                             image_dims(X, Y, B))) < 1e-6
    assert rel_l2(restate.sense_normal(ph, cm, pat, 0.05), _sense(ref64, "mdnn_sense_normal", cm, pat, ph,
                                                                   image_dims(X, Y, B), 0.05)) < 1e-6


def test_spec_examples_sense_and_cg(ref):
    # unit map + full pattern => A^H A = I; A = 0, lam = 2 => x = b/2
    X, Y = 8, 6
    cm = np.zeros(coil_dims(X, Y, 1), dtype=np.complex64, order="F") + 1
    pat = np.ones(pattern_dims(Y), dtype=np.complex64, order="F")
    x = crand(np.random.default_rng(3), image_dims(X, Y))
    assert rel_l2(_sense(ref, "mdnn_sense_normal", cm, pat, x, image_dims(X, Y), 0.0), x) < 1e-6
    assert rel_l2(restate.sense_normal(x, cm, pat), x) < 1e-12
    zero = np.zeros(pattern_dims(Y), dtype=np.complex64, order="F")
    xs, it = restate.cg_solve(lambda v: restate.sense_normal(v, cm, zero, 2.0), x.astype(np.complex128), 10, 1e-9)
    assert rel_l2(xs, x / 2) < 1e-12


def test_restated_cg_matches_reference(ref64):
    X, Y, NC = 12, 10, 3
    ph, cm, pat = sim_data(ref64, X, Y, NC, 1, accel=3, acl=2)
    b = restate.sense_adjoint(restate.sense_forward(ph, cm, pat), cm, pat)
    xs, it = restate.cg_solve(lambda v: restate.sense_normal(v, cm, pat, 0.05), b, 10, 0.0, fp32_scalars=False)
    out = np.zeros(image_dims(X, Y), dtype=np.complex64, order="F")
    bb = np.asfortranarray(b.astype(np.complex64))
    ni, rr = C.c_long(), C.c_double()
    ref64.check(ref64.so.mdnn_cg_normal_solve(C.byref(ref64.arr(cm)), C.byref(ref64.arr(pat)), C.c_float(0.05),
                                              C.byref(ref64.arr(bb)), 10, 0.0, C.byref(ref64.arr(out)),
                                              C.byref(ni), C.byref(rr)))
    assert it == ni.value == 10
    assert rel_l2(xs, out) < 1e-6


def test_restated_conv_and_bn_match_reference(ref64):
    rng = np.random.default_rng(4)
    in_dims = list(d16(9, 7, 3))
    in_dims[15] = 2
    m = Model.conv_layer(ref64, "c", in_dims, (3, 3), 4)
    n = m.nlop
    x, w = crand(rng, n.in_dims(0)), crand(rng, n.in_dims(1))
    assert rel_l2(restate.conv_same(x, w), n.apply([x, w])[0]) < 1e-6
    mt = Model.conv_layer(ref64, "c", in_dims, (3, 3), 4, transposed=True)
    nt = mt.nlop
    y = crand(rng, nt.in_dims(1))
    assert rel_l2(restate.conv_transposed_same(y, w), nt.apply([w, y])[0]) < 1e-6
    bd = list(d16(9, 7, 4))
    bd[15] = 2
    bn = Nlop.batchnorm(ref64, bd, (1 << 0) | (1 << 1) | (1 << 15), True)
    xb = crand(rng, bd)
    z = np.zeros(bn.in_dims(1), dtype=np.complex64, order="F")
    o = np.ones(bn.in_dims(2), dtype=np.complex64, order="F")
    yb, _, _ = restate.batchnorm_train(xb.astype(np.complex128), (0, 1, 15))
    assert rel_l2(yb, bn.apply([xb, z, o])[0]) < 1e-6


def _model_inputs(lib, m, X, Y, NC, B, seed=42, rbf=False):
    ph, cm, pat = sim_data(lib, X, Y, NC, B, accel=3, acl=2)
    ks = restate.sense_forward(ph, cm, pat).astype(np.complex64)
    ks = np.asfortranarray(ks)
    data = {"kspace": ks, "coils": cm, "pattern": pat}
    w = m.init_weights(seed)
    if rbf:
        r = np.random.default_rng(7)
        for k in w:
            if k.endswith("_rbf_w"):
                w[k] = np.asfortranarray(r.uniform(-0.2, 0.2, w[k].shape).astype(np.complex64))
    ins = [data[a] if kind == ARG_DATA else w[a] for a, kind, _ in m.args]
    return data, w, ins


def test_fixed_modl_builder_implements_eq10(ref64):
    """The re-assembled MoDL graph (oracle shim) equals the paper's update
    equation restated independently in numpy."""
    X, Y, NC, B = 10, 8, 2, 2
    cfg = dict(iterations=2, layers=3, filters=3, cg_iter=4, cg_tol=0.0, im_x=X, im_y=Y, coils=NC, batch=B)
    m = Model.modl(ref64, **cfg)
    data, w, ins = _model_inputs(ref64, m, X, Y, NC, B)
    out = m.nlop.apply(ins)[m.output_index("out")]
    wd = {k: v.astype(np.complex128) for k, v in w.items()}
    exp = restate.modl_forward(data["kspace"], data["coils"], data["pattern"], wd, T=2, L=3, cg_iter=4, cg_tol=0.0)
    assert rel_l2(out, exp) < 1e-6


def test_fixed_varnet_builder_implements_eq9(ref64):
    X, Y, NC, B = 10, 8, 2, 1
    cfg = dict(iterations=2, filters=3, kernel=3, rbf=5, im_x=X, im_y=Y, coils=NC, batch=B)
    m = Model.varnet(ref64, **cfg)
    data, w, ins = _model_inputs(ref64, m, X, Y, NC, B, rbf=True)
    out = m.nlop.apply(ins)[0]
    wd = {k: v.astype(np.complex128) for k, v in w.items()}
    exp = restate.varnet_forward(data["kspace"], data["coils"], data["pattern"], wd, T=2, n_rbf=5)
    assert rel_l2(out, exp) < 1e-6


@pytest.mark.parametrize("name", sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))
                         if os.path.isdir(GOLDEN) else [])
def test_restatement_against_golden(name):
    g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    kind = str(g["kind"])
    if kind == "sense_normal":
        got = restate.sense_normal(g["x"], g["coils"], g["pattern"], float(g["lam"]))
    elif kind == "sense_adjoint":
        got = restate.sense_adjoint(g["y"], g["coils"], g["pattern"])
    elif kind == "dft":
        got = restate.dft(g["x"], int(g["flags"]), bool(g["inverse"]))
    elif kind == "conv":
        got = restate.conv_same(g["x"], g["w"])
    elif kind == "cg":
        got, _ = restate.cg_solve(lambda v: restate.sense_normal(v, g["coils"], g["pattern"], float(g["lam"])),
                                  g["b"].astype(np.complex128), int(g["iters"]), 0.0)
    else:
        pytest.skip(kind)
    assert rel_l2(got, g["out"]) < float(g["tol"])
