"""CheckpointNode (nlop.hpp:439-522), mirroring test_nlop.cpp:300-336: the
checkpointed graph reproduces the plain graph bitwise (values, adjoint and
tangent), counts one re-execution per derivative batch, and refuses
derivatives before a forward (StaleDerivativeError).  CPU cases run the
reference shim; GPU cases run the product and compare with the reference."""
import numpy as np
import pytest

from paper_2202_14005_b200.capi import MdnnError
from paper_2202_14005_b200.mdnn import Model, Nlop, sense_dims
from util import crand, d16, image_dims, rel_l2, sim_data


def _square_crelu_dft(lib, n=4):
    d = (n,)
    one = (1,)
    sq = Nlop.tenmul(lib, d, d, one, d, one, d, one).duplicate(0, 1)   # x * x
    return sq.chain(Nlop.unary(lib, "crelu", d)).chain(Nlop.dft(lib, d, 1))


def _check(lib, build, x, dy):
    plain, wrapped0 = build(lib), build(lib)
    wrapped = wrapped0.checkpoint()
    assert wrapped.reexecutions() == 0
    y1, y2 = plain.apply([x])[0], wrapped.apply([x])[0]
    assert np.array_equal(y1, y2)
    assert wrapped.reexecutions() == 0
    g1, g2 = plain.adjoint_all(0, dy)[0], wrapped.adjoint_all(0, dy)[0]
    assert np.array_equal(g1, g2)
    assert wrapped.reexecutions() == 1
    d1, d2 = plain.derivative(0, 0, dy), wrapped.derivative(0, 0, dy)
    assert np.array_equal(d1, d2)
    assert wrapped.reexecutions() == 2
    fresh = build(lib).checkpoint()
    with pytest.raises(MdnnError) as e:
        fresh.derivative(0, 0, x)
    assert e.value.code == 8
    return y2, g2, d2


def test_reference_checkpoint_semantics(ref):
    rng = np.random.default_rng(91)
    x, dy = crand(rng, (4,)), crand(rng, (4,))
    _check(ref, _square_crelu_dft, x, dy)


@pytest.mark.gpu
def test_gpu_checkpoint_matches_plain_and_reference(gpu, ref):
    rng = np.random.default_rng(91)
    x, dy = crand(rng, (4,)), crand(rng, (4,))
    outs_g = _check(gpu, _square_crelu_dft, x, dy)
    outs_r = _check(ref, _square_crelu_dft, x, dy)
    for a, b in zip(outs_g, outs_r):
        assert rel_l2(a, b) <= 1e-5


@pytest.mark.gpu
def test_gpu_checkpointed_data_consistency_block(gpu, ref):
    """A MoDL data-consistency block (InverseNode over A^H A + lambda) under
    checkpoint: identical to the plain block on the GPU, within 1e-5 of the
    reference."""
    X, Y, NC = 32, 40, 3
    ph, cm, pat = sim_data(ref, X, Y, NC, 1)
    sd = sense_dims(X, Y, NC, 1, 1)
    lam = np.full(d16(), 0.05, dtype=np.complex64, order="F")

    def build(lib):
        return Model.modl_normal_plus_lambda(lib, sd).nlop.inverse(10, 0.0)

    rng = np.random.default_rng(3)
    y = crand(rng, image_dims(X, Y))
    dy = crand(rng, image_dims(X, Y))
    res = {}
    for name, lib in (("gpu", gpu), ("ref", ref)):
        plain, ck = build(lib), build(lib).checkpoint()
        ins = [y, cm, pat, lam]
        a, b = plain.apply(ins)[0], ck.apply(ins)[0]
        ga, gb = plain.adjoint_all(0, dy), ck.adjoint_all(0, dy)
        assert np.array_equal(a, b)
        for u, v in zip(ga, gb):
            assert np.array_equal(u, v)
        assert ck.reexecutions() == 1
        res[name] = (b, gb)
    assert rel_l2(res["gpu"][0], res["ref"][0]) <= 1e-5
    for u, v in zip(res["gpu"][1], res["ref"][1]):
        assert rel_l2(u, v) <= 1e-5
