"""Optimizer selection through the C ABI on the reference shim (CPU): the
TrainConfig defaults (optim.hpp:20-56), SGD / iPALM trajectories that move
the weights, iPALM's refusal of the split forward/backward + update path."""
import numpy as np
import pytest

from paper_2202_14005_b200.capi import ALGO_ADAM, ALGO_IPALM, ALGO_SGD, MdnnError, mdnn_train_cfg
from paper_2202_14005_b200.mdnn import Model, Trainer
from util import sim_data


def test_train_cfg_defaults(ref):
    import ctypes as C
    c = mdnn_train_cfg()
    ref.so.mdnn_train_cfg_default(C.byref(c))
    assert (c.lr, c.beta1, c.beta2, c.eps, c.clip) == (1e-3, 0.9, 0.999, 1e-8, 0.0)
    assert c.algo == ALGO_ADAM and (c.ipalm_alpha, c.ipalm_beta) == (0.5, 0.5)


@pytest.mark.parametrize("algo", [ALGO_SGD, ALGO_IPALM])
def test_reference_optimizers_step(ref, algo):
    X, Y, NC = 8, 8, 2
    m = Model.varnet(ref, iterations=1, filters=2, kernel=3, rbf=5, im_x=X, im_y=Y, coils=NC)
    ph, cm, pat = sim_data(ref, X, Y, NC, 1)
    t = Trainer(ref, m, seed=1, lr=1e-2, algo=algo)
    import ctypes as C
    from util import kspace_dims
    ks = np.zeros(kspace_dims(X, Y, NC), dtype=np.complex64, order="F")
    ref.check(ref.so.mdnn_sense_forward(C.byref(ref.arr(cm)), C.byref(ref.arr(pat)), C.byref(ref.arr(ph)),
                                        C.byref(ref.arr(ks))))
    for k, v in (("kspace", ks), ("coils", cm), ("pattern", pat), ("reference", ph)):
        t.set_data(k, v)
    w0 = {n: t.get_weight(n) for n in t.weight_names()}
    l0 = t.step()
    assert np.isfinite(l0)
    assert any(not np.array_equal(w0[n], t.get_weight(n)) for n in w0)
    if algo == ALGO_IPALM:
        with pytest.raises(MdnnError) as e:
            ref.check(ref.so.mdnn_trainer_update(t.h, 1.0))
        assert e.value.code == 4


def test_stage_data_queue_order(ref):
    """mdnn_trainer_stage_data on the shim: queued batches are consumed one per
    step, oldest first, and match feeding the same batches with set_data."""
    import ctypes as C
    from util import kspace_dims
    X, Y, NC = 8, 8, 2
    ph, cm, pat = sim_data(ref, X, Y, NC, 1)
    ks = np.zeros(kspace_dims(X, Y, NC), dtype=np.complex64, order="F")
    ref.check(ref.so.mdnn_sense_forward(C.byref(ref.arr(cm)), C.byref(ref.arr(pat)), C.byref(ref.arr(ph)),
                                        C.byref(ref.arr(ks))))
    batches = [dict(kspace=ks, coils=cm, pattern=pat, reference=np.asfortranarray(ph * s)) for s in (1.0, 0.5)]
    losses = []
    for staged in (False, True):
        m = Model.varnet(ref, iterations=1, filters=2, kernel=3, rbf=5, im_x=X, im_y=Y, coils=NC)
        t = Trainer(ref, m, seed=1, lr=1e-2)
        ls = []
        if staged:
            for b in batches:
                for k, v in b.items():
                    t.stage_data(k, v)
            ls = [t.step(), t.step()]
        else:
            for b in batches:
                for k, v in b.items():
                    t.set_data(k, v)
                ls.append(t.step())
        losses.append(ls)
    assert losses[0] == losses[1] and losses[0][0] != losses[0][1]
