"""End-to-end MoDL / VarNet parity (recon.hpp:499-904, fixed builders) and
training steps (optim.hpp:314-415).

End-to-end outputs and weight gradients are judged against the fp64
reference with the criterion of SURVEY §8c: GPU error <= max(tol, 2 x the
CPU-fp32 reference's own error) — train-mode batch norm is ill-conditioned
even for the reference itself.
"""
import numpy as np
import pytest

from paper_2202_14005_b200.mdnn import ARG_DATA, ARG_WEIGHTS, Model, Trainer
from util import crand, kspace_dims, rel_l2, sim_data

pytestmark = pytest.mark.gpu


def _inputs(ref, model, X, Y, NC, B, seed=42, rbf_perturb=False):
    # 3-fold regular + 2 ACL lines: genuinely undersampled at these toy sizes
    ph, cm, pat = sim_data(ref, X, Y, NC, B, accel=3, acl=2)
    import ctypes as C
    ks = np.zeros(kspace_dims(X, Y, NC, B), dtype=np.complex64, order="F")
    ref.check(ref.so.mdnn_sense_forward(C.byref(ref.arr(cm)), C.byref(ref.arr(pat)), C.byref(ref.arr(ph)),
                                        C.byref(ref.arr(ks))))
    data = {"kspace": ks, "coils": cm, "pattern": pat, "reference": ph}
    w = model.init_weights(seed)
    if rbf_perturb:
        rng = np.random.default_rng(99)
        for k in w:
            if k.endswith("_rbf_w"):
                w[k] = np.asfortranarray(rng.uniform(-0.05, 0.05, w[k].shape).astype(np.complex64))
    return data, w


def _run(lib, build, cfg, data, w):
    m = build(lib, **cfg)
    n = m.nlop
    ins = [data[a] if k == ARG_DATA else w[a] for a, k, _ in m.args]
    outs = n.apply(ins)
    oi = m.output_index("out")
    rng = np.random.default_rng(5)
    dy = crand(rng, n.out_dims(oi))
    wanted = [k == ARG_WEIGHTS for _, k, _ in m.args]
    g = n.adjoint_all(oi, dy, wanted)
    grads = {a: g[i] for i, (a, k, _) in enumerate(m.args) if k == ARG_WEIGHTS}
    # tangents (Nlop::derivative) along the first two weights' directions
    for a, k, _ in [x for x in m.args if x[1] == ARG_WEIGHTS][:3]:
        i = m.arg_index(a)
        dx = crand(np.random.default_rng(7 + i), n.in_dims(i), 0.01)
        grads["tangent:" + a] = n.derivative(oi, i, dx)
    return dict(zip(m.out_names, outs)), grads


def _e2e(gpu, ref, ref64, build, cfg, X, Y, NC, B, out_tol, grad_tol, rbf_perturb=False):
    mref = build(ref, **cfg)
    data, w = _inputs(ref, mref, X, Y, NC, B, rbf_perturb=rbf_perturb)
    og, gg = _run(gpu, build, cfg, data, w)
    orf, gr = _run(ref, build, cfg, data, w)
    o64, g64 = _run(ref64, build, cfg, data, w)
    for k in o64:
        e_gpu, e_cpu = rel_l2(og[k], o64[k]), rel_l2(orf[k], o64[k])
        assert e_gpu <= max(out_tol, 2 * e_cpu), (k, e_gpu, e_cpu)
    for k in g64:
        e_gpu, e_cpu = rel_l2(gg[k], g64[k]), rel_l2(gr[k], g64[k])
        assert e_gpu <= max(grad_tol, 2 * e_cpu), (k, e_gpu, e_cpu)


def test_modl_parameter_count_and_args(gpu, ref):
    kw = dict(im_x=16, im_y=12, coils=2, filters=32)
    mg, mr = Model.modl(gpu, **kw), Model.modl(ref, **kw)
    assert mg.num_real_params() == mr.num_real_params() == 56963
    assert mg.args == mr.args
    assert mg.out_names == mr.out_names


def test_varnet_parameter_count(gpu, ref):
    kw = dict(im_x=16, im_y=12, coils=2)
    mg, mr = Model.varnet(gpu, **kw), Model.varnet(ref, **kw)
    assert mg.num_real_params() == mr.num_real_params() == 65530
    assert mg.args == mr.args


def test_modl_end_to_end_train_mode(gpu, ref, ref64):
    cfg = dict(iterations=2, layers=3, filters=4, cg_iter=5, im_x=16, im_y=12, coils=3, batch=2)
    _e2e(gpu, ref, ref64, Model.modl, cfg, 16, 12, 3, 2, 1e-5, 1e-3)


def test_modl_end_to_end_inference_bn(gpu, ref, ref64):
    cfg = dict(iterations=2, layers=3, filters=4, cg_iter=5, im_x=16, im_y=12, coils=3, batch=1, train_mode=0)
    _e2e(gpu, ref, ref64, Model.modl, cfg, 16, 12, 3, 1, 1e-5, 1e-3)


def test_varnet_end_to_end(gpu, ref, ref64):
    cfg = dict(iterations=2, filters=3, kernel=5, rbf=7, im_x=16, im_y=12, coils=3, batch=2)
    _e2e(gpu, ref, ref64, Model.varnet, cfg, 16, 12, 3, 2, 1e-5, 1e-3, rbf_perturb=True)


@pytest.mark.parametrize("net", ["modl", "varnet"])
def test_training_steps_match_reference(gpu, ref, net):
    X, Y, NC, B = 16, 12, 3, 2
    if net == "modl":
        cfg = dict(iterations=2, layers=3, filters=4, cg_iter=5, im_x=X, im_y=Y, coils=NC, batch=B)
        build = Model.modl
    else:
        cfg = dict(iterations=2, filters=3, kernel=5, rbf=7, im_x=X, im_y=Y, coils=NC, batch=B)
        build = Model.varnet
    mref = build(ref, **cfg)
    data, _ = _inputs(ref, mref, X, Y, NC, B)
    losses = []
    trainers = []
    for lib in (gpu, ref):
        m = build(lib, **cfg)
        t = Trainer(lib, m, seed=42, lr=1e-3)
        for k, v in data.items():
            t.set_data(k, v)
        losses.append([t.step() for _ in range(3)])
        trainers.append(t)
    np.testing.assert_allclose(losses[0], losses[1], rtol=1e-4)
    for name in trainers[1].weight_names():
        wg, wr = trainers[0].get_weight(name), trainers[1].get_weight(name)
        assert rel_l2(wg, wr) <= 1e-3, name


@pytest.mark.parametrize("net,algo", [("varnet", "ipalm"), ("modl", "ipalm"), ("modl", "sgd"), ("varnet", "sgd")])
def test_optimizer_trajectories_match_reference(gpu, ref, net, algo):
    """SGD and iPALM (optim.hpp:66-71, 110-153; run_step's iPALM branch
    :331-370, Gauss-Seidel block order, VarNet's CLI default cli.hpp:194)
    against the reference's own run_step."""
    from paper_2202_14005_b200.capi import ALGO_IPALM, ALGO_SGD
    X, Y, NC, B = 16, 12, 3, 2
    if net == "modl":
        cfg = dict(iterations=2, layers=3, filters=4, cg_iter=5, im_x=X, im_y=Y, coils=NC, batch=B)
        build = Model.modl
    else:
        cfg = dict(iterations=2, filters=3, kernel=5, rbf=7, im_x=X, im_y=Y, coils=NC, batch=B)
        build = Model.varnet
    mref = build(ref, **cfg)
    data, _ = _inputs(ref, mref, X, Y, NC, B)
    code = {"sgd": ALGO_SGD, "ipalm": ALGO_IPALM}[algo]
    losses, trainers = [], []
    for lib in (gpu, ref):
        t = Trainer(lib, build(lib, **cfg), seed=42, lr=1e-3, algo=code, ipalm_alpha=0.5, ipalm_beta=0.5)
        for k, v in data.items():
            t.set_data(k, v)
        losses.append([t.step() for _ in range(3)])
        trainers.append(t)
    np.testing.assert_allclose(losses[0], losses[1], rtol=1e-4)
    for name in trainers[1].weight_names():
        wg, wr = trainers[0].get_weight(name), trainers[1].get_weight(name)
        assert rel_l2(wg, wr) <= 1e-3, name


@pytest.mark.parametrize("algo", ["adam", "ipalm"])
def test_staged_batches_match_reference(gpu, ref, algo):
    """Prefetch queue (mdnn_trainer_stage_data): three different batches queued
    ahead of the steps, one taken per step, against the reference fed the same
    batches in order (the shim's synchronous queue)."""
    from paper_2202_14005_b200.capi import ALGO_ADAM, ALGO_IPALM
    X, Y, NC, B = 16, 12, 3, 2
    cfg = dict(iterations=2, layers=3, filters=4, cg_iter=5, im_x=X, im_y=Y, coils=NC, batch=B)
    mref = Model.modl(ref, **cfg)
    batches = []
    for s in range(3):
        data, _ = _inputs(ref, mref, X, Y, NC, B)
        rng = np.random.default_rng(s)
        data["reference"] = np.asfortranarray(data["reference"] * (1 + 0.1 * s)
                                              + 0.01 * crand(rng, data["reference"].shape))
        batches.append(data)
    code = {"adam": ALGO_ADAM, "ipalm": ALGO_IPALM}[algo]
    losses = []
    for lib in (gpu, ref):
        t = Trainer(lib, Model.modl(lib, **cfg), seed=42, lr=1e-3, algo=code)
        for d in batches[:2]:
            for k, v in d.items():
                t.stage_data(k, v)
        ls = [t.step()]
        for k, v in batches[2].items():
            t.stage_data(k, v)
        ls += [t.step(), t.step()]
        losses.append(ls)
    np.testing.assert_allclose(losses[0], losses[1], rtol=1e-4)
    assert len(set(np.round(losses[1], 12))) == 3  # three distinct batches were consumed


def test_modl_64_filters_bn_fusion(gpu, ref):
    """64-filter MoDL (the tensor-core conv path): batch-norm statistics taken
    from the conv epilogue and the BN backward reduction folded into the
    bwd-data conv epilogue agree with the unfused passes (summation order only)
    and with the reference (TF32 budget)."""
    X, Y, NC, B = 24, 40, 2, 2
    cfg = dict(iterations=1, layers=3, filters=64, cg_iter=3, im_x=X, im_y=Y, coils=NC, batch=B)
    mref = Model.modl(ref, **cfg)
    data, _ = _inputs(ref, mref, X, Y, NC, B)
    res = []
    for fuse in (1, 0):
        gpu.check(gpu.so.mdnn_set_option(b"conv_bn_fuse", fuse))
        try:
            t = Trainer(gpu, Model.modl(gpu, **cfg), seed=42, lr=1e-3)
            for k, v in data.items():
                t.set_data(k, v)
            loss = t.forward_backward()
            res.append((loss, {n: t.get_grad(n) for n in t.weight_names()}))
        finally:
            gpu.check(gpu.so.mdnn_set_option(b"conv_bn_fuse", 1))
    tr = Trainer(ref, mref, seed=42, lr=1e-3)
    for k, v in data.items():
        tr.set_data(k, v)
    lref = tr.forward_backward()
    (lf, gf), (lu, gu) = res
    assert abs(lf - lu) <= 1e-5 * abs(lu)
    assert abs(lf - lref) <= 1e-3 * abs(lref)
    # the fused path ran: BN statistics summed in a different order somewhere
    assert any(not np.array_equal(gf[n], gu[n]) for n in gu)
    for n in gu:
        assert rel_l2(gf[n], gu[n]) <= 1e-4, n
        assert rel_l2(gf[n], tr.get_grad(n)) <= 5e-3, n


def test_varnet_complex_values_in_real_weight_args(gpu, ref):
    """Real-weight arguments are tagged known-real for the real-operand conv
    kernels only when their values are real: a caller-provided complex value
    (set_weight) must take the general kernels and match the reference."""
    X, Y, NC, B = 16, 12, 3, 2
    cfg = dict(iterations=2, filters=3, kernel=5, rbf=7, im_x=X, im_y=Y, coils=NC, batch=B)
    mref = Model.varnet(ref, **cfg)
    data, _ = _inputs(ref, mref, X, Y, NC, B)
    rng = np.random.default_rng(17)
    losses, pert = [], {}
    for lib in (gpu, ref):
        t = Trainer(lib, Model.varnet(lib, **cfg), seed=42, lr=1e-3)
        for k, v in data.items():
            t.set_data(k, v)
        for name in t.weight_names():
            if name.endswith("_k_w"):
                w = t.get_weight(name)
                if name not in pert:  # the same complex values on both sides
                    pert[name] = (0.2j * rng.standard_normal(w.shape)).astype(np.complex64)
                t.set_weight(name, np.asfortranarray(w + pert[name]))
        losses.append(t.forward_backward())
    assert pert
    np.testing.assert_allclose(losses[0], losses[1], rtol=1e-4)
