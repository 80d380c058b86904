"""reconet driver (cli.hpp:94-265): estimate_pattern, normalize, seeded
mini-batch training to a weights bundle, chunked batched apply with inverse
scaling — the product (device arrays) against the reference's own train /
normalize / cfl functions driven by the same options.  Tolerances: the conv
layers run in TF32 on the GPU (1e-3, BASELINE.json north_star)."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2202_14005_b200.capi import MdnnError, mdnn_reconet_opts
from paper_2202_14005_b200.mdnn import cfl_read, cfl_write, weights_meta
from util import kspace_dims, pattern_dims, rel_l2, sim_data

X, Y, NC, N = 24, 20, 3, 4


def _dataset(ref, d, accel=2, acl=6):
    ph, cm, pat = sim_data(ref, X, Y, NC, N, accel=accel, acl=acl)
    ks = np.zeros(kspace_dims(X, Y, NC, N), dtype=np.complex64, order="F")
    ref.check(ref.so.mdnn_sense_forward(C.byref(ref.arr(cm)), C.byref(ref.arr(pat)), C.byref(ref.arr(ph)),
                                        C.byref(ref.arr(ks))))
    for name, a in (("kspace", ks), ("coils", cm), ("reference", ph), ("pattern", pat)):
        cfl_write(ref, os.path.join(d, name), a)
    return ph, pat


def _opts(d, network, train, weights, target, **kw):
    o = mdnn_reconet_opts()
    keep = []

    def s(v):
        b = str(v).encode()
        keep.append(b)
        return b
    import paper_2202_14005_b200.capi as capi  # noqa: F401
    o.network = s(network)
    o.do_train, o.do_apply = int(train), int(not train)
    o.normalize = int(kw.pop("normalize", False))
    o.pattern_file = s(os.path.join(d, "pattern")) if kw.pop("with_pattern", True) else None
    o.init_weights = None
    for f in ("iterations", "filters", "kernel", "rbf", "layers", "cg_iter"):
        setattr(o, f, kw.pop(f, -1))
    o.epochs = kw.pop("epochs", 2)
    o.batch_size = kw.pop("batch_size", 2)
    o.lr = kw.pop("lr", -1.0)
    o.optimizer = None
    o.seed = kw.pop("seed", 7)
    o.verbose = 0
    o.kspace_file = s(os.path.join(d, "kspace"))
    o.coils_file = s(os.path.join(d, "coils"))
    o.weights_dir = s(weights)
    o.target_file = s(target)
    assert not kw, kw
    o._keep = keep
    return o


def _run(lib, o):
    lib.check(lib.so.mdnn_reconet(C.byref(o)))


def test_reference_reconet_roundtrip_cpu(ref, tmp_path):
    """Oracle-only (CPU): estimate_pattern recovers the simulated pattern; a
    MoDL train + apply round trip writes a bundle and an output of the right
    shape; option errors map to ConfigError."""
    ph, pat = _dataset(ref, str(tmp_path))
    ks = cfl_read(ref, str(tmp_path / "kspace"))
    est = np.zeros(pattern_dims(Y), np.complex64, order="F")
    ref.check(ref.so.mdnn_estimate_pattern(C.byref(ref.arr(ks)), C.byref(ref.arr(est))))
    assert np.array_equal(est, pat)
    mk = dict(iterations=1, layers=3, filters=4, cg_iter=3, epochs=1)
    _run(ref, _opts(str(tmp_path), "modl", True, tmp_path / "w", tmp_path / "reference", **mk))
    assert weights_meta(ref, tmp_path / "w", "network") == "modl"
    assert weights_meta(ref, tmp_path / "w", "epochs") == "1"
    _run(ref, _opts(str(tmp_path), "modl", False, tmp_path / "w", tmp_path / "out", with_pattern=False))
    out = cfl_read(ref, str(tmp_path / "out"))
    assert out.shape[:2] == (X, Y) and out.shape[15] == N and np.isfinite(out).all()
    bad = _opts(str(tmp_path), "modl", True, tmp_path / "w2", tmp_path / "reference")
    bad.do_apply = 1
    with pytest.raises(MdnnError) as e:
        _run(ref, bad)
    assert e.value.code == 4


@pytest.mark.gpu
@pytest.mark.parametrize("normalize", [False, True])
def test_reconet_modl_train_and_apply_match_reference(gpu, ref, tmp_path, normalize):
    d = str(tmp_path)
    _dataset(ref, d)
    mk = dict(iterations=1, layers=3, filters=8, cg_iter=4, epochs=2, batch_size=2, normalize=normalize)
    _run(gpu, _opts(d, "modl", True, tmp_path / "wg", tmp_path / "reference", **mk))
    _run(ref, _opts(d, "modl", True, tmp_path / "wr", tmp_path / "reference", **mk))
    mg = open(tmp_path / "wg" / "manifest.txt").read()
    mr = open(tmp_path / "wr" / "manifest.txt").read()
    assert mg == mr  # same meta, same sorted array list
    for line in mr.splitlines():
        if line.startswith("array "):
            name = line.split(" ", 1)[1]
            a, b = cfl_read(ref, str(tmp_path / "wg" / name)), cfl_read(ref, str(tmp_path / "wr" / name))
            assert rel_l2(a, b) <= 1e-3 or np.abs(a - b).max() <= 1e-6, name
    # apply the reference-trained bundle on both (inference-mode BN, chunked batches of 3)
    for lib, out in ((gpu, "og"), (ref, "or")):
        o = _opts(d, "modl", False, tmp_path / "wr", tmp_path / out, batch_size=3)
        _run(lib, o)
    og, orf = cfl_read(ref, str(tmp_path / "og")), cfl_read(ref, str(tmp_path / "or"))
    assert rel_l2(og, orf) <= 1e-3


@pytest.mark.gpu
def test_reconet_varnet_ipalm_and_estimated_pattern(gpu, ref, tmp_path):
    d = str(tmp_path)
    _dataset(ref, d)
    vk = dict(iterations=2, filters=3, kernel=5, rbf=7, epochs=1, batch_size=2, with_pattern=False)
    _run(gpu, _opts(d, "varnet", True, tmp_path / "wg", tmp_path / "reference", **vk))
    _run(ref, _opts(d, "varnet", True, tmp_path / "wr", tmp_path / "reference", **vk))
    assert open(tmp_path / "wg" / "manifest.txt").read() == open(tmp_path / "wr" / "manifest.txt").read()
    for f in sorted(os.listdir(tmp_path / "wr")):
        if f.endswith(".cfl"):
            base = f[:-4]
            a, b = cfl_read(ref, str(tmp_path / "wg" / base)), cfl_read(ref, str(tmp_path / "wr" / base))
            assert rel_l2(a, b) <= 1e-3 or np.abs(a - b).max() <= 1e-6, base
    for lib, out in ((gpu, "og"), (ref, "or")):
        _run(lib, _opts(d, "varnet", False, tmp_path / "wr", tmp_path / out, with_pattern=False))
    assert rel_l2(cfl_read(ref, str(tmp_path / "og")), cfl_read(ref, str(tmp_path / "or"))) <= 1e-3
    # a bundle for one network refuses the other (ConfigError)
    with pytest.raises(MdnnError) as e:
        _run(gpu, _opts(d, "modl", False, tmp_path / "wr", tmp_path / "x"))
    assert e.value.code == 4
