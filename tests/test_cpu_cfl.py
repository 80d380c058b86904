"""cfl I/O and weight bundles of the reference (oracle shim over cfl.hpp),
checked on CPU against an independent numpy restatement of the file format
(cfl.hpp:15-88) and the reference's own error taxonomy (IoError, code 3)."""
import os

import numpy as np
import pytest

from paper_2202_14005_b200.capi import MdnnError
from paper_2202_14005_b200.mdnn import Model, Trainer, cfl_dims, cfl_read, cfl_write, weights_meta
from util import crand, d16


def _np_write(base, a):
    dims = list(a.shape) + [1] * (16 - a.ndim)
    with open(base + ".hdr", "w") as f:
        f.write("# Dimensions\n" + " ".join(str(d) for d in dims) + "\n")
    np.asfortranarray(a.astype(np.complex64)).ravel(order="F").tofile(base + ".cfl")


def test_reference_cfl_matches_numpy_format(ref, tmp_path):
    rng = np.random.default_rng(0)
    a = crand(rng, (5, 7, 3))
    base = str(tmp_path / "a")
    cfl_write(ref, base, a)
    hdr = open(base + ".hdr").read()
    assert hdr == "# Dimensions\n5 7 3 1 1 1 1 1 1 1 1 1 1 1 1 1\n"
    raw = np.fromfile(base + ".cfl", dtype=np.complex64)
    assert np.array_equal(raw, a.ravel(order="F"))
    # numpy-written file read by the reference
    _np_write(str(tmp_path / "b"), a)
    assert cfl_dims(ref, str(tmp_path / "b")) == d16(5, 7, 3)
    assert np.array_equal(cfl_read(ref, str(tmp_path / "b"), np.zeros((5, 7, 3), np.complex64, order="F")), a)


def test_reference_cfl_errors(ref, tmp_path):
    base = str(tmp_path / "missing")
    with pytest.raises(MdnnError) as e:
        cfl_dims(ref, base)
    assert e.value.code == 3 and "missing file" in str(e.value)
    a = crand(np.random.default_rng(1), (4, 4))
    _np_write(base, a)
    with open(base + ".cfl", "ab") as f:
        f.write(b"\0" * 8)
    with pytest.raises(MdnnError) as e:
        cfl_read(ref, base, np.zeros((4, 4), np.complex64, order="F"))
    assert e.value.code == 3 and "header implies" in str(e.value)


def test_reference_weights_bundle_roundtrip(ref, tmp_path):
    m = Model.modl(ref, iterations=1, layers=3, filters=4, cg_iter=2, im_x=8, im_y=8, coils=2)
    t1 = Trainer(ref, m, seed=3)
    t1.save_weights(tmp_path / "w", {"network": "modl", "seed": 3})
    assert weights_meta(ref, tmp_path / "w", "network") == "modl"
    assert weights_meta(ref, tmp_path / "w", "nope", "fb") == "fb"
    lines = open(tmp_path / "w" / "manifest.txt").read().splitlines()
    assert lines[0] == "format 1" and lines[1:3] == ["network modl", "seed 3"]
    names = [ln.split(" ", 1)[1] for ln in lines if ln.startswith("array ")]
    assert names == sorted(names) and set(t1.weight_names()) <= set(names)
    assert any(n.endswith("_bn_mean") for n in names)  # moving statistics travel with the weights
    t2 = Trainer(ref, m, seed=99)
    t2.load_weights(tmp_path / "w")
    for n in t1.weight_names():
        assert np.array_equal(t1.get_weight(n), t2.get_weight(n)), n
    os.remove(tmp_path / "w" / "manifest.txt")
    with pytest.raises(MdnnError) as e:
        t2.load_weights(tmp_path / "w")
    assert e.value.code == 3
