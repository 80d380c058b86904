"""GPU build cfl I/O and weight bundles against the reference (cfl.hpp:15-142):
files are byte-identical in both directions, device and host buffers, large
arrays cross the double-buffered pinned staging, errors map to IoError."""
import filecmp
import os

import numpy as np
import pytest

from paper_2202_14005_b200.capi import MdnnError, to_device, to_host
from paper_2202_14005_b200.mdnn import Model, Trainer, cfl_dims, cfl_read, cfl_write, weights_meta
from util import crand, d16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", [(3,), (5, 7, 3), (320, 368, 1, 15), (1024, 1024, 5)])
def test_cfl_bytes_identical_both_ways(gpu, ref, tmp_path, shape):
    rng = np.random.default_rng(len(shape))
    a = crand(rng, shape)
    cfl_write(gpu, str(tmp_path / "g"), to_device(a))          # device array
    cfl_write(ref, str(tmp_path / "r"), a)
    for ext in (".hdr", ".cfl"):
        assert filecmp.cmp(str(tmp_path / "g") + ext, str(tmp_path / "r") + ext, shallow=False)
    assert cfl_dims(gpu, str(tmp_path / "r")) == cfl_dims(ref, str(tmp_path / "r")) == d16(*shape)
    dev = cfl_read(gpu, str(tmp_path / "r"), to_device(np.zeros(shape, np.complex64, order="F")))
    assert np.array_equal(to_host(dev), a)
    host = cfl_read(gpu, str(tmp_path / "r"), np.zeros(shape, np.complex64, order="F"))
    assert np.array_equal(host, a)


def test_cfl_errors_match_reference(gpu, ref, tmp_path):
    for lib in (gpu, ref):
        with pytest.raises(MdnnError) as e:
            cfl_dims(lib, str(tmp_path / "none"))
        assert e.value.code == 3 and "missing file" in str(e.value)
    base = str(tmp_path / "bad")
    cfl_write(ref, base, crand(np.random.default_rng(2), (4, 4)))
    with open(base + ".cfl", "ab") as f:
        f.write(b"\0" * 8)
    msgs = []
    for lib in (gpu, ref):
        with pytest.raises(MdnnError) as e:
            cfl_read(lib, base, np.zeros((4, 4), np.complex64, order="F"))
        assert e.value.code == 3
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1]


def test_weights_bundle_interchange(gpu, ref, tmp_path):
    kw = dict(iterations=1, layers=3, filters=8, cg_iter=3, im_x=16, im_y=12, coils=3)
    tg = Trainer(gpu, Model.modl(gpu, **kw), seed=5)
    tr = Trainer(ref, Model.modl(ref, **kw), seed=5)
    meta = {"network": "modl", "seed": 5}
    tg.save_weights(tmp_path / "g", meta)
    tr.save_weights(tmp_path / "r", meta)
    cmp = filecmp.dircmp(tmp_path / "g", tmp_path / "r")
    assert not cmp.left_only and not cmp.right_only
    for f in sorted(os.listdir(tmp_path / "r")):
        assert filecmp.cmp(tmp_path / "g" / f, tmp_path / "r" / f, shallow=False), f
    # a bundle written by the reference warm-starts the GPU trainer bitwise
    t2 = Trainer(gpu, Model.modl(gpu, **kw), seed=77)
    t2.load_weights(tmp_path / "r")
    for n in tr.weight_names():
        assert np.array_equal(t2.get_weight(n), tr.get_weight(n)), n
    assert weights_meta(gpu, tmp_path / "g", "network") == "modl"
