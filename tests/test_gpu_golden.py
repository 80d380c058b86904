"""GPU path vs the committed golden vectors (tests/golden, generated from the
fp32 reference by make_golden.py) — parity without the live oracle."""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import REPO
from paper_2202_14005_b200.mdnn import Model
from util import d16, rel_l2

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(REPO, "tests", "golden")
NAMES = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))


@pytest.mark.parametrize("name", NAMES)
def test_gpu_against_golden(gpu, name):
    g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    kind = str(g["kind"])
    lib = gpu

    def arr(a):
        return np.asfortranarray(a.astype(np.complex64))

    if kind == "dft":
        x = arr(g["x"])
        out = np.zeros(x.shape, dtype=np.complex64, order="F")
        lib.check(lib.so.mdnn_dft(C.byref(lib.arr(x)), int(g["flags"]), int(bool(g["inverse"])),
                                  C.byref(lib.arr(out))))
    elif kind in ("sense_normal", "sense_adjoint"):
        cm, pat = arr(g["coils"]), arr(g["pattern"])
        inp = arr(g["x"] if kind == "sense_normal" else g["y"])
        out = np.zeros(g["out"].shape, dtype=np.complex64, order="F")
        if kind == "sense_normal":
            lib.check(lib.so.mdnn_sense_normal(C.byref(lib.arr(cm)), C.byref(lib.arr(pat)), C.c_float(float(g["lam"])),
                                               C.byref(lib.arr(inp)), C.byref(lib.arr(out))))
        else:
            lib.check(lib.so.mdnn_sense_adjoint(C.byref(lib.arr(cm)), C.byref(lib.arr(pat)), C.byref(lib.arr(inp)),
                                                C.byref(lib.arr(out))))
    elif kind == "cg":
        cm, pat, b = arr(g["coils"]), arr(g["pattern"]), arr(g["b"])
        out = np.zeros(b.shape, dtype=np.complex64, order="F")
        it, rr = C.c_long(), C.c_double()
        lib.check(lib.so.mdnn_cg_normal_solve(C.byref(lib.arr(cm)), C.byref(lib.arr(pat)), C.c_float(float(g["lam"])),
                                              C.byref(lib.arr(b)), int(g["iters"]), 0.0, C.byref(lib.arr(out)),
                                              C.byref(it), C.byref(rr)))
    elif kind == "conv":
        x, w = arr(g["x"]), arr(g["w"])
        n = Model.conv_layer(lib, "c", list(x.shape), (w.shape[0], w.shape[1]), w.shape[3]).nlop
        out = n.apply([x, w])[0]
    else:
        pytest.skip(kind)
    assert rel_l2(out, g["out"]) <= float(g["tol"])
