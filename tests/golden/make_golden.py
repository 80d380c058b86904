"""Generate the committed golden vectors from the fp32 reference (oracle/_ref,
the unmodified reference headers compiled in place).  Run in the dev
container, where /root/reference exists:  python tests/golden/make_golden.py

Each .npz holds inputs, the reference output and the tolerance the product must
meet (the north_star parity bars: 1e-5 SENSE/CG/DFT, 1e-3 TF32 conv)."""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
from paper_2202_14005_b200.capi import Lib  # noqa: E402
from paper_2202_14005_b200.mdnn import Model  # noqa: E402
from util import crand, d16, image_dims, kspace_dims, sim_data  # noqa: E402


def main():
    ref = Lib(os.path.join(REPO, "oracle", "_ref", "libmdnn_ref.so"))
    rng = np.random.default_rng(2022)

    def save(name, **kw):
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **kw)

    # DFT: odd prime and Bluestein lengths (fft.hpp:143-157)
    for dims, flags, inv in [((23, 16), 3, False), ((20, 9, 2), 1, True)]:
        x = crand(rng, dims)
        y = np.zeros(dims, dtype=np.complex64, order="F")
        ref.check(ref.so.mdnn_dft(C.byref(ref.arr(x)), flags, int(inv), C.byref(ref.arr(y))))
        save(f"dft_{'x'.join(map(str, dims))}_{flags}_{int(inv)}", kind="dft", x=x, flags=flags, inverse=inv, out=y,
             tol=1e-5)

    X, Y, NC, B = 24, 23, 4, 2
    ph, cm, pat = sim_data(ref, X, Y, NC, B, accel=3, acl=4)
    out = np.zeros(image_dims(X, Y, B), dtype=np.complex64, order="F")
    ref.check(ref.so.mdnn_sense_normal(C.byref(ref.arr(cm)), C.byref(ref.arr(pat)), C.c_float(0.05),
                                       C.byref(ref.arr(ph)), C.byref(ref.arr(out))))
    save("sense_normal_24x23x4", kind="sense_normal", x=ph, coils=cm, pattern=pat, lam=0.05, out=out, tol=1e-5)

    k = crand(rng, kspace_dims(X, Y, NC, B))
    out = np.zeros(image_dims(X, Y, B), dtype=np.complex64, order="F")
    ref.check(ref.so.mdnn_sense_adjoint(C.byref(ref.arr(cm)), C.byref(ref.arr(pat)), C.byref(ref.arr(k)),
                                        C.byref(ref.arr(out))))
    save("sense_adjoint_24x23x4", kind="sense_adjoint", y=k, coils=cm, pattern=pat, out=out, tol=1e-5)

    b = crand(rng, image_dims(X, Y, B))
    out = np.zeros(image_dims(X, Y, B), dtype=np.complex64, order="F")
    it, rr = C.c_long(), C.c_double()
    ref.check(ref.so.mdnn_cg_normal_solve(C.byref(ref.arr(cm)), C.byref(ref.arr(pat)), C.c_float(0.05),
                                          C.byref(ref.arr(b)), 8, 0.0, C.byref(ref.arr(out)), C.byref(it),
                                          C.byref(rr)))
    save("cg8_24x23x4", kind="cg", b=b, coils=cm, pattern=pat, lam=0.05, iters=8, out=out, tol=1e-5)

    in_dims = list(d16(20, 12, 8))
    in_dims[15] = 2
    n = Model.conv_layer(ref, "c", in_dims, (3, 3), 8).nlop
    x, w = crand(rng, n.in_dims(0)), crand(rng, n.in_dims(1), 0.2)
    save("conv3x3_8to8", kind="conv", x=x, w=w, out=n.apply([x, w])[0], tol=1e-5)


if __name__ == "__main__":
    main()
