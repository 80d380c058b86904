"""Tensor-core conv micro-benchmark at the MoDL C2 layer shape (64->64, 3x3,
320x368, batch 8): forward, bwd-data and bwd-weight kernel times from the
library's per-tag CUDA-event profile.  Option sets (--set "k=v k=v", repeatable)
are measured alternately for --rounds rounds in one process; the median per set
is reported.  Usage:
    python tools/conv_bench.py [--set "key=value ..."]... [--reps N] [--rounds R]"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", action="append", default=[])
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--shape", default="320,368,64,64,8")
    args = ap.parse_args()
    from paper_2202_14005_b200 import load_library
    from paper_2202_14005_b200.mdnn import Model
    from util import crand, d16

    lib = load_library()
    lib.check(lib.so.mdnn_set_device(0))
    sets = args.set or [""]

    def apply_set(st):
        for kv in st.split():
            k, v = kv.split("=")
            lib.check(lib.so.mdnn_set_option(k.encode(), int(v)))

    X, Y, cin, cout, B = (int(v) for v in args.shape.split(","))
    dims = list(d16(X, Y, cin))
    dims[15] = B
    lib.check(lib.so.mdnn_set_option(b"conv_chlast", 1))
    m = Model.conv_layer(lib, "c", dims, (3, 3), cout)
    n = m.nlop
    rng = np.random.default_rng(0)
    x, w = crand(rng, n.in_dims(0)), crand(rng, n.in_dims(1), 0.05)
    dy = crand(rng, n.out_dims(0))
    n.apply([x, w])
    n.adjoint_all(0, dy)
    tags = ("conv_tc_fwd", "conv_tc_bwd_data", "conv_tc_bwd_weight")
    res = {st: {t: [] for t in tags} for st in sets}
    for _ in range(args.rounds):
        for st in sets:
            apply_set(st)
            n.apply([x, w])
            lib.check(lib.so.mdnn_profile_reset())
            lib.check(lib.so.mdnn_profile_enable(1))
            for _ in range(args.reps):
                n.apply([x, w])
                n.adjoint_all(0, dy)
            lib.check(lib.so.mdnn_synchronize())
            lib.check(lib.so.mdnn_profile_enable(0))
            for tag in tags:
                L, ms, work = C.c_long(), C.c_double(), C.c_double()
                lib.check(lib.so.mdnn_profile_read(tag.encode(), C.byref(L), C.byref(ms), C.byref(work)))
                if L.value:
                    res[st][tag].append((1e3 * ms.value / L.value, work.value / ms.value / 1e9))
            apply_set(" ".join(kv.split("=")[0] + "=0" for kv in st.split() if kv.startswith("conv_tc_debug")))
    for st in sets:
        out = {"set": st, "shape": [X, Y, cin, cout, B]}
        for tag in tags:
            v = sorted(res[st][tag])
            if v:
                us, tf = v[len(v) // 2]
                out[tag] = {"us_med": round(us, 1), "us_min": round(v[0][0], 1), "tflops_med": round(tf, 1)}
        print(out)


if __name__ == "__main__":
    main()
