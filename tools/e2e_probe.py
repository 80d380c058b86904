"""Host-side cost breakdown of one training step (where e2e time goes):
set_data per input, forward_backward, all-reduce, update — host wall clock
with a device sync after each phase.  Usage: python tools/e2e_probe.py [workload]"""
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import bench  # noqa: E402


def main(workload="modl_c2"):
    import torch
    from paper_2202_14005_b200 import load_library
    from paper_2202_14005_b200.mdnn import Trainer

    lib = load_library()
    kw, X, Y, NC, B = bench.WORKLOADS[workload]
    data = bench.make_data(lib, X, Y, NC, B, first_item=0)
    model = bench.build_model(lib, workload, B)
    tr = Trainer(lib, model, seed=42)
    pinned = {k: torch.from_numpy(np.ascontiguousarray(v.transpose())).pin_memory() for k, v in data.items()}
    dev = {k: v.cuda() for k, v in pinned.items()}
    for k, v in dev.items():
        tr.set_data(k, v)

    def sync():
        torch.cuda.synchronize()
        lib.check(lib.so.mdnn_synchronize())

    for _ in range(3):
        tr.forward_backward()
        tr.update(1.0)
    sync()
    for rep in range(3):
        t = {}
        t0 = time.perf_counter()
        for k, v in pinned.items():
            a = time.perf_counter()
            tr.set_data(k, v)
            sync()
            t["set_" + k] = time.perf_counter() - a
        a = time.perf_counter()
        tr.forward_backward()
        sync()
        t["fwd_bwd"] = time.perf_counter() - a
        a = time.perf_counter()
        tr.update(1.0)
        sync()
        t["update"] = time.perf_counter() - a
        t["total"] = time.perf_counter() - t0
        print({k: round(v * 1e3, 2) for k, v in t.items()}, "ms", flush=True)
    # spike hunt: per-step wall time and per-tag device time
    import ctypes as C
    tags = ["sense_normal_y_cg", "sense_normal_y", "fft", "conv_tc_fwd", "conv_tc_bwd_data", "conv_tc_bwd_weight",
            "conv_thin_fwd", "conv_thin_bwd_data", "conv_thin_bwd_weight", "bnblock_fwd", "bnblock_bwd",
            "conv_fwd", "conv_bwd_data", "conv_bwd_weight"]
    for rep in range(10):
        lib.check(lib.so.mdnn_profile_reset())
        lib.check(lib.so.mdnn_profile_enable(1))
        a = time.perf_counter()
        tr.forward_backward()
        tr.update(1.0)
        sync()
        wall = time.perf_counter() - a
        lib.check(lib.so.mdnn_profile_enable(0))
        dev = {}
        for tg in tags:
            n, ms, work = C.c_long(), C.c_double(), C.c_double()
            lib.check(lib.so.mdnn_profile_read(tg.encode(), C.byref(n), C.byref(ms), C.byref(work)))
            if n.value:
                dev[tg] = round(ms.value, 1)
        print(f"rep {rep}: wall {wall * 1e3:.1f} ms, tagged device {sum(dev.values()):.1f} ms", dev, flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
