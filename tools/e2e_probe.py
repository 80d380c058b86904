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
    # host launch overhead: time to enqueue (no sync) vs device time
    lib.check(lib.so.mdnn_profile_enable(0))
    a = time.perf_counter()
    tr.forward_backward()
    b = time.perf_counter()
    print("forward_backward wall incl. final sync", round((b - a) * 1e3, 2), "ms")


if __name__ == "__main__":
    main(*sys.argv[1:])
