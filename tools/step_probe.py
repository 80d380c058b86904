"""Per-step wall vs device time of the bench workload, alternating A/B options.
Usage: python tools/step_probe.py [workload] [option] [values...]"""
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
import bench  # noqa: E402


def main(workload="modl_c2", opt="sense_rank", *vals):
    import torch
    from paper_2202_14005_b200 import load_library
    from paper_2202_14005_b200.mdnn import Trainer
    lib = load_library()
    lib.check(lib.so.mdnn_set_device(0))
    stream = torch.cuda.ExternalStream(lib.so.mdnn_stream(), device=torch.device("cuda", 0))
    kw, X, Y, NC, B = bench.WORKLOADS[workload]
    data = bench.make_data(lib, X, Y, NC, B, first_item=0)
    tr = Trainer(lib, bench.build_model(lib, workload, B), seed=42)
    for k, v in data.items():
        tr.set_data(k, torch.from_numpy(np.ascontiguousarray(v.transpose())).cuda())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nsteps = int(os.environ.get("PROBE_STEPS", 4))
    for v in (vals or ("1", "0", "1", "0")):
        lib.check(lib.so.mdnn_set_option(opt.encode(), int(v)))
        for s in range(nsteps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0.record(stream)
            tr.step()
            e1.record(stream)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            print(f"{opt}={v} step {s}: wall {1e3 * (t1 - t0):8.2f} ms  device {e0.elapsed_time(e1):8.2f} ms", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
