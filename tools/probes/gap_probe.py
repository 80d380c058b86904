"""Device-timeline gaps of one training step (CUPTI through torch.profiler):
kernel time vs the step's span, the largest idle gaps and the kernels around
them.  Usage: python tools/probes/gap_probe.py [workload]"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main():
    import numpy as np
    import torch
    import bench
    from paper_2202_14005_b200 import load_library
    from paper_2202_14005_b200.mdnn import Trainer

    wl = sys.argv[1] if len(sys.argv) > 1 else "modl_c2"
    lib = load_library()
    lib.check(lib.so.mdnn_set_device(0))
    kw, X, Y, NC, B = bench.WORKLOADS[wl]
    data = bench.make_data(lib, X, Y, NC, B, first_item=0)
    model = bench.build_model(lib, wl, B)
    tr = Trainer(lib, model, seed=42)
    dev = {k: torch.from_numpy(np.ascontiguousarray(v.transpose())).to("cuda:0") for k, v in data.items()}
    for k, v in dev.items():
        tr.set_data(k, v)
    for _ in range(3):
        tr.step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(2):
            tr.step()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    if not ev:
        print("no device events")
        return
    span = ev[-1].time_range.end - ev[0].time_range.start
    busy = sum(e.time_range.end - e.time_range.start for e in ev)
    gaps = []
    end = ev[0].time_range.end
    prev = ev[0]
    for e in ev[1:]:
        g = e.time_range.start - end
        if g > 0:
            gaps.append((g, prev.name, e.name))
        if e.time_range.end > end:
            end = e.time_range.end
            prev = e
    tot_gap = sum(g for g, _, _ in gaps)
    print(f"{wl}: 2 steps span {span / 1000:.2f} ms, device busy {busy / 1000:.2f} ms, idle gaps {tot_gap / 1000:.2f} ms "
          f"over {len(gaps)} gaps, {len(ev)} device events")
    hist = {}
    for g, a, b in gaps:
        k = (a[:60], b[:60])
        h = hist.setdefault(k, [0, 0.0])
        h[0] += 1
        h[1] += g
    print("largest gap totals by (before, after):")
    for (a, b), (n, t) in sorted(hist.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"  {t / 1000:8.3f} ms  n={n:4d}  {a}  ->  {b}")
    sizes = sorted(g for g, _, _ in gaps)
    print("gap quantiles (us):", [round(sizes[int(q * (len(sizes) - 1))], 2) for q in (0.1, 0.5, 0.9, 0.99)])


if __name__ == "__main__":
    main()
