#!/usr/bin/env python
"""Benchmark: MoDL training samples/s on B200 (BASELINE.json metric).

Default workload (configs[1]): MoDL, 5 unrolls x 10 CG iterations, 5-layer
64-channel complex CNN, synthetic 15-coil 320x368 k-space, batch 8 per GPU.
Data parallel over N GPUs (torchrun, one process per GPU): every rank trains
its own batch shard, the flat fp32 weight-gradient buffer is all-reduced with
NCCL on the library's stream, and every rank applies the same Adam update.

One JSON line on rank 0 (contract in the task statement):
  value  : whole-job samples/s, device-timed (CUDA events on the library
           stream, max over ranks), inputs resident in HBM (> L2: 226 MB of
           k-space + coils per GPU, so no L2 flush is needed)
  e2e    : same metric through the public C ABI with this step's inputs copied
           from pinned host memory inside the timed region and the loss read back
  roofline, cpu_baseline, clocks, gpu_launches

`--impl reference` times the reference CPU implementation (oracle/_ref, the
unmodified reference headers compiled in place) on the host cores instead.
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOADS = {
    # name: (builder kwargs, geometry X, Y, coils, per-GPU batch)
    "modl_c2": (dict(iterations=5, layers=5, filters=64, cg_iter=10), 320, 368, 15, 8),
    "modl_c1": (dict(iterations=1, layers=3, filters=32, cg_iter=5), 128, 128, 8, 1),
    "varnet_c3": (dict(iterations=10, filters=24, kernel=11, rbf=31), 640, 368, 15, 4),
}
METRIC = "MoDL/VarNet train samples/s @1/2/4/8 B200; A^HA GB/s vs HBM peak"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


# ---------------------------------------------------------------------------
def make_data(lib, X, Y, NC, B, first_item, seed=1):
    """Synthetic knee-shaped data (simulate.hpp:119-167 generators): phantom,
    unit-normalised smooth coils, 4x regular + 28 ACL pattern, k-space =
    P (F C x + CN(0, 0.001^2))."""
    from util import coil_dims, image_dims, kspace_dims, pattern_dims  # noqa: F401
    ph = np.zeros(image_dims(X, Y, B), dtype=np.complex64, order="F")
    cm = np.zeros(coil_dims(X, Y, NC, B), dtype=np.complex64, order="F")
    for s in range(B):
        p1 = np.zeros((X, Y), dtype=np.complex64, order="F")
        c1 = np.zeros((X, Y, NC), dtype=np.complex64, order="F")
        lib.check(lib.so.mdnn_sim_item(seed, first_item + s, X, Y, NC, p1.ctypes.data, c1.ctypes.data))
        ph[:, :, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, s] = p1
        cm[:, :, 0, :, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, s] = c1
    pat = np.zeros(pattern_dims(Y), dtype=np.complex64, order="F")
    lib.check(lib.so.mdnn_sim_pattern(Y, 4, 28, pat.ctypes.data))
    ks = np.zeros(kspace_dims(X, Y, NC, B), dtype=np.complex64, order="F")
    lib.check(lib.so.mdnn_sense_forward(C.byref(lib.arr(cm)), C.byref(lib.arr(pat)), C.byref(lib.arr(ph)),
                                        C.byref(lib.arr(ks))))
    rng = np.random.default_rng(0x6E015E + first_item)
    noise = (rng.standard_normal(ks.shape) + 1j * rng.standard_normal(ks.shape)).astype(np.complex64) * 1e-3
    ks = np.asfortranarray((ks + noise) * pat.reshape((1, Y) + (1,) * 14, order="F"))
    return {"kspace": ks, "coils": cm, "pattern": pat, "reference": ph}


def build_model(lib, workload, B):
    from paper_2202_14005_b200.mdnn import Model
    kw, X, Y, NC, _ = WORKLOADS[workload]
    kw = dict(kw, im_x=X, im_y=Y, coils=NC, batch=B)
    return (Model.varnet if workload.startswith("varnet") else Model.modl)(lib, **kw)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def wait_first(self, timeout=5.0):
        t0 = time.monotonic()
        while self.proc and not self.lines and time.monotonic() - t0 < timeout:
            time.sleep(0.05)

    def mark(self):
        return time.monotonic()

    def stop(self, t_begin=None, t_end=None):
        """Samples inside [t_begin, t_end] (plus the nearest one on each side,
        so a short timed region still has its bracketing samples)."""
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        time.sleep(0.25)  # one more sample after the region
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        lines = self.lines
        if t_begin is not None and lines:
            inside = [k for k, (t, _) in enumerate(lines) if t_begin <= t <= t_end]
            before = [k for k, (t, _) in enumerate(lines) if t < t_begin][-1:]
            after = [k for k, (t, _) in enumerate(lines) if t > t_end][:1]
            lines = [lines[k] for k in before + inside + after]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
def cpu_sample(workload):
    """Reference CPU implementation on the host cores (oracle/_ref, all
    threads): one training step of ONE unroll at batch 1 and the workload's
    geometry; the full step is T unrolls of identical cost, so samples/s is
    extrapolated as 1 / (T * t).  Returns (samples/s, seconds, description)."""
    from paper_2202_14005_b200.capi import Lib
    from paper_2202_14005_b200.mdnn import Trainer
    path = os.path.join(REPO, "oracle", "_ref", "libmdnn_ref.so")
    if not os.path.exists(path):
        return None
    ref = Lib(path)
    kw, X, Y, NC, _ = WORKLOADS[workload]
    T = kw["iterations"]
    data = make_data(ref, X, Y, NC, 1, 0)
    sample_kw = dict(kw, iterations=1, im_x=X, im_y=Y, coils=NC, batch=1)
    from paper_2202_14005_b200.mdnn import Model
    model = (Model.varnet if workload.startswith("varnet") else Model.modl)(ref, **sample_kw)
    tr = Trainer(ref, model, seed=42)
    for k, v in data.items():
        tr.set_data(k, v)
    t0 = time.perf_counter()
    tr.step()
    dt = time.perf_counter() - t0
    desc = (f"reference fp32 train step (Adam) of 1 of {T} unrolls, batch 1, {X}x{Y}x{NC} "
            f"(x{T} extrapolated per sample), OMP threads={os.environ.get('OMP_NUM_THREADS', os.cpu_count())}")
    return 1.0 / (T * dt), dt, desc


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
    kw, X, Y, NC, B = WORKLOADS[args.workload]
    vals = []
    n = max(1, min(args.steps, 2))  # each sample is ~10-60 s of CPU work
    for _ in range(n):
        r = cpu_sample(args.workload)
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libmdnn_ref.so not built"}))
            return
        vals.append(r)
    v = float(np.median([x[0] for x in vals]))
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": n, "warmup": 0, "ms_per_step": 1000.0 / v, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c64 (fp32)", "data": "synthetic",
            "config": config_of(args, B, world=1),
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "reference",
                             "sample": vals[0][2]},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_of(args, B, world):
    kw, X, Y, NC, _ = WORKLOADS[args.workload]
    return {"workload": args.workload, "network": "varnet" if args.workload.startswith("varnet") else "modl",
            **{k: v for k, v in kw.items()}, "image": [X, Y], "coils": NC, "batch_per_gpu": B,
            "global_batch": B * world, "parallelism": f"dp{world}", "l2": "inputs > L2 (no flush)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="modl_c2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, os.path.join(REPO, "tests"))

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2202_14005_b200 import load_library
    from paper_2202_14005_b200.dp import DataParallelTrainer
    from paper_2202_14005_b200.mdnn import Trainer

    torch.cuda.set_device(local)
    lib = load_library()
    lib.check(lib.so.mdnn_set_device(local))
    for opt in ("sense_rank", "conv_tc"):  # A/B switches for experiments (default: product path)
        if os.environ.get("MDNN_" + opt.upper()) is not None:
            lib.check(lib.so.mdnn_set_option(opt.encode(), int(os.environ["MDNN_" + opt.upper()])))
    stream = torch.cuda.ExternalStream(lib.so.mdnn_stream(), device=torch.device("cuda", local))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    kw, X, Y, NC, B = WORKLOADS[args.workload]
    data = make_data(lib, X, Y, NC, B, first_item=rank * B)
    model = build_model(lib, args.workload, B)
    tr = Trainer(lib, model, seed=42)
    dpt = DataParallelTrainer(tr, world=world, device=torch.device("cuda", local))
    dev = {k: torch.from_numpy(np.ascontiguousarray(v.transpose())).to(f"cuda:{local}") for k, v in data.items()}
    for k, v in dev.items():
        tr.set_data(k, v)
    # pinned host copies for the end-to-end leg
    pinned = {k: torch.from_numpy(np.ascontiguousarray(v.transpose())).pin_memory() for k, v in data.items()}
    h2d = sum(int(v.numel()) * 8 for k, v in pinned.items())

    def step():
        dpt.step()  # forward + backward, NCCL all-reduce on the library stream, Adam

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        lib.check(lib.so.mdnn_synchronize())

    clk = ClockSampler(local)
    clk.start()
    for _ in range(args.warmup):
        step()
    barrier()
    clk.wait_first()

    # ---- device-timed region (inputs resident in HBM) --------------------
    t_begin = clk.mark()
    l0 = lib.so.mdnn_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    launches = lib.so.mdnn_launch_count() - l0
    clocks = clk.stop(t_begin, clk.mark())
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = world * B * args.steps / (ms / 1000.0)

    # ---- per-kernel live timing: a separate profiled pass (the per-launch event
    # pairs cost host time, so they stay out of the timed region above)
    np_steps = max(1, min(args.steps, 2))
    barrier()
    lib.check(lib.so.mdnn_profile_reset())
    lib.check(lib.so.mdnn_profile_enable(1))
    for _ in range(np_steps):
        step()
    barrier()
    lib.check(lib.so.mdnn_profile_enable(0))
    roof = roofline(lib, ms_step * np_steps)

    # ---- end-to-end leg through the public C ABI (host inputs each step) ----
    e2e = None
    if not args.no_e2e:
        # Each step's inputs cross from pinned host memory inside the timed
        # region; they go through the trainer's prefetch queue (copy stream),
        # so batch i+1 is copied while step i computes -- the way a loader
        # feeds training.  Batch 0 is staged inside the region too.
        barrier()
        e0.record(stream)
        for k, v in pinned.items():
            tr.stage_data(k, v)
        for i in range(args.steps):
            if i + 1 < args.steps:
                for k, v in pinned.items():
                    tr.stage_data(k, v)     # H2D copy of the next step's inputs (async)
            step()                          # takes the oldest staged batch; loss D2H read
        e1.record(stream)
        barrier()
        me = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([me], device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            me = float(t.item())
        e2e = {"value": world * B * args.steps / (me / 1000.0), "unit": "samples/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 8, "ms_per_step": me / args.steps}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
            r = cpu_sample(args.workload)
            if r:
                cpu = {"value": r[0], "unit": "samples/s", "cores": int(os.environ["OMP_NUM_THREADS"]),
                       "kind": "reference", "sample": r[2], "sample_seconds": r[1]}
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "c64 (fp32 complex)", "data": "synthetic",
                "config": config_of(args, B, world), "roofline": roof["dominant"],
                "roofline_ahha": roof["ahha"], "roofline_kernels": roof["all"], "cpu_baseline": cpu, "e2e": e2e,
                "clocks": clocks,
                "gpu_launches": int(launches)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def roofline(lib, step_ms_total):
    """Per-kernel live timing (CUDA events around each tagged launch on the
    library stream, from the profiled pass): achieved = algorithmic work per
    launch / mean launch duration; share = kernel ms / (unprofiled step time x
    profiled steps).  The dominant kernel is the one with the largest share;
    `ahha` is the fused A^H A kernel the metric names."""
    p, src = peaks()
    hbm = p["hbm_gbs"]
    # dense TF32 tensor peak: MEASURED_PEAKS.json has none, and our own TF32
    # kernels beat the cuBLAS TF32 figure measured on this pool
    # (profiles/tf32_peak.json, 741 TFLOP/s burst), so the denominator is the
    # nominal dense TF32 rate of B200_PROFILING.md (1.1 PFLOP/s)
    tf32, tf32_src = 1100.0, "nominal tf32 dense 1.1 PFLOP/s (B200_PROFILING.md; cuBLAS TF32 measured 741)"
    traffic = {}
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f)
    except Exception:
        pass
    tags = {"sense_normal_y_cg": "hbm", "sense_normal_y": "hbm", "cg_update_rank": "hbm", "fft": "hbm", "conv_fwd": "tensor",
            "conv_bwd_data": "tensor", "conv_bwd_weight": "tensor", "conv_tc_fwd": "tensor",
            "conv_tc_bwd_data": "tensor", "conv_tc_bwd_weight": "tensor", "conv_thin_fwd": "hbm",
            "conv_thin_bwd_data": "hbm", "conv_thin_bwd_weight": "hbm", "bnblock_fwd": "hbm", "bnblock_bwd": "hbm"}
    rows = []
    for tag, bound in tags.items():
        n, ms, work = C.c_long(), C.c_double(), C.c_double()
        lib.check(lib.so.mdnn_profile_read(tag.encode(), C.byref(n), C.byref(ms), C.byref(work)))
        if n.value == 0 or ms.value <= 0:
            continue
        if bound == "hbm":
            ach = work.value / (ms.value / 1e3) / 1e9
            peak, unit = hbm, "GB/s"
        else:
            ach = work.value / (ms.value / 1e3) / 1e12
            peak, unit = tf32, "TFLOP/s"
        rows.append({"kernel": tag, "bound": bound, "achieved": ach, "peak": peak, "unit": unit,
                     "frac": ach / peak, "launches": n.value, "ms_total": ms.value,
                     "share_of_step_time": ms.value / step_ms_total,
                     "traffic": traffic.get(tag), "peak_source": f"measured hbm_gbs ({src})" if bound == "hbm" else tf32_src})
    rows.sort(key=lambda r: -r["ms_total"])
    dom = rows[0] if rows else None
    ahha = next((r for r in rows if r["kernel"].startswith("sense_normal_y")), None)
    return {"dominant": dom, "ahha": ahha, "all": rows}


if __name__ == "__main__":
    main()
