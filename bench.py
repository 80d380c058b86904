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

Workloads (--workload): modl_c2 (default, BASELINE configs[1]), modl_c1,
varnet_c3, modl_c5 (512x512, 32 coils, 4 items per GPU; configs[4]) and
sense_c4 (the SENSE normal operator A^H A + lambda and a 10-iteration CG solve
alone, configs[3]; unit GB/s of algorithmic bytes, with a coils x image sweep).

`--gpus N` without torchrun re-launches itself under torch.distributed.run
with N ranks (127.0.0.1); under torchrun WORLD_SIZE must equal --gpus.

`--impl reference` times the reference CPU implementation (oracle/_ref, the
unmodified reference headers compiled in place) on the host cores instead;
each step is one bounded sample of the workload (see cpu_sample()).
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
    "modl_c5": (dict(iterations=5, layers=5, filters=64, cg_iter=10), 512, 512, 32, 4),
}
# sense_c4: (X, Y, coils, items per GPU); the first shape is the headline
# value, items sized so the per-GPU working set is >= 4x L2
SENSE_C4 = [(512, 512, 32, 8), (512, 512, 16, 16), (512, 512, 8, 32), (256, 256, 32, 32), (256, 256, 16, 64),
            (256, 256, 8, 128)]
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
# Reference CPU implementation (oracle/_ref: the unmodified reference headers
# compiled in place) on the host cores -- a baseline only, never the product.
def _ref_lib():
    from paper_2202_14005_b200.capi import Lib
    path = os.path.join(REPO, "oracle", "_ref", "libmdnn_ref.so")
    return Lib(path) if os.path.exists(path) else None


def cpu_train_sample(workload):
    """One bounded sample of a training workload: the reference's own run_step
    (forward + backward + Adam, optim.hpp:314-399) at batch 1 with the
    workload's geometry and network.  Workloads with T > 1 unrolls are sampled
    with ONE unroll (the T unrolls cost the same: samples/s = 1 / (T t));
    modl_c1 (T = 1) is its full configuration.  Returns (samples/s, seconds,
    description)."""
    from paper_2202_14005_b200.mdnn import Model, Trainer
    ref = _ref_lib()
    if ref is None:
        return None
    kw, X, Y, NC, _ = WORKLOADS[workload]
    T = kw["iterations"]
    data = make_data(ref, X, Y, NC, 1, 0)
    model = (Model.varnet if workload.startswith("varnet") else Model.modl)(
        ref, **dict(kw, iterations=1, im_x=X, im_y=Y, coils=NC, batch=1))
    tr = Trainer(ref, model, seed=42)
    for k, v in data.items():
        tr.set_data(k, v)
    t0 = time.perf_counter()
    tr.step()
    dt = time.perf_counter() - t0
    what = "full step" if T == 1 else f"1 of {T} unrolls (x{T} per sample)"
    desc = f"reference fp32 run_step (Adam), {what}, batch 1, {X}x{Y}x{NC}"
    return 1.0 / (T * dt), dt, desc


def sense_bytes(X, Y, NC, B, cg=False):
    """SURVEY §8d algorithmic bytes: S apply 8 B X Y (C + 2); CG iteration 8 B X Y (C + 10)."""
    return 8.0 * B * X * Y * (NC + (10 if cg else 2))


def cpu_sense_sample(shape):
    """Reference S = A^H A + lambda (modl_normal_plus_lambda, recon.hpp:807-820)
    applied once at batch 1: algorithmic GB/s.  Returns (GB/s, seconds, desc)."""
    from util import image_dims
    ref = _ref_lib()
    if ref is None:
        return None
    X, Y, NC = shape[:3]
    ph, cm, pat = sim_inputs(ref, X, Y, NC, 1)
    y = np.zeros(image_dims(X, Y), dtype=np.complex64, order="F")
    A = [ref.arr(a) for a in (cm, pat, ph, y)]
    t0 = time.perf_counter()
    ref.check(ref.so.mdnn_sense_normal(C.byref(A[0]), C.byref(A[1]), C.c_float(0.05), C.byref(A[2]), C.byref(A[3])))
    dt = time.perf_counter() - t0
    return sense_bytes(X, Y, NC, 1) / dt / 1e9, dt, f"reference S = A^H A + lambda apply, batch 1, {X}x{Y}x{NC}"


def sim_inputs(lib, X, Y, NC, B, first_item=0):
    d = make_data(lib, X, Y, NC, B, first_item)
    return d["reference"], d["coils"], d["pattern"]


def cpu_sample(workload):
    if workload == "sense_c4":
        return cpu_sense_sample(SENSE_C4[0])
    return cpu_train_sample(workload)


def _subprocess_samples(workload, nproc):
    """`nproc` concurrent single-threaded reference processes, one sample each
    (the P-process throughput estimate of BASELINE.md §3: the reference's SENSE
    / CG path does not scale with OpenMP threads).  Returns per-process values."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-sample-worker", workload]
    procs = [subprocess.Popen(cmd, env=env, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
             for _ in range(nproc)]
    vals = []
    for p in procs:
        out, _ = p.communicate(timeout=900)
        try:
            vals.append(json.loads(out.strip().splitlines()[-1]))
        except Exception:
            pass
    return vals


def run_reference_arm(args, rank, world):
    if rank != 0:
        return  # the reference is a single-host CPU implementation: rank 0 alone runs it
    cores = os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(cores)
    unit = "GB/s" if args.workload == "sense_c4" else "samples/s"
    n = max(1, min(args.steps, 3))  # each sample is ~1-15 s of CPU work
    vals = []
    for _ in range(n):
        r = cpu_sample(args.workload)
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libmdnn_ref.so not built"}))
            return
        vals.append(r)
    v = float(np.median([x[0] for x in vals]))
    sec = float(np.median([x[1] for x in vals]))
    cpu = {"value": v, "unit": unit, "cores": cores, "kind": "reference",
           "sample": vals[0][2] + f"; OMP threads {cores}; median of {n}", "sample_seconds": sec}
    if not args.no_thread_sweep:
        one = _subprocess_samples(args.workload, 1)
        par = _subprocess_samples(args.workload, cores)
        if one:
            cpu["single_thread"] = {"value": one[0]["value"], "unit": unit, "cores": 1,
                                    "sample_seconds": one[0]["seconds"]}
        if par:
            cpu["p_process"] = {"value": float(sum(p["value"] for p in par)), "unit": unit, "cores": cores,
                                "processes": len(par), "sample_seconds": float(max(p["seconds"] for p in par)),
                                "note": "aggregate of concurrent single-threaded reference processes on independent "
                                        "items (valid under the per-shard semantics, SURVEY §8e)"}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": unit, "n_gpus": args.gpus,
            "steps": n, "warmup": 0, "ms_per_step": 1000.0 * sec, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c64 (fp32 complex)", "data": "synthetic",
            "config": config_of(args, world=1), "cpu_baseline": cpu,
            "step_definition": "one bounded sample per step: " + vals[0][2],
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_of(args, world):
    if args.workload == "sense_c4":
        X, Y, NC, B = SENSE_C4[0]
        return {"workload": "sense_c4", "operator": "S = A^H A + lambda (lambda 0.05) and CG-10 (tol 0)",
                "image": [X, Y], "coils": NC, "batch_per_gpu": B, "global_batch": B * world,
                "sweep": [list(s) for s in SENSE_C4], "parallelism": f"replicas{world}",
                "l2": "working set >= 4x L2 per GPU (no flush)"}
    kw, X, Y, NC, B = WORKLOADS[args.workload]
    return {"workload": args.workload, "network": "varnet" if args.workload.startswith("varnet") else "modl",
            **{k: v for k, v in kw.items()}, "image": [X, Y], "coils": NC, "batch_per_gpu": B,
            "global_batch": B * world, "parallelism": f"dp{world}", "l2": "inputs > L2 (no flush)",
            "conv_arithmetic": "TF32 tensor cores (operands rounded RN to TF32), fp32 accumulate"}


def relaunch_under_torchrun(args):
    """`bench.py --gpus N` outside torchrun: one rank per GPU on this node."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="modl_c2", choices=sorted(WORKLOADS) + ["sense_c4"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-thread-sweep", action="store_true", help="reference arm: skip the 1-thread / P-process figures")
    ap.add_argument("--dp", default="library", choices=["library", "torch"],
                    help="gradient exchange for N > 1: NCCL inside the library (default) or torch.distributed")
    ap.add_argument("--cpu-sample-worker", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    sys.path.insert(0, os.path.join(REPO, "tests"))

    if args.cpu_sample_worker:
        r = cpu_sample(args.cpu_sample_worker)
        print(json.dumps({"value": r[0], "seconds": r[1]}) if r else "{}", flush=True)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}")

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2202_14005_b200 import load_library

    torch.cuda.set_device(local)
    lib = load_library()
    lib.check(lib.so.mdnn_set_device(local))
    for opt in ("sense_rank", "conv_tc", "cg_pdl", "cg_fuse", "pdl", "rbf_pair", "rbf_cut"):  # A/B switches for experiments (default: product path)
        if os.environ.get("MDNN_" + opt.upper()) is not None:
            lib.check(lib.so.mdnn_set_option(opt.encode(), int(os.environ["MDNN_" + opt.upper()])))
    stream = torch.cuda.ExternalStream(lib.so.mdnn_stream(), device=torch.device("cuda", local))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        lib.check(lib.so.mdnn_synchronize())

    def max_over_ranks(ms):
        if world > 1:
            t = torch.tensor([ms], device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    ctx = dict(torch=torch, dist=dist, lib=lib, stream=stream, rank=rank, world=world, local=local,
               barrier=barrier, max_over_ranks=max_over_ranks)
    line = (run_sense_arm if args.workload == "sense_c4" else run_train_arm)(args, ctx)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def timed(ctx, steps, fn, clk=None):
    """CUDA events on the library stream around `steps` calls of fn, barrier +
    synchronize on both sides; returns (max-over-ranks ms, launches, clocks)."""
    torch, lib, stream = ctx["torch"], ctx["lib"], ctx["stream"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_begin = clk.mark() if clk else None
    l0 = lib.so.mdnn_launch_count()
    ctx["barrier"]()
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    ctx["barrier"]()
    launches = lib.so.mdnn_launch_count() - l0
    clocks = clk.stop(t_begin, clk.mark()) if clk else None
    return ctx["max_over_ranks"](e0.elapsed_time(e1)), launches, clocks


def run_train_arm(args, ctx):
    torch, lib, stream = ctx["torch"], ctx["lib"], ctx["stream"]
    rank, world, local = ctx["rank"], ctx["world"], ctx["local"]
    from paper_2202_14005_b200.dp import DataParallelTrainer
    from paper_2202_14005_b200.mdnn import Trainer

    kw, X, Y, NC, B = WORKLOADS[args.workload]
    data = make_data(lib, X, Y, NC, B, first_item=rank * B)
    model = build_model(lib, args.workload, B)
    tr = Trainer(lib, model, seed=42)
    dpt = DataParallelTrainer(tr, world=world, device=torch.device("cuda", local), comm=args.dp, rank=rank)
    dev = {k: torch.from_numpy(np.ascontiguousarray(v.transpose())).to(f"cuda:{local}") for k, v in data.items()}
    for k, v in dev.items():
        tr.set_data(k, v)
    # pinned host copies for the end-to-end leg
    pinned = {k: torch.from_numpy(np.ascontiguousarray(v.transpose())).pin_memory() for k, v in data.items()}
    h2d = sum(int(v.numel()) * 8 for k, v in pinned.items())

    def step():
        dpt.step()  # forward + backward, gradient all-reduce (N > 1), Adam

    clk = ClockSampler(local)
    clk.start()
    for _ in range(args.warmup):
        step()
    ctx["barrier"]()
    clk.wait_first()

    # ---- device-timed region (inputs resident in HBM) --------------------
    ms, launches, clocks = timed(ctx, args.steps, step, clk)
    ms_step = ms / args.steps
    value = world * B * args.steps / (ms / 1000.0)

    # ---- per-kernel live timing: a separate profiled pass (the per-launch event
    # pairs cost host time, so they stay out of the timed region above)
    np_steps = max(1, min(args.steps, 2))
    ctx["barrier"]()
    lib.check(lib.so.mdnn_profile_reset())
    lib.check(lib.so.mdnn_profile_enable(1))
    for _ in range(np_steps):
        step()
    ctx["barrier"]()
    lib.check(lib.so.mdnn_profile_enable(0))
    roof = roofline(lib, ms_step * np_steps, args.workload)

    # ---- end-to-end leg through the public C ABI (host inputs each step) ----
    e2e = None
    if not args.no_e2e:
        # Each step's inputs cross from pinned host memory inside the timed
        # region through the trainer's prefetch queue (copy stream), so batch
        # i+1 is copied while step i computes -- the way a loader feeds
        # training.  Batch 0 is staged inside the region too.
        state = {"i": 0}

        def e2e_step():
            if state["i"] == 0:
                for k, v in pinned.items():
                    tr.stage_data(k, v)
            if state["i"] + 1 < args.steps:
                for k, v in pinned.items():
                    tr.stage_data(k, v)  # H2D copy of the next step's inputs (async)
            state["i"] += 1
            step()  # takes the oldest staged batch; loss D2H read
        me, _, _ = timed(ctx, args.steps, e2e_step)
        e2e = {"value": world * B * args.steps / (me / 1000.0), "unit": "samples/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 8, "ms_per_step": me / args.steps}

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            os.environ["OMP_NUM_THREADS"] = str(os.cpu_count())
            r = cpu_sample(args.workload)
            if r:
                cpu = {"value": r[0], "unit": "samples/s", "cores": os.cpu_count(), "kind": "reference",
                       "sample": r[2], "sample_seconds": r[1]}
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "c64 (fp32 complex; convolutions TF32-RN operands, fp32 accumulate)",
                "data": "synthetic", "config": config_of(args, world), "roofline": roof["dominant"],
                "roofline_ahha": roof["ahha"], "roofline_kernels": roof["all"], "cpu_baseline": cpu, "e2e": e2e,
                "clocks": clocks, "gpu_launches": int(launches),
                "dp": {"exchange": "nccl-in-library (bucketed, comm stream)" if world > 1 and args.dp == "library"
                       else ("torch.distributed" if world > 1 else "none"), "ranks": world}}
    return line


def run_sense_arm(args, ctx):
    """configs[3]: S = A^H A + lambda alone and a 10-iteration CG solve (tol 0),
    device arrays through the C ABI, CUDA events on the library stream.  value
    = aggregate algorithmic GB/s of the S apply at the headline shape over all
    ranks (each rank its own items: no collective); the sweep adds every shape's
    S-apply and CG-10 GB/s."""
    torch, lib = ctx["torch"], ctx["lib"]
    rank, world, local = ctx["rank"], ctx["world"], ctx["local"]
    from util import image_dims
    p, src = peaks()
    clk = ClockSampler(local)
    sweep, head = [], None
    launches = 0
    for si, (X, Y, NC, B) in enumerate(SENSE_C4):
        ph, cm, pat = sim_inputs(lib, X, Y, NC, B, first_item=rank * B) if si == 0 else _rand_inputs(X, Y, NC, B)
        dev = [torch.from_numpy(np.ascontiguousarray(a.transpose())).to(f"cuda:{local}") for a in (cm, pat, ph)]
        y = torch.zeros_like(dev[2])
        A = [lib.arr(t) for t in dev + [y]]

        def apply():
            lib.check(lib.so.mdnn_sense_normal(C.byref(A[0]), C.byref(A[1]), C.c_float(0.05), C.byref(A[2]),
                                               C.byref(A[3])))
        it, st = C.c_long(), (C.c_double * 3)()

        def solve():
            lib.check(lib.so.mdnn_cg_normal_solve(C.byref(A[0]), C.byref(A[1]), C.c_float(0.05), C.byref(A[2]), 10,
                                                  C.c_double(0.0), C.byref(A[3]), C.byref(it), st))
        for _ in range(max(3, args.warmup)):
            apply()
            solve()
        ctx["barrier"]()
        if si == 0:
            clk.start()
            clk.wait_first()
        ms, l1, clocks = timed(ctx, args.steps, apply, clk if si == 0 else None)
        n_cg = max(1, args.steps // 4)
        mcg, l2, _ = timed(ctx, n_cg, solve)
        launches += l1 + l2
        gbs = world * sense_bytes(X, Y, NC, B) * args.steps / (ms / 1e3) / 1e9
        cg_gbs = world * 10 * sense_bytes(X, Y, NC, B, cg=True) * n_cg / (mcg / 1e3) / 1e9
        row = {"image": [X, Y], "coils": NC, "batch_per_gpu": B, "apply_us": 1e3 * ms / args.steps,
               "apply_gbs": gbs, "apply_frac": gbs / world / p["hbm_gbs"], "cg10_ms": mcg / n_cg,
               "cg10_gbs": cg_gbs, "cg10_frac": cg_gbs / world / p["hbm_gbs"]}
        if si == 0:
            head = (ms, gbs, clocks, dev, A)
            # per-kernel live timing of the headline shape (profiled pass)
            lib.check(lib.so.mdnn_profile_reset())
            lib.check(lib.so.mdnn_profile_enable(1))
            for _ in range(2):
                apply()
                solve()
            ctx["barrier"]()
            lib.check(lib.so.mdnn_profile_enable(0))
            roof = roofline(lib, 0.0, "sense_c4")
        sweep.append(row)
    ms, gbs, clocks, dev, A = head
    X, Y, NC, B = SENSE_C4[0]

    # e2e: the same S apply through the C ABI on HOST arrays (H2D of coils and
    # x, D2H of the result inside the timed region, every call)
    e2e = None
    if not args.no_e2e:
        host = [t.cpu().pin_memory() for t in dev]
        hy = torch.zeros_like(host[2]).pin_memory()
        H = [lib.arr(t) for t in host + [hy]]

        def apply_host():
            lib.check(lib.so.mdnn_sense_normal(C.byref(H[0]), C.byref(H[1]), C.c_float(0.05), C.byref(H[2]),
                                               C.byref(H[3])))
        apply_host()
        n_e = max(1, args.steps // 4)
        me, _, _ = timed(ctx, n_e, apply_host)
        e2e = {"value": world * sense_bytes(X, Y, NC, B) * n_e / (me / 1e3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(sum(t.numel() * 8 for t in host)), "d2h_bytes_per_step": int(hy.numel() * 8),
               "ms_per_step": me / n_e}
    line = None
    if ctx["rank"] == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            os.environ["OMP_NUM_THREADS"] = str(os.cpu_count())
            r = cpu_sample("sense_c4")
            if r:
                cpu = {"value": r[0], "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference", "sample": r[2],
                       "sample_seconds": r[1]}
        line = {"metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "c64 (fp32 complex)", "data": "synthetic",
                "config": config_of(args, world), "roofline": roof["dominant"], "roofline_ahha": roof["ahha"],
                "roofline_kernels": roof["all"], "sweep": sweep, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
                "gpu_launches": int(launches)}
    return line


def _rand_inputs(X, Y, NC, B):
    """Sweep shapes past the headline: random unit-normalised coils, random
    image, the 4x + 28 ACL pattern (timing only)."""
    from util import coil_dims, image_dims, pattern_dims
    rng = np.random.default_rng(X * 1000 + NC)
    cm = (rng.standard_normal(coil_dims(X, Y, NC, B)) + 1j * rng.standard_normal(coil_dims(X, Y, NC, B)))
    cm /= np.sqrt((np.abs(cm) ** 2).sum(axis=3, keepdims=True))
    ph = rng.standard_normal(image_dims(X, Y, B)) + 1j * rng.standard_normal(image_dims(X, Y, B))
    pat = np.zeros(pattern_dims(Y), dtype=np.complex64)
    pv = pat.reshape(-1)
    for i in range(Y):
        if i % 4 == 0 or min(i, Y - i) < 14:
            pv[i] = 1
    f = lambda a: np.asfortranarray(a.astype(np.complex64))  # noqa: E731
    return f(ph), f(cm), f(pat)


def roofline(lib, step_ms_total, workload="modl_c2"):
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
    tf32, tf32_src = 1100.0, "nominal tf32 dense 1.1 PFLOP/s (B200_PROFILING.md)"
    # second denominator for the tensor-bound rows: the TF32 rate measured on
    # this pool (cuBLAS fp32 GEMM with TF32 tensor cores, profiles/tf32_peak.json),
    # else half the measured bf16 rate of MEASURED_PEAKS.json
    tf32_meas, tf32_meas_src = None, None
    try:
        with open(os.path.join(REPO, "profiles", "tf32_peak.json")) as f:
            tf32_meas = float(json.load(f)["tf32_tflops"])
            tf32_meas_src = "cuBLAS TF32 GEMM 8192^3 measured on this pool (profiles/tf32_peak.json)"
    except Exception:
        if "bf16_tflops" in p:
            tf32_meas, tf32_meas_src = p["bf16_tflops"] / 2, "bf16_tflops / 2 (MEASURED_PEAKS.json)"
    traffic = {}
    try:
        # per-launch DRAM bytes of each tag from one ncu capture of THIS workload
        # (tools/ncu_traffic.py); other workloads report traffic = null
        with open(os.path.join(REPO, "profiles", f"ncu_traffic_{workload}.json")) as f:
            traffic = json.load(f)
    except Exception:
        pass
    tags = {"sense_normal_y_cg": "hbm", "sense_normal_y": "hbm", "cg_update_rank": "hbm", "fft": "hbm", "conv_fwd": "tensor",
            "conv_bwd_data": "tensor", "conv_bwd_weight": "tensor", "conv_tc_fwd": "tensor",
            # VarNet 11x11 layers: 2-channel side, memory-bound (bytes); flops rows alongside (_tf)
            "conv_vn_fwd": "hbm", "conv_vn_bwd_data": "hbm", "conv_vn_bwd_weight": "hbm",
            "conv_vn_fwd_tf": "tensor", "conv_vn_bwd_data_tf": "tensor", "conv_vn_bwd_weight_tf": "tensor",
            "rbf": "hbm", "rbf_adjoint": "hbm",
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
                     "share_of_step_time": ms.value / step_ms_total if step_ms_total > 0 else None,
                     "traffic": traffic.get(tag), "peak_source": f"measured hbm_gbs ({src})" if bound == "hbm" else tf32_src})
        if bound == "tensor" and tf32_meas:
            rows[-1].update({"peak_measured": tf32_meas, "frac_vs_measured": ach / tf32_meas,
                             "peak_measured_source": tf32_meas_src})
    names = {r["kernel"] for r in rows}
    # the generic conv_* scopes wrap the VarNet kernels (plus their operand checks):
    # report the inner rows only; the _tf rows repeat the same launches in flops
    rows = [r for r in rows if not (r["kernel"] in ("conv_fwd", "conv_bwd_data", "conv_bwd_weight")
                                    and "conv_vn_" + r["kernel"][5:] in names)]
    rows.sort(key=lambda r: -r["ms_total"])
    dom = next((r for r in rows if not r["kernel"].endswith("_tf")), None)
    ahha = next((r for r in rows if r["kernel"].startswith("sense_normal_y")), None)
    return {"dominant": dom, "ahha": ahha, "all": rows}


if __name__ == "__main__":
    main()
