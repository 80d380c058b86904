"""C4-style SENSE micro-benchmark: S = A^H A + lambda and a 10-iteration CG
solve through the C ABI on device arrays, CUDA-event timed on the library
stream.  Prints one line per shape with algorithmic GB/s:
  S apply: 8 B X Y (C + 2);  CG iteration: 8 B X Y (C + 10).
Usage: python tools/sense_bench.py [X Y C B ...] [--iters N] [--cg 0/1]"""
import argparse
import ctypes as C
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shape", nargs="*", type=int, default=[320, 368, 15, 8])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--cg", type=int, default=1)
    ap.add_argument("--apply", type=int, default=1)
    ap.add_argument("--opt", action="append", default=[], help="library option key=value (mdnn_set_option)")
    args = ap.parse_args()
    import torch
    from paper_2202_14005_b200 import load_library
    from util import coil_dims, image_dims, pattern_dims

    lib = load_library()
    lib.check(lib.so.mdnn_set_device(0))
    for kv in args.opt:
        k, v = kv.split("=")
        lib.check(lib.so.mdnn_set_option(k.encode(), int(v)))
    stream = torch.cuda.ExternalStream(lib.so.mdnn_stream(), device=torch.device("cuda", 0))
    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(REPO, "MEASURED_PEAKS.json")) else 6650.0
    sh = args.shape
    for k in range(0, len(sh), 4):
        X, Y, NC, B = sh[k:k + 4]
        g = torch.Generator(device="cuda").manual_seed(0)
        cm = torch.randn(tuple(reversed(coil_dims(X, Y, NC, B))), dtype=torch.complex64, device="cuda", generator=g)
        cm /= cm.abs().pow(2).sum(dim=12, keepdim=True).sqrt()  # ref dim 3 (coil) = torch dim 12
        x = torch.randn(tuple(reversed(image_dims(X, Y, B))), dtype=torch.complex64, device="cuda", generator=g)
        y = torch.zeros_like(x)
        pat = torch.zeros(tuple(reversed(pattern_dims(Y))), dtype=torch.complex64)
        pv = pat.view(-1)
        for i in range(Y):
            d = min(i, Y - i)
            if i % 4 == 0 or d < 14:
                pv[i] = 1
        pat = pat.cuda()
        A = [lib.arr(t) for t in (cm, pat, x, y)]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        res = {"X": X, "Y": Y, "coils": NC, "B": B}
        if args.apply:
            for _ in range(3):
                lib.check(lib.so.mdnn_sense_normal(C.byref(A[0]), C.byref(A[1]), C.c_float(0.05), C.byref(A[2]),
                                                   C.byref(A[3])))
            lib.check(lib.so.mdnn_synchronize())
            e0.record(stream)
            for _ in range(args.iters):
                lib.check(lib.so.mdnn_sense_normal(C.byref(A[0]), C.byref(A[1]), C.c_float(0.05), C.byref(A[2]),
                                                   C.byref(A[3])))
            e1.record(stream)
            lib.check(lib.so.mdnn_synchronize())
            ms = e0.elapsed_time(e1) / args.iters
            gb = 8.0 * B * X * Y * (NC + 2) / 1e9
            res.update(apply_us=1e3 * ms, apply_gbs=gb / (ms / 1e3), apply_frac=gb / (ms / 1e3) / peak)
        if args.cg:
            it = C.c_long()
            st = (C.c_double * 3)()

            def solve():
                lib.check(lib.so.mdnn_cg_normal_solve(C.byref(A[0]), C.byref(A[1]), C.c_float(0.05), C.byref(A[2]),
                                                      10, C.c_double(0.0), C.byref(A[3]), C.byref(it), st))
            for _ in range(2):
                solve()
            lib.check(lib.so.mdnn_synchronize())
            n = max(1, args.iters // 4)
            e0.record(stream)
            for _ in range(n):
                solve()
            e1.record(stream)
            lib.check(lib.so.mdnn_synchronize())
            ms = e0.elapsed_time(e1) / n
            gb = 10 * 8.0 * B * X * Y * (NC + 10) / 1e9
            res.update(cg10_ms=ms, cg10_gbs=gb / (ms / 1e3), cg10_frac=gb / (ms / 1e3) / peak, cg_iters=it.value)
            # per-kernel device times from a separate profiled pass (events cost launch gaps)
            lib.check(lib.so.mdnn_profile_reset())
            lib.check(lib.so.mdnn_profile_enable(1))
            for _ in range(n):
                solve()
            lib.check(lib.so.mdnn_synchronize())
            cnt, tms, work = C.c_long(), C.c_double(), C.c_double()
            for tag in ("sense_normal_y_cg", "cg_update_rank"):
                lib.check(lib.so.mdnn_profile_read(tag.encode(), C.byref(cnt), C.byref(tms), C.byref(work)))
                if cnt.value:
                    res[tag + "_us"] = 1e3 * tms.value / cnt.value
                    res[tag + "_gbs"] = work.value / (tms.value / 1e3) / 1e9
            lib.check(lib.so.mdnn_profile_enable(0))
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
