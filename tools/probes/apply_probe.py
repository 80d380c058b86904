"""Standalone S-apply cost split: live per-kernel time of the A^H A launch
inside mdnn_sense_normal (profile events) vs the whole call (events around
the C-ABI call).  Usage: python tools/probes/apply_probe.py [X Y C B]"""
import ctypes as C
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main():
    import torch
    from paper_2202_14005_b200 import load_library
    from util import coil_dims, image_dims, pattern_dims
    X, Y, NC, B = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (320, 368, 15, 8)))
    lib = load_library()
    lib.check(lib.so.mdnn_set_device(0))
    g = torch.Generator(device="cuda").manual_seed(0)
    cm = torch.randn(tuple(reversed(coil_dims(X, Y, NC, B))), dtype=torch.complex64, device="cuda", generator=g)
    x = torch.randn(tuple(reversed(image_dims(X, Y, B))), dtype=torch.complex64, device="cuda", generator=g)
    y = torch.zeros_like(x)
    pat = torch.zeros(tuple(reversed(pattern_dims(Y))), dtype=torch.complex64)
    pv = pat.view(-1)
    for i in range(Y):
        if i % 4 == 0 or min(i, Y - i) < 14:
            pv[i] = 1
    pat = pat.cuda()
    A = [lib.arr(t) for t in (cm, pat, x, y)]

    def apply():
        lib.check(lib.so.mdnn_sense_normal(C.byref(A[0]), C.byref(A[1]), C.c_float(0.05), C.byref(A[2]),
                                           C.byref(A[3])))
    for _ in range(3):
        apply()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        apply()
    e1.record()
    torch.cuda.synchronize()
    call_us = e0.elapsed_time(e1) * 1e3 / n
    lib.check(lib.so.mdnn_profile_reset())
    lib.check(lib.so.mdnn_profile_enable(1))
    for _ in range(n):
        apply()
    lib.check(lib.so.mdnn_profile_enable(0))
    out = {}
    for tag in ("sense_normal_y", "sense_normal_y_cg"):
        l, ms, w = C.c_long(), C.c_double(), C.c_double()
        lib.check(lib.so.mdnn_profile_read(tag.encode(), C.byref(l), C.byref(ms), C.byref(w)))
        if l.value:
            out[tag] = (l.value, 1e3 * ms.value / l.value)
    print(f"{X}x{Y}x{NC}x{B}: call {call_us:.1f} us; kernels {out}")


if __name__ == "__main__":
    main()
