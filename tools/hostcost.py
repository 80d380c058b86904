import ctypes as C, time, sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import torch
from paper_2202_14005_b200 import load_library
from util import coil_dims, image_dims, pattern_dims
lib = load_library(); lib.check(lib.so.mdnn_set_device(0))
X, Y, NC, B = 320, 368, 15, 8
cm = torch.randn(tuple(reversed(coil_dims(X, Y, NC, B))), dtype=torch.complex64, device="cuda")
x = torch.randn(tuple(reversed(image_dims(X, Y, B))), dtype=torch.complex64, device="cuda")
y = torch.zeros_like(x)
pat = torch.ones(tuple(reversed(pattern_dims(Y))), dtype=torch.complex64, device="cuda")
A = [lib.arr(t) for t in (cm, pat, x, y)]
it = C.c_long(); st = (C.c_double * 3)()
for rank in (1, 0, 1):
    lib.check(lib.so.mdnn_set_option(b"sense_rank", rank))
    for _ in range(3):
        lib.check(lib.so.mdnn_cg_normal_solve(C.byref(A[0]), C.byref(A[1]), C.c_float(0.05), C.byref(A[2]), 10, C.c_double(0.0), C.byref(A[3]), C.byref(it), st))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        lib.check(lib.so.mdnn_cg_normal_solve(C.byref(A[0]), C.byref(A[1]), C.c_float(0.05), C.byref(A[2]), 10, C.c_double(0.0), C.byref(A[3]), C.byref(it), st))
    t1 = time.perf_counter()
    print("rank", rank, "solve wall ms", (t1 - t0) * 100, flush=True)
