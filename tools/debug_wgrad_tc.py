import sys, os
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np
from paper_2202_14005_b200 import load_library
from paper_2202_14005_b200.mdnn import Model
from util import d16
lib = load_library()
X, Y, C = 64, 8, 64
m = Model.conv_layer(lib, "c", list(d16(X, Y, C)), (3, 3), C)
n = m.nlop
rng = np.random.default_rng(0)
x = np.asfortranarray((rng.standard_normal(n.in_dims(0)) + 1j * rng.standard_normal(n.in_dims(0))).astype(np.complex64))
w = np.asfortranarray((0.05 * rng.standard_normal(n.in_dims(1))).astype(np.complex64))
dy = np.asfortranarray((rng.standard_normal(n.out_dims(0)) + 1j * rng.standard_normal(n.out_dims(0))).astype(np.complex64))
res = {}
for tc in (1, 0):
    lib.check(lib.so.mdnn_set_option(b"conv_tc", tc))
    n.apply([x, w])
    res[tc] = n.adjoint_all(0, dy)[1]
a, b = res[1], res[0]
print("norms tc", np.linalg.norm(a), "cuda", np.linalg.norm(b))
for t in range(9):
    kx, ky = t % 3, t // 3
    at, bt = a[kx, ky], b[kx, ky]
    print(f"tap {kx},{ky}: |tc| {np.linalg.norm(at):.3f} |ref| {np.linalg.norm(bt):.3f} rel {np.linalg.norm(at-bt)/np.linalg.norm(bt):.3e}")
print("tc[0,0,:4,:4]", a[1,1,:3,:3])
print("ref[0,0,:4,:4]", b[1,1,:3,:3])
