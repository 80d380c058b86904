"""Small-shape workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck) over the hand-written TMA / mbarrier / tcgen05 kernels:
the channel-major and CTA-pair tensor-core convolutions (fwd, bwd-data with
the BN-backward epilogue, bwd-weight), the thin tensor-core layers, the fused
BN block, the warp-specialised A^H A kernel (W = 8 and W = 4 strips, contiguous,
split and round-robin unit assignments) and the round-1 rank kernel with the
device CG, the VarNet 11x11 tensor-core convolutions, the windowed RBF, and one
MoDL training step.  Runs on the product library only (no oracle).

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import ctypes as C
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "tests")]
import numpy as np  # noqa: E402

from paper_2202_14005_b200 import load_library  # noqa: E402
from paper_2202_14005_b200.mdnn import Model, Trainer, sense_dims  # noqa: E402
from paper_2202_14005_b200.mdnn import Nlop  # noqa: E402
from util import crand, d16, image_dims, kspace_dims, rrand  # noqa: E402

gpu = load_library()
gpu.check(gpu.so.mdnn_set_device(0))
rng = np.random.default_rng(0)


def conv(cin, cout, X, Y, B):
    dims = list(d16(X, Y, cin))
    dims[15] = B
    n = Model.conv_layer(gpu, "c", dims, (3, 3), cout).nlop
    ins = [crand(rng, n.in_dims(i)) for i in range(n.n_in)]
    n.apply(ins)
    n.adjoint_all(0, crand(rng, n.out_dims(0)))


for cin, cout in ((64, 64), (32, 32), (1, 64), (64, 1)):
    conv(cin, cout, 24, 40, 2)
    print("conv", cin, cout, "ok", flush=True)

# fused denoiser (conv-epilogue BN statistics, BN backward in the bwd-data epilogue)
kw = dict(iterations=1, layers=5, filters=64, im_x=24, im_y=40, coils=2, batch=2)
m = Model.modl_denoiser(gpu, **kw)
n = m.nlop
w = m.init_weights(1)
x0 = crand(rng, image_dims(24, 40, 2))
ins = [x0 if a not in w else w[a] for a, _, _ in m.args]
n.apply(ins)
o = m.output_index("out")
n.adjoint_all(o, crand(rng, n.out_dims(o)))
print("denoiser ok", flush=True)

# A^H A kernels + CG solve: ws (default), ws with split strips (3 CTAs), the
# round-1 rank kernel; 368 = 16 x 23 rows (W = 8) and 512 = 16 x 32 (W = 4, round robin)
def sense(X, Y, NC, opts):
    for k, v in opts:
        gpu.check(gpu.so.mdnn_set_option(k, v))
    pat = np.zeros(d16(1, Y), dtype=np.complex64, order="F")
    gpu.check(gpu.so.mdnn_sim_pattern(Y, 4, 28, pat.ctypes.data))
    cm = crand(rng, d16(X, Y, 1, NC))
    ph = crand(rng, image_dims(X, Y))
    y = np.zeros(image_dims(X, Y), dtype=np.complex64, order="F")
    gpu.check(gpu.so.mdnn_sense_normal(C.byref(gpu.arr(cm)), C.byref(gpu.arr(pat)), C.c_float(0.05),
                                       C.byref(gpu.arr(ph)), C.byref(gpu.arr(y))))
    x = np.zeros(image_dims(X, Y), dtype=np.complex64, order="F")
    it, st = C.c_long(), (C.c_double * 3)()
    gpu.check(gpu.so.mdnn_cg_normal_solve(C.byref(gpu.arr(cm)), C.byref(gpu.arr(pat)), C.c_float(0.05),
                                          C.byref(gpu.arr(ph)), 5, C.c_double(0.0), C.byref(gpu.arr(x)),
                                          C.byref(it), st))
    for k, _ in opts:
        gpu.check(gpu.so.mdnn_set_option(k, {b"sense_ws": 1, b"sense_rank_ctas": 0, b"rank_rr": 1}[k]))
    return pat


pat = sense(16, 368, 3, [])
sense(36, 368, 3, [(b"sense_rank_ctas", 3)])
sense(16, 368, 3, [(b"sense_ws", 0)])
sense(36, 512, 3, [])
sense(36, 512, 3, [(b"rank_rr", 0), (b"sense_rank_ctas", 3)])
print("sense ok", flush=True)

# VarNet 11x11 tensor-core convolutions (real operands: 2 -> 24 -> 2) and the windowed RBF
for cin, cout in ((2, 24), (24, 2)):
    dims = list(d16(24, 40, cin))
    dims[15] = 2
    n = Model.conv_layer(gpu, "v", dims, (11, 11), cout).nlop
    ins = [rrand(rng, n.in_dims(i), 1.0) for i in range(n.n_in)]
    n.apply(ins)
    n.adjoint_all(0, rrand(rng, n.out_dims(0), 1.0))
z = list(d16(24, 40, 6))
centers = [-1 + 2 * j / 30 for j in range(31)]
r = Nlop.rbf(gpu, z, 2, centers, 2 / 30)
r.apply([rrand(rng, z, 1.5), rrand(rng, r.in_dims(1), 0.05)])
r.adjoint_all(0, rrand(rng, r.out_dims(0), 1.0))
print("varnet convs + rbf ok", flush=True)

# one MoDL training step (F = 64: channel-major conv, thin layers, BN block, CG)
kw = dict(iterations=1, layers=3, filters=64, cg_iter=3, im_x=16, im_y=368, coils=2, batch=1)
t = Trainer(gpu, Model.modl(gpu, **kw), seed=1)
cm = crand(rng, d16(16, 368, 1, 2))
ph = crand(rng, image_dims(16, 368))
ks = np.zeros(kspace_dims(16, 368, 2), dtype=np.complex64, order="F")
gpu.check(gpu.so.mdnn_sense_forward(C.byref(gpu.arr(cm)), C.byref(gpu.arr(pat)), C.byref(gpu.arr(ph)),
                                    C.byref(gpu.arr(ks))))
for k, v in (("kspace", ks), ("coils", cm), ("pattern", pat), ("reference", ph)):
    t.set_data(k, v)
t.step()
gpu.check(gpu.so.mdnn_synchronize())
print("train step ok", flush=True)
