"""Diagnostics for the tcgen05 conv: delta-weight probes vs expected shifts."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from paper_2202_14005_b200 import load_library
from paper_2202_14005_b200.mdnn import Model
from util import d16

lib = load_library()
X, Y, C = 32, 16, 64
in_dims = list(d16(X, Y, C))
m = Model.conv_layer(lib, "c", in_dims, (3, 3), C)
n = m.nlop
rng = np.random.default_rng(0)
x = np.asfortranarray((rng.standard_normal(n.in_dims(0)) + 1j * rng.standard_normal(n.in_dims(0))).astype(np.complex64))

def run(w, tc):
    lib.check(lib.so.mdnn_set_option(b"conv_tc", tc))
    return n.apply([x, w])[0]

for (kx, ky) in [(1, 1), (0, 1), (2, 1), (1, 0), (0, 0)]:
    w = np.zeros(n.in_dims(1), dtype=np.complex64, order="F")
    for c in range(C):
        w[kx, ky, c, c] = 1.0
    a = run(w, 1)[:, :, :, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]
    b = run(w, 0)[:, :, :, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]
    err = np.abs(a - b)
    print(f"tap kx={kx} ky={ky}: rel {np.linalg.norm(a-b)/np.linalg.norm(b):.3e}  bad px frac {np.mean(err.max(axis=2) > 1e-2):.3f}")
    bad = np.argwhere(err.max(axis=2) > 1e-2)
    if len(bad):
        print("   first bad (x,y):", bad[:8].tolist())
        px, py = bad[0]
        # which input pixel / channel does the TC value come from?
        v = a[px, py, :]
        xs = x[:, :, :, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]
        flat = xs.reshape(-1, order="F")
        for ch in range(2):
            idx = np.argmin(np.abs(flat - v[ch]))
            ix, iy, ic = np.unravel_index(idx, xs.shape, order="F")
            print(f"   out ch{ch} = {v[ch]:.3f} best match in x at {(ix, iy, ic)} val {flat[idx]:.3f}; expected from {(px+kx-1, py+ky-1, ch)}")
    # channel mixing probe: only re part
# tap-sum probe with random weights, per output channel error profile
w = np.asfortranarray((rng.standard_normal(n.in_dims(1)) * 0.1 + 1j * rng.standard_normal(n.in_dims(1)) * 0.1).astype(np.complex64))
a, b = run(w, 1), run(w, 0)
print("random rel", np.linalg.norm(a - b) / np.linalg.norm(b))
