"""Run the VarNet 11x11 tensor-core kernels once on small shapes (debug aid)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [REPO, os.path.join(REPO, "tests")]
import numpy as np  # noqa: E402

from paper_2202_14005_b200 import load_library  # noqa: E402
from paper_2202_14005_b200.mdnn import Model  # noqa: E402
from util import d16, rrand  # noqa: E402

gpu = load_library()
X, Y, B, F = [int(a) for a in (sys.argv[1:] or ["36", "20", "2", "24"])]
rng = np.random.default_rng(0)
in_dims = list(d16(X, Y, 2))
in_dims[15] = B
n = Model.conv_layer(gpu, "c", in_dims, (11, 11), F, transposed=False, bias=False).nlop
ins = [rrand(rng, n.in_dims(i)) for i in range(2)]
y = n.apply(ins)[0]
print("fwd ok", float(np.abs(y).sum()), flush=True)
dx = n.adjoint_all(0, rrand(rng, n.out_dims(0)))[0]
print("bwd ok", float(np.abs(dx).sum()), flush=True)
