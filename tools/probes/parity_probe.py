"""Investigation: error of the GPU path and of the fp32 reference against the
fp64 reference for the config-level cases (prints a table)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [REPO, os.path.join(REPO, "tests")]
import numpy as np  # noqa: E402

from paper_2202_14005_b200 import load_library  # noqa: E402
from paper_2202_14005_b200.capi import Lib  # noqa: E402
from paper_2202_14005_b200.mdnn import ARG_DATA, Model  # noqa: E402
import test_gpu_configs as T  # noqa: E402
from util import crand, d16, rel_l2  # noqa: E402

gpu = load_library()
ref = Lib(os.path.join(REPO, "oracle/_ref/libmdnn_ref.so"))
ref64 = Lib(os.path.join(REPO, "oracle/_ref/libmdnn_ref64.so"))


def table(title, res):
    (og, gg), (orf, gr), (o64, g64) = res
    print("==", title)
    for k in o64:
        print(f"  out  {k:24s} gpu {rel_l2(og[k], o64[k]):.3e}  ref32 {rel_l2(orf[k], o64[k]):.3e}")
    for k in g64:
        print(f"  grad {k:24s} gpu {rel_l2(gg[k], g64[k]):.3e}  ref32 {rel_l2(gr[k], g64[k]):.3e}")


def c1(conv_tc):
    for k in ("conv_tc", "conv_thin_tc"):
        gpu.check(gpu.so.mdnn_set_option(k.encode(), conv_tc))
    data = T._c1_data(ref)
    res = []
    for lib in (gpu, ref, ref64):
        m = Model.modl(lib, **T.C1)
        w = T._perturbed_weights(m)
        ins = [data[a] if k == ARG_DATA else w[a] for a, k, _ in m.args]
        res.append(T._apply_and_grads(lib, m, ins))
    table(f"C1 conv_tc={conv_tc}", res)
    for k in ("conv_tc", "conv_thin_tc"):
        gpu.check(gpu.so.mdnn_set_option(k.encode(), 1))


def bn(offset, dims, scale=2.0, off_mag=None, seed=3):
    rng = np.random.default_rng(seed)
    C = dims[2]
    if off_mag is not None:
        offs = (rng.uniform(*off_mag, C) * np.exp(1j * rng.uniform(0, 6.3, C))).astype(np.complex64)
        x = np.asfortranarray(crand(rng, dims, scale) + offs.reshape((1, 1, C) + (1,) * 13))
    else:
        x = crand(rng, dims, scale) + np.complex64(offset)
    vals = {"x": x, "b_bn_mean": crand(rng, d16(1, 1, C), 0.1), "b_bn_var": crand(rng, d16(1, 1, C), 0.1) + 1,
            "b_g": crand(rng, d16(1, 1, C)), "b_beta": crand(rng, d16(1, 1, C), 0.3)}
    res = []
    for lib in (gpu, ref, ref64):
        m = Model.bn_block(lib, "b", dims)
        n = m.nlop
        outs = dict(zip(m.out_names, n.apply([vals[a] for a in m.arg_names])))
        dy = crand(np.random.default_rng(9), n.out_dims(m.output_index("out")))
        g = n.adjoint_all(m.output_index("out"), dy)
        res.append((outs, {k: v for k, v in zip(m.arg_names, g) if k in ("x", "b_g", "b_beta")}))
    table(f"BN block dims {dims[:3]} B={dims[15]} offset {offset} offmag {off_mag}", res)


def denoiser(fuse):
    x0 = T._denoiser_inputs(ref, 5, 320, 368)
    kw = dict(iterations=1, layers=5, filters=64, im_x=320, im_y=368, coils=15, batch=1)
    for k in ("conv_bn_fuse", "conv_thin_tc_bnb"):
        gpu.check(gpu.so.mdnn_set_option(k.encode(), fuse))
    res = []
    for lib in (gpu, ref, ref64):
        m = Model.modl_denoiser(lib, **kw)
        w = T._perturbed_weights(m)
        ins = [x0 if k == ARG_DATA else w[a] for a, k, _ in m.args]
        res.append(T._apply_and_grads(lib, m, ins, want_x=True))
    for k in ("conv_bn_fuse", "conv_thin_tc_bnb"):
        gpu.check(gpu.so.mdnn_set_option(k.encode(), 1))
    table(f"denoiser L5 fuse={fuse}", res)


what = sys.argv[1:] or ["c1", "bn", "den"]
if "c1" in what:
    c1(1)
    c1(0)
if "bn" in what:
    d = list(d16(320, 368, 64))
    bn(0.3 - 0.2j, d)
    d = list(d16(96, 80, 64))
    d[15] = 2
    bn(0, d, 0.05, (50, 200), 4)
    bn(0, d, 1.0, None, 4)
if "den" in what:
    denoiser(1)
    denoiser(0)


def traj():
    from paper_2202_14005_b200.mdnn import Trainer
    data = T._c1_data(ref)
    out = {}
    for name, lib, tc in (("gpu_tf32", gpu, 1), ("gpu_fp32", gpu, 0), ("ref32", ref, 1), ("ref64", ref64, 1)):
        if lib is gpu:
            for k in ("conv_tc", "conv_thin_tc"):
                gpu.check(gpu.so.mdnn_set_option(k.encode(), tc))
        t = Trainer(lib, Model.modl(lib, **T.C1), seed=42)
        for k, v in data.items():
            t.set_data(k, v)
        losses = [t.step() for _ in range(3)]
        out[name] = (losses, {n: t.get_weight(n) for n in t.weight_names()})
    for k in ("conv_tc", "conv_thin_tc"):
        gpu.check(gpu.so.mdnn_set_option(k.encode(), 1))
    l64, w64 = out["ref64"]
    for name, (ls, ws) in out.items():
        print(f"  {name:9s} losses {ls}  rel-dev {[abs(a - b) / abs(b) for a, b in zip(ls, l64)]}")
        print("     weights rel-L2 vs fp64:", {k: f"{rel_l2(ws[k], w64[k]):.2e}" for k in w64})


if "traj" in what:
    traj()
