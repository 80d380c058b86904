"""GPU parity of the persistent mask-pruned A^H A kernels -- the warp-specialised
k_normal_ws (csrc/sense_ws.cuh, default) and the round-1 k_normal_rank
(csrc/sense_rank.cuh, option `sense_ws` = 0), each with contiguous unit ranges
and with whole strips round robin (option `rank_rr`, used for 32-B strips) --
against the reference CPU implementation (oracle/_ref).

Covers every row mode of the pruned stage B (identity, rank-1 terms added to
the identity, terms replacing it, full in-register DFT rows, zero rows),
partial column strips, strips split between two CTAs (forced with the
`sense_rank_ctas` option), non-binary complex patterns (through the
modl_normal_plus_lambda fragment, whose pattern is a data input:
recon.hpp:371-379, 807-820), the CG variant, and agreement with the previous
register-resident kernel (`sense_rank` = 0).  Tolerance: rel-L2 <= 1e-5
(BASELINE.json north_star, fp32 SENSE/CG path).  The ws kernel's contiguous
ranges are cost-balanced (option `rank_vh`, per-strip overhead weight; "ws-equal"
runs the equal-unit-count ranges), including CTAs left without units.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2202_14005_b200.mdnn import Model, sense_dims
from util import crand, d16, image_dims, kspace_dims, pattern_dims, rel_l2, sim_data

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(params=[(1, 1, 9), (1, 0, 9), (1, 0, 0), (0, 1, 9)], ids=["ws", "ws-contiguous", "ws-equal", "rank"])
def rank_opts(gpu, request):
    ws, rr, vh = request.param
    gpu.check(gpu.so.mdnn_set_option(b"sense_ws", ws))
    gpu.check(gpu.so.mdnn_set_option(b"rank_rr", rr))
    gpu.check(gpu.so.mdnn_set_option(b"rank_vh", vh))
    yield gpu
    gpu.check(gpu.so.mdnn_set_option(b"rank_vh", 9))
    gpu.check(gpu.so.mdnn_set_option(b"sense_rank", 1))
    gpu.check(gpu.so.mdnn_set_option(b"sense_rank_ctas", 0))
    gpu.check(gpu.so.mdnn_set_option(b"sense_ws", 1))
    gpu.check(gpu.so.mdnn_set_option(b"rank_rr", 1))


def _normal(lib, cm, pat, x, lam=0.05):
    out = np.zeros(x.shape, dtype=np.complex64, order="F")
    lib.check(lib.so.mdnn_sense_normal(C.byref(lib.arr(cm)), C.byref(lib.arr(pat)), C.c_float(lam),
                                       C.byref(lib.arr(x)), C.byref(lib.arr(out))))
    return out


def _cg(lib, cm, pat, b, iters=10):
    x = np.zeros(b.shape, dtype=np.complex64, order="F")
    it, rr = C.c_long(), C.c_double()
    lib.check(lib.so.mdnn_cg_normal_solve(C.byref(lib.arr(cm)), C.byref(lib.arr(pat)), C.c_float(0.05),
                                          C.byref(lib.arr(b)), iters, 0.0, C.byref(lib.arr(x)), C.byref(it),
                                          C.byref(rr)))
    return x, it.value


def _pattern(Y, kind, seed=0, lib=None):
    p = np.zeros(pattern_dims(Y), dtype=np.complex64, order="F")
    v = p.reshape(-1, order="F")
    rng = np.random.default_rng(seed)
    if kind == "std":          # make_pattern(Y, 4, 28): every 4th line + 28 ACL lines
        lib.check(lib.so.mdnn_sim_pattern(Y, 4, 28, p.ctypes.data))
    elif kind == "random":     # dense random: most rows need the full DFT
        v[:] = rng.random(Y) < 0.5
    elif kind == "sparse":     # few lines: zero rows + single terms
        v[rng.choice(Y, 5, replace=False)] = 1
    elif kind == "ones":       # fully sampled: every row is the identity
        v[:] = 1
    elif kind == "accel2":     # every 2nd line + 6 ACL: terms subtracted from identity rows
        for i in range(Y):
            if i % 2 == 0 or min(i, Y - i) <= 3:
                v[i] = 1
    return p


@pytest.mark.parametrize("Y", [128, 256, 320, 368, 512, 640])
@pytest.mark.parametrize("kind", ["std", "random", "sparse", "ones", "accel2"])
def test_rank_normal_patterns(gpu, ref, rank_opts, Y, kind):
    X, NC, B = 36, 3, 2            # 36 columns: a partial last strip for W = 8 and W = 4
    ph, cm, _ = sim_data(ref, X, Y, NC, B)
    pat = _pattern(Y, kind, seed=Y, lib=ref)
    rng = np.random.default_rng(Y)
    x = crand(rng, image_dims(X, Y, B))
    r = _normal(ref, cm, pat, x)
    for ctas in (0, 3):            # 3 CTAs: every strip range straddles CTAs
        gpu.check(gpu.so.mdnn_set_option(b"sense_rank_ctas", ctas))
        g = _normal(gpu, cm, pat, x)
        assert rel_l2(g, r) <= TOL, (kind, ctas)


@pytest.mark.parametrize("Y", [320, 368, 640])
def test_rank_cg_split_strips(gpu, ref, rank_opts, Y):
    X, NC, B = 48, 4, 2
    ph, cm, pat = sim_data(ref, X, Y, NC, B)
    rng = np.random.default_rng(5)
    b = crand(rng, image_dims(X, Y, B))
    xr, itr = _cg(ref, cm, pat, b)
    for ctas in (0, 5):
        gpu.check(gpu.so.mdnn_set_option(b"sense_rank_ctas", ctas))
        xg, itg = _cg(gpu, cm, pat, b)
        assert itg == itr == 10
        assert rel_l2(xg, xr) <= TOL, ctas


def test_rank_nonbinary_pattern_fragment(gpu, ref, rank_opts):
    """Complex-valued pattern through the normal+lambda fragment (pattern is a
    data input there): every row becomes terms or full rows with complex
    coefficients."""
    X, Y, NC, B = 40, 368, 3, 1
    ph, cm, _ = sim_data(ref, X, Y, NC, B)
    rng = np.random.default_rng(11)
    pat = _pattern(Y, "std", lib=ref)
    v = pat.reshape(-1, order="F")
    idx = np.nonzero(v)[0]
    v[idx[::3]] = (0.5 + 0.25j)    # a third of the sampled lines weighted
    sd = sense_dims(X, Y, NC, 1, B)
    x = crand(rng, image_dims(X, Y, B))
    lam = np.full(d16(), 0.05, dtype=np.complex64, order="F")
    outs = []
    for lib in (gpu, ref):
        m = Model.modl_normal_plus_lambda(lib, sd)
        ins = {"coils": cm, "pattern": pat, "lambda": lam}
        args = [ins.get(n, x) for n in m.arg_names]
        outs.append(m.nlop.apply(args)[0])
    assert rel_l2(outs[0], outs[1]) <= TOL


def test_rank_matches_previous_kernel_at_c2(gpu, ref, rank_opts):
    """C2 geometry (320 x 368, 15 coils, batch 2): the rank kernel, the
    previous register-resident kernel and the reference agree."""
    X, Y, NC, B = 320, 368, 15, 2
    ph, cm, pat = sim_data(ref, X, Y, NC, B)
    r = _normal(ref, cm, pat, ph)
    g1 = _normal(gpu, cm, pat, ph)
    gpu.check(gpu.so.mdnn_set_option(b"sense_rank", 0))
    g0 = _normal(gpu, cm, pat, ph)
    assert rel_l2(g1, r) <= TOL
    assert rel_l2(g0, r) <= TOL
    assert rel_l2(g1, g0) <= TOL


def test_rank_deterministic(gpu, ref, rank_opts):
    X, Y, NC, B = 64, 368, 5, 2
    ph, cm, pat = sim_data(ref, X, Y, NC, B)
    gpu.check(gpu.so.mdnn_set_option(b"sense_rank_ctas", 7))
    a = _normal(gpu, cm, pat, ph)
    b = _normal(gpu, cm, pat, ph)
    assert np.array_equal(np.ascontiguousarray(a).view(np.uint32), np.ascontiguousarray(b).view(np.uint32))


@pytest.mark.parametrize("tol", [0.0, 0.1])
def test_cg_deferred_x_bitwise(gpu, ref, rank_opts, tol):
    """CG with every search direction kept and x summed once after the loop
    (`cg_defer_x`, default) is bitwise equal to the per-iteration x update, with
    and without early convergence; both match the reference."""
    X, Y, NC, B = 48, 368, 4, 2
    ph, cm, pat = sim_data(ref, X, Y, NC, B)
    rng = np.random.default_rng(8)
    b = crand(rng, image_dims(X, Y, B))

    def solve(lib):
        x = np.zeros(b.shape, dtype=np.complex64, order="F")
        it, rr = C.c_long(), C.c_double()
        lib.check(lib.so.mdnn_cg_normal_solve(C.byref(lib.arr(cm)), C.byref(lib.arr(pat)), C.c_float(0.05),
                                              C.byref(lib.arr(b)), 10, tol, C.byref(lib.arr(x)), C.byref(it),
                                              C.byref(rr)))
        return x, it.value

    xr, itr = solve(ref)
    res = []
    try:
        for d in (1, 0):
            gpu.check(gpu.so.mdnn_set_option(b"cg_defer_x", d))
            res.append(solve(gpu))
    finally:
        gpu.check(gpu.so.mdnn_set_option(b"cg_defer_x", 1))
    (x1, i1), (x0, i0) = res
    assert i1 == i0 == itr
    if tol > 0:
        assert itr < 10
    assert np.array_equal(np.ascontiguousarray(x1).view(np.uint32), np.ascontiguousarray(x0).view(np.uint32))
    assert rel_l2(x1, xr) <= TOL


@pytest.mark.parametrize("tol", [0.0, 0.1])
def test_cg_fused_update(gpu, ref, tol):
    """The CG r-update fused into the warp-specialised A^H A launch (grid barrier;
    option `cg_fuse` 1 default, 2 with a cooperative launch) against the separate
    update kernel (`cg_fuse` = 0) and the reference, with programmatic dependent
    launch on and off; strips split between CTAs and early convergence included."""
    X, Y, NC, B = 320, 368, 6, 2
    ph, cm, pat = sim_data(ref, X, Y, NC, B)
    rng = np.random.default_rng(11)
    b = crand(rng, image_dims(X, Y, B))

    def solve(lib):
        x = np.zeros(b.shape, dtype=np.complex64, order="F")
        it, rr = C.c_long(), C.c_double()
        lib.check(lib.so.mdnn_cg_normal_solve(C.byref(lib.arr(cm)), C.byref(lib.arr(pat)), C.c_float(0.05),
                                              C.byref(lib.arr(b)), 10, tol, C.byref(lib.arr(x)), C.byref(it),
                                              C.byref(rr)))
        return x, it.value

    xr, itr = solve(ref)
    res = {}
    try:
        for fuse, pdl in ((0, 1), (1, 1), (2, 1), (1, 0)):
            gpu.check(gpu.so.mdnn_set_option(b"cg_fuse", fuse))
            gpu.check(gpu.so.mdnn_set_option(b"cg_pdl", pdl))
            res[(fuse, pdl)] = solve(gpu)
    finally:
        gpu.check(gpu.so.mdnn_set_option(b"cg_fuse", 1))
        gpu.check(gpu.so.mdnn_set_option(b"cg_pdl", 1))
    x0, i0 = res[(0, 1)]
    for k, (x, i) in res.items():
        assert i == itr, k
        assert rel_l2(x, xr) <= TOL, k
        assert rel_l2(x, x0) <= 1e-6, k
    if tol > 0:
        assert itr < 10


@pytest.mark.parametrize("vh", [9, 40])
def test_ws_cost_ranges_with_empty_ctas(gpu, ref, vh):
    """Cost-balanced ranges with many CTAs: some CTAs own no unit (their range
    lies in a strip-overhead gap) and strips are split across several CTAs; the
    normal operator and CG still match the reference."""
    X, Y, NC, B = 36, 368, 3, 2    # 10 strips x 3 coils = 30 units
    ph, cm, pat = sim_data(ref, X, Y, NC, B)
    rng = np.random.default_rng(21)
    x = crand(rng, image_dims(X, Y, B))
    r = _normal(ref, cm, pat, x)
    xr, itr = _cg(ref, cm, pat, x)
    try:
        gpu.check(gpu.so.mdnn_set_option(b"sense_ws", 1))
        gpu.check(gpu.so.mdnn_set_option(b"rank_rr", 0))
        gpu.check(gpu.so.mdnn_set_option(b"rank_vh", vh))
        for ctas in (7, 24, 30):
            gpu.check(gpu.so.mdnn_set_option(b"sense_rank_ctas", ctas))
            assert rel_l2(_normal(gpu, cm, pat, x), r) <= TOL, ctas
            xg, itg = _cg(gpu, cm, pat, x)
            assert itg == itr
            assert rel_l2(xg, xr) <= TOL, ctas
    finally:
        gpu.check(gpu.so.mdnn_set_option(b"sense_rank_ctas", 0))
        gpu.check(gpu.so.mdnn_set_option(b"rank_rr", 1))
        gpu.check(gpu.so.mdnn_set_option(b"rank_vh", 9))
