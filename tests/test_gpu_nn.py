"""GPU parity of the CNN regulariser atoms and layers (per node, oracle-fed
inputs, SURVEY §8c protocol): conv fwd / bwd-data / bwd-weight (plain and
transposed, with bias), batch norm (train and inference), CReLU, RBF, MSE,
exp, complex/real split, broadcast add and generic TenMul.

Tolerances: 1e-3 for convolution paths (TF32 target, BASELINE north_star),
1e-5 for everything else.
"""
import numpy as np
import pytest

from paper_2202_14005_b200.mdnn import Model, Nlop
from util import crand, d16, rel_l2, rrand

pytestmark = pytest.mark.gpu
TOL = 1e-5
CONV_TOL = 1e-3


def _check_node(ng, nr, ins, rng, tol, names=None):
    og, orf = ng.apply(ins), nr.apply(ins)
    assert len(og) == len(orf)
    for o in range(len(og)):
        assert rel_l2(og[o], orf[o]) <= tol, ("out", o)
    for o in range(nr.n_out):
        for i in range(nr.n_in):
            dx = crand(rng, nr.in_dims(i))
            try:
                r = nr.derivative(o, i, dx)
            except Exception:
                continue
            assert rel_l2(ng.derivative(o, i, dx), r) <= tol, ("deriv", o, i)
        dy = crand(rng, nr.out_dims(o))
        ag, ar = ng.adjoint_all(o, dy), nr.adjoint_all(o, dy)
        for i in range(nr.n_in):
            assert rel_l2(ag[i], ar[i]) <= tol, ("adjoint", o, i, names and names[i])


@pytest.mark.parametrize("cin,cout,k,X,Y,B,bias", [
    (1, 8, 3, 20, 17, 2, False), (8, 8, 3, 33, 24, 1, False), (8, 1, 3, 16, 16, 2, True),
    (2, 6, 11, 24, 20, 1, False), (2, 24, 11, 40, 24, 2, False), (4, 4, 5, 16, 12, 3, True), (64, 64, 3, 40, 32, 1, False),
    # tcgen05 TF32 path: full and partial 32x16 super-tiles, 32- and 64-channel variants
    (64, 64, 3, 64, 48, 2, False), (32, 32, 3, 36, 20, 1, False), (32, 64, 3, 33, 17, 1, False),
    (64, 32, 3, 32, 16, 2, True),
])
@pytest.mark.parametrize("transposed", [False, True])
def test_conv_layer(gpu, ref, cin, cout, k, X, Y, B, bias, transposed):
    rng = np.random.default_rng(cin * 31 + cout + k)
    in_dims = list(d16(X, Y, cin))
    in_dims[15] = B
    mg = Model.conv_layer(gpu, "c", in_dims, (k, k), cout, transposed=transposed, bias=bias)
    mr = Model.conv_layer(ref, "c", in_dims, (k, k), cout, transposed=transposed, bias=bias)
    assert mg.arg_names == mr.arg_names
    ng, nr = mg.nlop, mr.nlop
    ins = [crand(rng, nr.in_dims(i)) for i in range(nr.n_in)]
    _check_node(ng, nr, ins, rng, CONV_TOL, mr.arg_names)


@pytest.mark.parametrize("cin,cout,k,X,Y,B,bias", [
    # one side single-channel, wide side channels-last: the thin-conv kernels
    (1, 64, 3, 40, 36, 2, False), (64, 1, 3, 33, 20, 2, True), (1, 8, 5, 20, 17, 1, True),
    (16, 1, 3, 17, 35, 3, False), (1, 32, 3, 64, 48, 1, False),
    # multi-channel non-TC shape stored channels-last (CUDA-core CHLAST path)
    (8, 8, 3, 20, 12, 2, False),
])
@pytest.mark.parametrize("transposed", [False, True])
def test_conv_layer_chlast(gpu, ref, cin, cout, k, X, Y, B, bias, transposed):
    rng = np.random.default_rng(cin * 37 + cout + k)
    in_dims = list(d16(X, Y, cin))
    in_dims[15] = B
    gpu.check(gpu.so.mdnn_set_option(b"conv_chlast", 1))
    try:
        mg = Model.conv_layer(gpu, "c", in_dims, (k, k), cout, transposed=transposed, bias=bias)
    finally:
        gpu.check(gpu.so.mdnn_set_option(b"conv_chlast", 0))
    mr = Model.conv_layer(ref, "c", in_dims, (k, k), cout, transposed=transposed, bias=bias)
    ng, nr = mg.nlop, mr.nlop
    ins = [crand(rng, nr.in_dims(i)) for i in range(nr.n_in)]
    _check_node(ng, nr, ins, rng, CONV_TOL, mr.arg_names)


def test_conv_tensor_core_vs_cuda_core(gpu):
    """The tcgen05 TF32 path agrees with the fp32 CUDA-core path within the
    TF32 budget (per pass: RN operands ~3e-4)."""
    import ctypes as C
    rng = np.random.default_rng(21)
    in_dims = list(d16(96, 64, 64))
    in_dims[15] = 2
    m = Model.conv_layer(gpu, "c", in_dims, (3, 3), 64)
    n = m.nlop
    x, w = crand(rng, n.in_dims(0)), crand(rng, n.in_dims(1), 0.05)
    dy = crand(rng, n.out_dims(0))
    res = []
    for tc in (1, 0):
        gpu.check(gpu.so.mdnn_set_option(b"conv_tc", tc))
        y = n.apply([x, w])[0]
        dx = n.adjoint_all(0, dy)
        res.append((y, dx[0], dx[1]))
    gpu.check(gpu.so.mdnn_set_option(b"conv_tc", 1))
    for a, b in zip(res[0], res[1]):
        assert rel_l2(a, b) <= 1e-3


@pytest.mark.parametrize("cin,cout,X,Y,B", [(64, 64, 40, 70, 2), (32, 64, 17, 33, 1), (64, 32, 24, 16, 3),
                                           (32, 32, 40, 50, 2)])
def test_conv_tc_kernel_variants(gpu, ref, cin, cout, X, Y, B):
    """Both tcgen05 conv kernel forms -- channel-major k_conv_tc_t (2 Cout = 128)
    and the CTA-pair pixel-major k_conv_tc_pair (2 Cout = 64) -- against the
    reference, fwd + bwd-data + bwd-weight, partial super-tiles in x and y."""
    rng = np.random.default_rng(cin + cout + X)
    in_dims = list(d16(X, Y, cin))
    in_dims[15] = B
    mg = Model.conv_layer(gpu, "c", in_dims, (3, 3), cout)
    mr = Model.conv_layer(ref, "c", in_dims, (3, 3), cout)
    ins = [crand(rng, mr.nlop.in_dims(i)) for i in range(mr.nlop.n_in)]
    _check_node(mg.nlop, mr.nlop, ins, rng, CONV_TOL, mr.arg_names)


@pytest.mark.parametrize("transposed", [False, True])
@pytest.mark.parametrize("X,Y,B", [(40, 36, 2), (33, 70, 1)])
def test_thin_reduce_tensor_core(gpu, ref, transposed, X, Y, B):
    """64 -> 1 (and the bwd-data of 1 -> 64) through the tcgen05 projection +
    gather path (conv_thin_tc.cu) and through the CUDA-core kernel, against the
    reference: fwd, bwd-data and bwd-weight at the TF32 budget."""
    rng = np.random.default_rng(X + Y)
    cin, cout = (1, 64) if transposed else (64, 1)
    in_dims = list(d16(X, Y, cin))
    in_dims[15] = B
    mr = Model.conv_layer(ref, "c", in_dims, (3, 3), cout, transposed=transposed, bias=not transposed)
    ins = [crand(rng, mr.nlop.in_dims(i)) for i in range(mr.nlop.n_in)]
    outs = []
    for tc in (1, 0):
        gpu.check(gpu.so.mdnn_set_option(b"conv_chlast", 1))
        gpu.check(gpu.so.mdnn_set_option(b"conv_thin_tc", tc))
        try:
            mg = Model.conv_layer(gpu, "c", in_dims, (3, 3), cout, transposed=transposed, bias=not transposed)
            _check_node(mg.nlop, mr.nlop, ins, np.random.default_rng(1), CONV_TOL, mr.arg_names)
            outs.append(mg.nlop.apply(ins)[0])
        finally:
            gpu.check(gpu.so.mdnn_set_option(b"conv_chlast", 0))
            gpu.check(gpu.so.mdnn_set_option(b"conv_thin_tc", 1))
    assert rel_l2(outs[0], outs[1]) <= CONV_TOL


@pytest.mark.parametrize("transposed", [False, True])
def test_thin_expand_tensor_core(gpu, ref, transposed):
    """1 -> 64 (and the bwd-data of 64 -> 1) through the split-precision tcgen05
    im2col kernel (option conv_thin_tc_expand) against the reference."""
    X, Y, B = 40, 36, 2
    rng = np.random.default_rng(7)
    cin, cout = (64, 1) if transposed else (1, 64)
    in_dims = list(d16(X, Y, cin))
    in_dims[15] = B
    mr = Model.conv_layer(ref, "c", in_dims, (3, 3), cout, transposed=transposed)
    ins = [crand(rng, mr.nlop.in_dims(i)) for i in range(mr.nlop.n_in)]
    gpu.check(gpu.so.mdnn_set_option(b"conv_chlast", 1))
    gpu.check(gpu.so.mdnn_set_option(b"conv_thin_tc_expand", 1))
    try:
        mg = Model.conv_layer(gpu, "c", in_dims, (3, 3), cout, transposed=transposed)
        _check_node(mg.nlop, mr.nlop, ins, np.random.default_rng(1), CONV_TOL, mr.arg_names)
    finally:
        gpu.check(gpu.so.mdnn_set_option(b"conv_chlast", 0))
        gpu.check(gpu.so.mdnn_set_option(b"conv_thin_tc_expand", 0))


def test_conv_weights_init_bitwise(gpu, ref):
    in_dims = list(d16(8, 8, 4))
    mg = Model.conv_layer(gpu, "dw1", in_dims, (3, 3), 16)
    mr = Model.conv_layer(ref, "dw1", in_dims, (3, 3), 16)
    assert np.array_equal(mg.init_weight(42, "dw1_w"), mr.init_weight(42, "dw1_w"))


@pytest.mark.parametrize("train", [True, False])
def test_batchnorm(gpu, ref, train):
    rng = np.random.default_rng(5)
    dims = list(d16(24, 20, 8))
    dims[15] = 2
    flags = (1 << 0) | (1 << 1) | (1 << 15)
    ng, nr = Nlop.batchnorm(gpu, dims, flags, train), Nlop.batchnorm(ref, dims, flags, train)
    x = crand(rng, dims)
    mean = crand(rng, nr.in_dims(1), 0.1)
    var = rrand(rng, nr.in_dims(2), 1.0) + np.float32(1.5)
    _check_node(ng, nr, [x, mean, np.asfortranarray(var)], rng, TOL)


@pytest.mark.parametrize("kind", ["crelu", "zconj", "zreal", "exp_real"])
def test_elementwise(gpu, ref, kind):
    rng = np.random.default_rng(11)
    dims = d16(17, 9, 3) if kind != "exp_real" else d16()
    _check_node(Nlop.unary(gpu, kind, dims), Nlop.unary(ref, kind, dims), [crand(rng, dims)], rng, TOL)


def test_mse(gpu, ref):
    rng = np.random.default_rng(12)
    dims = d16(20, 12)
    ins = [crand(rng, dims), crand(rng, dims)]
    _check_node(Nlop.unary(gpu, "mse", dims), Nlop.unary(ref, "mse", dims), ins, rng, TOL)


@pytest.mark.parametrize("join", [False, True])
def test_real_chan(gpu, ref, join):
    rng = np.random.default_rng(13)
    dims = list(d16(12, 10, 2 if join else 1))
    dims[15] = 2
    ng, nr = Nlop.real_chan(gpu, dims, 2, join), Nlop.real_chan(ref, dims, 2, join)
    _check_node(ng, nr, [crand(rng, dims)], rng, TOL)


@pytest.mark.parametrize("window", [1, 0], ids=["window", "all-centres"])
@pytest.mark.parametrize("nw,width,zscale", [(31, 1.0, 1.2), (64, 0.5, 3.0), (9, 1.0, 1.0)])
def test_rbf(gpu, ref, window, nw, width, zscale):
    """RbfNode (ops.hpp:1308-1427) against the reference: VarNet's 31 centres at
    sigma = spacing, narrow Gaussians over 64 centres with z far outside the
    centre range, and few centres (no window).  With evenly spaced centres the
    product evaluates only the centres within 8.5 sigma of z (option
    rbf_window); both paths are checked."""
    rng = np.random.default_rng(14 + nw)
    nf = 6
    z = list(d16(16, 12, nf))
    z[15] = 2
    centers = [-1 + 2 * j / (nw - 1) for j in range(nw)]
    sigma = width * 2 / (nw - 1)
    gpu.check(gpu.so.mdnn_set_option(b"rbf_window", window))
    try:
        ng, nr = Nlop.rbf(gpu, z, 2, centers, sigma), Nlop.rbf(ref, z, 2, centers, sigma)
        ins = [rrand(rng, z, zscale), rrand(rng, nr.in_dims(1), 0.05)]
        _check_node(ng, nr, ins, rng, TOL)
    finally:
        gpu.check(gpu.so.mdnn_set_option(b"rbf_window", 1))


@pytest.mark.parametrize("cut", [55, 85], ids=["K6", "K9"])
@pytest.mark.parametrize("pair", [1, 0], ids=["paired", "visit"])
def test_rbf_window_map_forms(gpu, ref, pair, cut):
    """VarNet's window (31 centres, sigma = spacing, z also outside the centre
    range) at both cut-offs (option rbf_cut: 5.5 sigma -> K = 6, the default;
    8.5 sigma -> K = 9): the paired-fp32 map (option rbf_pair, forward and
    z-adjoint), the rbf_visit_k form and the windowed weight-gradient pass all
    match the reference (which evaluates every centre)."""
    rng = np.random.default_rng(77)
    z = list(d16(40, 24, 24))
    z[15] = 2
    centers = [-1 + 2 * j / 30 for j in range(31)]
    gpu.check(gpu.so.mdnn_set_option(b"rbf_pair", pair))
    gpu.check(gpu.so.mdnn_set_option(b"rbf_cut", cut))
    try:
        ng, nr = Nlop.rbf(gpu, z, 2, centers, 2 / 30), Nlop.rbf(ref, z, 2, centers, 2 / 30)
        ins = [rrand(rng, z, 1.5), rrand(rng, nr.in_dims(1), 0.05)]
        _check_node(ng, nr, ins, rng, TOL)
    finally:
        gpu.check(gpu.so.mdnn_set_option(b"rbf_pair", 1))
        gpu.check(gpu.so.mdnn_set_option(b"rbf_cut", 55))


def test_bcast_add_and_tenmul(gpu, ref):
    rng = np.random.default_rng(15)
    x = d16(10, 8, 4)
    b = d16(1, 1, 4)
    _check_node(Nlop.bcast_add(gpu, x, b), Nlop.bcast_add(ref, x, b), [crand(rng, x), crand(rng, b)], rng, TOL)
    # per-channel scale (bn_scale TenMul, recon.hpp:756-763)
    s = (1, 10, 80) + (0,) * 13
    sg = (0, 0, 1) + (0,) * 13
    args = (x, x, s, x, s, b, sg)
    _check_node(Nlop.tenmul(gpu, *args), Nlop.tenmul(ref, *args), [crand(rng, x), crand(rng, b)], rng, TOL)
    # a genuine contraction: matrix-vector (dense_layer wiring, nn.hpp:232-239)
    it = (5, 7, 3) + (1,) * 13
    yd, wd, xd = (5, 3) + (1,) * 14, (5, 7) + (1,) * 14, (7, 3) + (1,) * 14
    so, sw, sx = (1, 0, 5) + (0,) * 13, (1, 5, 0) + (0,) * 13, (0, 1, 7) + (0,) * 13
    args = (it, yd, so, wd, sw, xd, sx)
    _check_node(Nlop.tenmul(gpu, *args), Nlop.tenmul(ref, *args), [crand(rng, wd), crand(rng, xd)], rng, TOL)


def test_tenmul_overlapping_window_adjoint_deterministic(gpu, ref):
    """A 2-D valid correlation written as one TenMul (conv_layer's wiring,
    nn.hpp:305-337 / ops.hpp:79-111): the adjoint wrt the windowed input has
    overlapping output strides.  Values match the reference and two runs are
    bitwise identical (serial launches over the overlapping dims, no float
    atomics)."""
    rng = np.random.default_rng(18)
    OX, OY, KX, KY, CI, CO = 9, 7, 3, 3, 2, 3
    IX, IY = OX + KX - 1, OY + KY - 1
    # iteration (ox, oy, kx, ky, ci, co); x[ox + kx, oy + ky, ci]; w[kx, ky, ci, co]; y[ox, oy, co]
    it = (OX, OY, KX, KY, CI, CO) + (1,) * 10
    xd, wd, yd = (IX, IY, CI) + (1,) * 13, (KX, KY, CI, CO) + (1,) * 12, (OX, OY, CO) + (1,) * 13
    sx = (1, IX, 1, IX, IX * IY, 0) + (0,) * 10
    sw = (0, 0, 1, KX, KX * KY, KX * KY * CI) + (0,) * 10
    sy = (1, OX, 0, 0, 0, OX * OY) + (0,) * 10
    args = (it, yd, sy, xd, sx, wd, sw)
    ins = [crand(rng, xd), crand(rng, wd)]
    _check_node(Nlop.tenmul(gpu, *args), Nlop.tenmul(ref, *args), ins, rng, TOL)
    dy = crand(rng, yd)
    runs = []
    for _ in range(2):
        n = Nlop.tenmul(gpu, *args)
        n.apply(ins)
        runs.append(n.adjoint_all(0, dy)[0])
    assert runs[0].tobytes(order="A") == runs[1].tobytes(order="A")


def test_pad_and_dft_nodes(gpu, ref):
    rng = np.random.default_rng(16)
    i, o, c = d16(6, 5, 2), d16(9, 8, 2), (1, 2) + (0,) * 14
    _check_node(Nlop.pad(gpu, i, o, c), Nlop.pad(ref, i, o, c), [crand(rng, i)], rng, TOL)
    d = d16(12, 10, 3)
    _check_node(Nlop.dft(gpu, d, 3), Nlop.dft(ref, d, 3), [crand(rng, d)], rng, TOL)


def test_graph_algebra(gpu, ref):
    """combine / link / duplicate / chain (nlop.hpp:265-350) on a small graph."""
    rng = np.random.default_rng(17)
    d = d16(8, 6)
    res = []
    for lib in (gpu, ref):
        mul = Nlop.tenmul(lib, d, d, (1, 8) + (0,) * 14, d, (1, 8) + (0,) * 14, d, (1, 8) + (0,) * 14)
        cr = Nlop.unary(lib, "crelu", d)
        cj = Nlop.unary(lib, "zconj", d)
        g = mul.combine(cr).link(0, 2)          # crelu(x1*x2)
        g = cj.combine(g).link(0, 1)            # crelu(conj(a) * b) : inputs (a, b)
        g = g.duplicate(0, 1)                   # crelu(conj(a) * a)
        res.append(g)
    x = crand(rng, d)
    _check_node(res[0], res[1], [x], rng, TOL)


@pytest.mark.parametrize("cin,cout,k", [(2, 24, 11), (2, 6, 11), (3, 5, 5)])
@pytest.mark.parametrize("transposed", [False, True])
@pytest.mark.parametrize("vn_tc", [1, 0], ids=["vn_tc", "cuda_core"])
def test_conv_layer_real_operands(gpu, ref, cin, cout, k, transposed, vn_tc):
    """VarNet-style real-valued activations, weights and cotangents.  The
    11 x 11, 2 <-> F layers run on the tensor cores (conv_vn_tc.cu, TF32 budget
    1e-3) unless option conv_vn_tc = 0 selects the fp32 real-operand CUDA-core
    kernels (conv.cu, 1e-5); the weight gradient is the CUDA-core kernel either
    way.  Values, tangents and adjoints match the reference's complex
    arithmetic, the imaginary parts stay exactly zero, and a complex cotangent
    switches to the complex path (1e-5)."""
    rng = np.random.default_rng(cin * 7 + cout + k)
    X, Y, B = 36, 20, 2
    in_dims = list(d16(X, Y, cin))
    in_dims[15] = B
    tc = vn_tc and k == 11 and cin == 2
    tol = CONV_TOL if tc else 1e-5
    gpu.check(gpu.so.mdnn_set_option(b"conv_vn_tc", vn_tc))
    try:
        mg = Model.conv_layer(gpu, "c", in_dims, (k, k), cout, transposed=transposed, bias=False)
        mr = Model.conv_layer(ref, "c", in_dims, (k, k), cout, transposed=transposed, bias=False)
        ng, nr = mg.nlop, mr.nlop
        ins = [rrand(rng, nr.in_dims(i)) for i in range(nr.n_in)]
        og, orf = ng.apply(ins)[0], nr.apply(ins)[0]
        assert rel_l2(og, orf) <= tol and not np.any(og.imag)
        dy = rrand(rng, nr.out_dims(0))
        ag, ar = ng.adjoint_all(0, dy), nr.adjoint_all(0, dy)
        for i in range(nr.n_in):
            assert rel_l2(ag[i], ar[i]) <= tol, i
            assert not np.any(ag[i].imag), i
        # a complex cotangent switches back to the complex path
        dyc = crand(rng, nr.out_dims(0))
        for u, v in zip(ng.adjoint_all(0, dyc), nr.adjoint_all(0, dyc)):
            assert rel_l2(u, v) <= 1e-5
    finally:
        gpu.check(gpu.so.mdnn_set_option(b"conv_vn_tc", 1))


@pytest.mark.parametrize("X,Y,B,F", [(640, 368, 1, 24), (258, 37, 2, 24), (100, 130, 3, 6)],
                         ids=["C3-geometry", "ragged", "F6"])
def test_vn_tensor_core_vs_fp32_kernels(gpu, ref, X, Y, B, F):
    """The tensor-core 11 x 11 kernels against the fp32 CUDA-core kernels and the
    reference at the C3 geometry (640 x 368: three 256-pixel expand tiles, the
    last one partial, six overlapping 118-pixel reduce tiles, 74 / 37 row
    chunks, 64-pixel weight-gradient columns) and ragged shapes (partial tiles
    and chunks in x and y): forward, bwd-data and bwd-weight."""
    rng = np.random.default_rng(X + Y + F)
    in_dims = list(d16(X, Y, 2))
    in_dims[15] = B
    mr = Model.conv_layer(ref, "c", in_dims, (11, 11), F, transposed=False, bias=False)
    ins = [rrand(rng, mr.nlop.in_dims(i)) for i in range(2)]
    dy = rrand(rng, mr.nlop.out_dims(0))
    res = []
    for tc in (1, 0):
        gpu.check(gpu.so.mdnn_set_option(b"conv_vn_tc", tc))
        try:
            n = Model.conv_layer(gpu, "c", in_dims, (11, 11), F, transposed=False, bias=False).nlop
            y = n.apply(ins)[0]
            res.append((y, *n.adjoint_all(0, dy)))
        finally:
            gpu.check(gpu.so.mdnn_set_option(b"conv_vn_tc", 1))
    nr = mr.nlop
    yr = nr.apply(ins)[0]
    dxr, dwr = nr.adjoint_all(0, dy)
    for got, want in zip(res[0], (yr, dxr, dwr)):  # forward, bwd-data, bwd-weight on the tensor cores
        assert rel_l2(got, want) <= CONV_TOL
    for got, want in zip(res[1], (yr, dxr, dwr)):  # fp32 CUDA-core kernels
        assert rel_l2(got, want) <= 1e-5
