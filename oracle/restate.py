"""TEST ORACLE — numpy float64 restatement of the reference algorithms on the
hot path.  Only tests/ may import this module; the product never does.

Each function cites the reference (/root/reference/proj/include/mdnn/...)
file:line it restates.  Arrays use the reference layout: numpy complex arrays
in Fortran order whose shape is the 16 reference dims (x=0, y=1, chan=2,
coil=3, map=4, batch=15; recon.hpp:10-16).  The forward MoDL / VarNet
restatements follow the paper's update equations (Eq. 9, Eq. 10), which is an
independent check of the re-assembled builders in oracle/ref_shim.cpp.
Pinned against the compiled reference by tests/test_cpu_oracle.py and the
golden vectors in tests/golden/.
"""
import numpy as np

DIM_X, DIM_Y, DIM_CHAN, DIM_COIL, DIM_MAPS, DIM_BATCH = 0, 1, 2, 3, 4, 15


def dft(a, flags, inverse=False):
    """Unitary, uncentred DFT along flagged dims (fft.hpp:180-226: 1/sqrt(n)
    per axis, DC at index 0, no fftshift)."""
    out = np.asarray(a, dtype=np.complex128)
    for d in range(out.ndim):
        if (flags >> d) & 1 and out.shape[d] > 1:
            out = (np.fft.ifft if inverse else np.fft.fft)(out, axis=d, norm="ortho")
    return out


def sense_forward(x, coils, pattern):
    """A x = P F (sum_maps C x)  (recon.hpp:100-110)."""
    ci = np.sum(coils * x, axis=DIM_MAPS, keepdims=True)  # [X,Y,1,C,1,...,B]
    return dft(ci, 3) * pattern


def sense_adjoint(y, coils, pattern):
    """A^H y = sum_coils conj(C) F^H (P y)  (recon.hpp:111-121)."""
    ci = dft(y * pattern, 3, inverse=True)
    return np.sum(np.conj(coils) * ci, axis=DIM_COIL, keepdims=True)


def sense_normal(x, coils, pattern, lam=0.0):
    """A^H A x + lam x, pattern applied once (recon.hpp:410-418, 807-820)."""
    ci = np.sum(coils * x, axis=DIM_MAPS, keepdims=True)
    v = dft(dft(ci, 3) * pattern, 3, inverse=True)
    return np.sum(np.conj(coils) * v, axis=DIM_COIL, keepdims=True) + lam * x


def cg_solve(op, b, max_iter, tol, fp32_scalars=True):
    """cg_solve (recon.hpp:143-181): x=0, r=b, p=r; stop when sqrt(rs) <= tol ||b||;
    batch-global scalars; with fp32_scalars the reference's float rounding of
    rs, pap, alpha, beta (md_zdot returns complex<R>) is reproduced."""
    f = (lambda v: float(np.float32(v))) if fp32_scalars else float
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    bnorm = float(np.sqrt(np.sum(np.abs(b) ** 2)))
    rs = f(np.sum(np.abs(r) ** 2))
    if bnorm == 0:
        return x, 0
    it = 0
    while it < max_iter:
        if np.sqrt(rs) <= tol * bnorm:
            break
        ap = op(p)
        pap = f(np.real(np.sum(p * np.conj(ap))))
        if not np.isfinite(pap) or pap <= 0:
            raise FloatingPointError("cg breakdown")
        alpha = f(rs / pap)
        x = x + alpha * p
        r = r - alpha * ap
        rs_new = f(np.sum(np.abs(r) ** 2))
        beta = f(rs_new / rs)
        p = r + beta * p
        rs = rs_new
        it += 1
    return x, it


def conv_same(x, w):
    """Complex 'same' cross-correlation over x, y (conv_tenmul + linop_pad,
    nn.hpp:305-384): y[p,f] = sum_{t,c} x[p + t - (k-1)//2, c] w[t,c,f], zero padding.
    x: [X,Y,C,...] (extra dims batched); w: [KX,KY,C,F]."""
    KX, KY, C, F = w.shape[:4]
    px, py = (KX - 1) // 2, (KY - 1) // 2
    X, Y = x.shape[0], x.shape[1]
    xp = np.zeros((X + KX - 1, Y + KY - 1) + x.shape[2:], dtype=np.complex128)
    xp[px:px + X, py:py + Y] = x
    out_shape = list(x.shape)
    out_shape[DIM_CHAN] = F
    y = np.zeros(out_shape, dtype=np.complex128)
    for kx in range(KX):
        for ky in range(KY):
            win = xp[kx:kx + X, ky:ky + Y]  # [X, Y, C, ...]
            # contract channel dim 2 with w[kx, ky, :, :]
            y += np.moveaxis(np.tensordot(win, w[kx, ky, :, :, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]
                                          if w.ndim == 16 else w[kx, ky], axes=([DIM_CHAN], [0])), -1, DIM_CHAN)
    return y


def conv_transposed_same(y, w):
    """Exact adjoint of conv_same with the same filters (conv_layer transposed,
    nn.hpp:385-413)."""
    KX, KY = w.shape[0], w.shape[1]
    wt = np.conj(w[::-1, ::-1]).swapaxes(2, 3)
    if KX % 2 == 0 or KY % 2 == 0:
        raise NotImplementedError("even kernels")
    return conv_same(y, wt)


def batchnorm_train(x, axes, eps=1e-5):
    """BatchNormNode train forward (ops.hpp:1104-1136): biased variance E|x-mu|^2."""
    mu = np.mean(x, axis=axes, keepdims=True)
    u = x - mu
    var = np.mean(np.abs(u) ** 2, axis=axes, keepdims=True)
    return u / np.sqrt(var + eps), mu, var


def crelu(x):
    """CReluNode (ops.hpp:451-475)."""
    return np.maximum(x.real, 0) + 1j * np.maximum(x.imag, 0)


def rbf(z, w, centers, sigma, filter_dim=DIM_CHAN):
    """RbfNode (ops.hpp:1308-1390) on Re z; w [nf, nw]."""
    zr = np.real(z)
    shape = [1] * z.ndim
    shape[filter_dim] = z.shape[filter_dim]
    out = np.zeros(z.shape, dtype=np.complex128)
    for j, mu in enumerate(centers):
        out += np.real(w[:, j]).reshape(shape) * np.exp(-((zr - mu) / sigma) ** 2 / 2)
    return out


def mse(p, r):
    """MseNode (ops.hpp:878-889): (1/n) sum |p - r|^2."""
    return float(np.mean(np.abs(p - r) ** 2))


def adam(theta, g, m, v, t, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
    """adam_step (optim.hpp:81-108): complex m, real v = |g|^2 moments."""
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * np.abs(g) ** 2
    c1, c2 = 1 / (1 - b1 ** t), 1 / (1 - b2 ** t)
    return theta - lr * (m * c1) / (np.sqrt(v * c2) + eps), m, v


def modl_forward(kspace, coils, pattern, weights, T, L, cg_iter, cg_tol=1e-7, eps=1e-5):
    """Unrolled MoDL in train mode (paper Eq. 10; recon.hpp:686-904):
    x0 = A^H y;  x^{t+1} = (A^H A + lam)^-1 (x0 + lam D_W(x^t)),
    D_W(x) = x + CNN(x), CNN = L conv layers with BN (over x, y, batch) + gamma,
    beta + CReLU between them and a bias on the last; lam = exp(Re lam_log)."""
    lam = float(np.exp(np.real(weights["lam_log"]).ravel()[0]))
    x0 = sense_adjoint(kspace, coils, pattern)
    x = x0
    bn_axes = (DIM_X, DIM_Y, DIM_BATCH)
    for _ in range(T):
        h = x
        for l in range(L):
            h = conv_same(h, weights[f"dw{l}_w"])
            if l == L - 1:
                h = h + weights[f"dw{l}_b"]
                break
            h, _, _ = batchnorm_train(h, bn_axes, eps)
            h = crelu(weights[f"dw{l}_g"] * h + weights[f"dw{l}_beta"])
        rhs = x0 + lam * (x + h)
        x, _ = cg_solve(lambda v: sense_normal(v, coils, pattern, lam), rhs, cg_iter, cg_tol, fp32_scalars=False)
    return x


def varnet_forward(kspace, coils, pattern, weights, T, n_rbf):
    """Variational network (paper Eq. 9; recon.hpp:499-680):
    x^{t+1} = x^t - K^T Phi'(Re K x^t) - lam_t (A^H A x^t - A^H y), with x as
    two real channels, real filters K and RBF activation on [-1, 1]."""
    centers = [-1 + 2 * j / (n_rbf - 1) for j in range(n_rbf)]
    sigma = 2 / (n_rbf - 1)
    x0 = sense_adjoint(kspace, coils, pattern)
    x = x0
    for t in range(T):
        w = np.real(weights[f"it{t}_k_w"]).astype(np.complex128)
        xc = np.concatenate([np.real(x), np.imag(x)], axis=DIM_CHAN).astype(np.complex128)
        z = np.real(conv_same(xc, w)).astype(np.complex128)
        phi = rbf(z, weights[f"it{t}_rbf_w"].reshape(w.shape[3], n_rbf, order="F"), centers, sigma)
        reg2 = conv_transposed_same(phi, w)
        reg = np.real(reg2[:, :, 0:1]) + 1j * np.real(reg2[:, :, 1:2])
        lam = float(np.real(weights[f"it{t}_lam"]).ravel()[0])
        dc = sense_normal(x, coils, pattern) - x0
        x = x - (reg + lam * dc)
    return x
