"""Shared helpers for the parity tests."""
import numpy as np

from paper_2202_14005_b200.capi import dims16  # noqa: F401


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    nb = np.linalg.norm(b.ravel())
    d = np.linalg.norm((a - b).ravel())
    return d / nb if nb > 0 else d


def crand(rng, dims, amp=1.0):
    dims = tuple(int(d) for d in dims)
    a = rng.uniform(-amp, amp, size=dims) + 1j * rng.uniform(-amp, amp, size=dims)
    return np.asfortranarray(a.astype(np.complex64))


def rrand(rng, dims, amp=1.0):
    dims = tuple(int(d) for d in dims)
    return np.asfortranarray(rng.uniform(-amp, amp, size=dims).astype(np.complex64))


def d16(*head):
    d = [1] * 16
    for k, v in enumerate(head):
        d[k] = int(v)
    return tuple(d)


def image_dims(x, y, batch=1, maps=1):
    d = [1] * 16
    d[0], d[1], d[4], d[15] = x, y, maps, batch
    return tuple(d)


def coil_dims(x, y, coils, batch=1, maps=1):
    d = [1] * 16
    d[0], d[1], d[3], d[4], d[15] = x, y, coils, maps, batch
    return tuple(d)


def kspace_dims(x, y, coils, batch=1):
    d = [1] * 16
    d[0], d[1], d[3], d[15] = x, y, coils, batch
    return tuple(d)


def pattern_dims(y):
    d = [1] * 16
    d[1] = y
    return tuple(d)


def sim_data(lib, x, y, coils, batch=1, seed=1, accel=4, acl=28):
    """Reference generators (simulate.hpp:40-133) via the library's C ABI:
    phantom, normalised coil maps, regular+ACL pattern, and A x k-space."""
    import ctypes as C
    ph = np.zeros(image_dims(x, y, batch), dtype=np.complex64, order="F")
    cm = np.zeros(coil_dims(x, y, coils, batch), dtype=np.complex64, order="F")
    for s in range(batch):
        p1 = np.zeros((x, y), dtype=np.complex64, order="F")
        c1 = np.zeros((x, y, coils), dtype=np.complex64, order="F")
        lib.check(lib.so.mdnn_sim_item(seed, s, x, y, coils, p1.ctypes.data, c1.ctypes.data))
        ph[:, :, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, s] = p1
        cm[:, :, 0, :, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, s] = c1
    pat = np.zeros(pattern_dims(y), dtype=np.complex64, order="F")
    lib.check(lib.so.mdnn_sim_pattern(y, accel, acl, pat.ctypes.data))
    return ph, cm, pat
