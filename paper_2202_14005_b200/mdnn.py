"""Thin Python handles over the C ABI (include/mdnn.h).

These mirror the reference's C++ API names (Nlop.apply / derivative /
adjoint_all / combine / link / duplicate / chain, Model.arg_index, ...,
nlop.hpp:89-437, nn.hpp:68-222) so tests read like the reference's own tests.
Every method is a direct C-ABI call; there is no Python compute path.  The
same classes drive the product library and (tests only) the reference shim.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .capi import (ARG_DATA, ARG_MOVING_STATS, ARG_WEIGHTS, MAX_RANK, Lib, MdnnError, mdnn_array,
                   mdnn_conv_spec, mdnn_modl_cfg, mdnn_sense_dims, mdnn_train_cfg, mdnn_varnet_cfg)

__all__ = ["Nlop", "Model", "Trainer", "cfl_zeros", "ARG_DATA", "ARG_WEIGHTS", "ARG_MOVING_STATS",
           "MdnnError", "modl_cfg", "varnet_cfg", "sense_dims"]


def cfl_zeros(dims):
    return np.zeros(tuple(int(d) for d in dims), dtype=np.complex64, order="F")


def _as_cfl(a, dims=None):
    a = np.asarray(a, dtype=np.complex64)
    if dims is not None:
        a = a.reshape(tuple(dims), order="F")
    return np.asfortranarray(a)


def _longs(seq):
    arr = (C.c_long * MAX_RANK)()
    for k, v in enumerate(seq):
        arr[k] = int(v)
    return arr


class Nlop:
    def __init__(self, lib: Lib, h):
        self.lib = lib
        self.h = lib.checkp(h)

    def __del__(self):
        try:
            self.lib.so.mdnn_nlop_free(self.h)
        except Exception:
            pass

    # --- signature
    @property
    def n_in(self):
        return self.lib.so.mdnn_nlop_n_in(self.h)

    @property
    def n_out(self):
        return self.lib.so.mdnn_nlop_n_out(self.h)

    def in_dims(self, i):
        return self.lib.nlop_dims(self.h, i)

    def out_dims(self, o):
        return self.lib.nlop_dims(self.h, o, out=True)

    # --- evaluation
    def apply(self, ins):
        ins = [_as_cfl(a, self.in_dims(i)) for i, a in enumerate(ins)]
        outs = [cfl_zeros(self.out_dims(o)) for o in range(self.n_out)]
        ia = (mdnn_array * len(ins))(*[self.lib.arr(a) for a in ins])
        oa = (mdnn_array * len(outs))(*[self.lib.arr(a) for a in outs])
        self.lib.check(self.lib.so.mdnn_nlop_apply(self.h, len(ins), ia, len(outs), oa))
        return outs

    def derivative(self, o, i, dx):
        dx = _as_cfl(dx, self.in_dims(i))
        dy = cfl_zeros(self.out_dims(o))
        self.lib.check(self.lib.so.mdnn_nlop_derivative(self.h, o, i, C.byref(self.lib.arr(dx)),
                                                        C.byref(self.lib.arr(dy))))
        return dy

    def adjoint(self, o, i, dy):
        dy = _as_cfl(dy, self.out_dims(o))
        dx = cfl_zeros(self.in_dims(i))
        self.lib.check(self.lib.so.mdnn_nlop_adjoint(self.h, o, i, C.byref(self.lib.arr(dy)),
                                                     C.byref(self.lib.arr(dx))))
        return dx

    def adjoint_all(self, o, dy, wanted=None):
        dy = _as_cfl(dy, self.out_dims(o))
        n = self.n_in
        dx = [cfl_zeros(self.in_dims(i)) for i in range(n)]
        da = (mdnn_array * n)(*[self.lib.arr(a) for a in dx])
        w = None
        if wanted is not None:
            w = (C.c_uint8 * n)(*[1 if x else 0 for x in wanted])
        self.lib.check(self.lib.so.mdnn_nlop_adjoint_all(self.h, o, C.byref(self.lib.arr(dy)), n, da, w))
        return [dx[i] if (wanted is None or wanted[i]) else None for i in range(n)]

    def cg_status(self):
        it, rel, conv = C.c_long(), C.c_double(), C.c_int()
        self.lib.check(self.lib.so.mdnn_nlop_cg_status(self.h, C.byref(it), C.byref(rel), C.byref(conv)))
        return it.value, rel.value, bool(conv.value)

    # --- algebra
    def combine(self, g):
        return Nlop(self.lib, self.lib.so.mdnn_nlop_combine(self.h, g.h))

    def link(self, o, i):
        return Nlop(self.lib, self.lib.so.mdnn_nlop_link(self.h, o, i))

    def duplicate(self, i, j):
        return Nlop(self.lib, self.lib.so.mdnn_nlop_duplicate(self.h, i, j))

    def chain(self, g):
        return Nlop(self.lib, self.lib.so.mdnn_nlop_chain(self.h, g.h))

    # --- atom factories
    @staticmethod
    def dft(lib, dims, flags, inverse=False):
        return Nlop(lib, lib.so.mdnn_nlop_dft(len(dims), _longs(dims), flags, int(inverse)))

    @staticmethod
    def tenmul(lib, iter_, od, so, i1, s1, i2, s2):
        r = len(iter_)
        return Nlop(lib, lib.so.mdnn_nlop_tenmul(r, *[_longs(x) for x in (iter_, od, so, i1, s1, i2, s2)]))

    @staticmethod
    def add(lib, dims, subtract=False):
        return Nlop(lib, lib.so.mdnn_nlop_add(len(dims), _longs(dims), int(subtract)))

    @staticmethod
    def bcast_add(lib, x, b):
        return Nlop(lib, lib.so.mdnn_nlop_bcast_add(len(x), _longs(x), _longs(b)))

    @staticmethod
    def fork(lib, dims, n):
        return Nlop(lib, lib.so.mdnn_nlop_fork(len(dims), _longs(dims), n))

    @staticmethod
    def unary(lib, kind, dims):
        fn = {"zconj": lib.so.mdnn_nlop_zconj, "zreal": lib.so.mdnn_nlop_zreal, "crelu": lib.so.mdnn_nlop_crelu,
              "exp_real": lib.so.mdnn_nlop_exp_real, "mse": lib.so.mdnn_nlop_mse}[kind]
        return Nlop(lib, fn(len(dims), _longs(dims)))

    @staticmethod
    def real_chan(lib, dims, chan_dim, join=False):
        fn = lib.so.mdnn_nlop_chan_cplx if join else lib.so.mdnn_nlop_real_chan
        return Nlop(lib, fn(len(dims), _longs(dims), chan_dim))

    @staticmethod
    def batchnorm(lib, dims, flags, train=True, eps=1e-5, mom=0.1):
        return Nlop(lib, lib.so.mdnn_nlop_batchnorm(len(dims), _longs(dims), flags, int(train), eps, mom))

    @staticmethod
    def rbf(lib, z_dims, filter_dim, centers, sigma):
        c = (C.c_float * len(centers))(*centers)
        return Nlop(lib, lib.so.mdnn_nlop_rbf(len(z_dims), _longs(z_dims), filter_dim, len(centers), c, sigma))

    @staticmethod
    def pad(lib, in_dims, out_dims, corner):
        return Nlop(lib, lib.so.mdnn_nlop_pad(len(in_dims), _longs(in_dims), _longs(out_dims), _longs(corner)))

    def inverse(self, max_iter=10, tol=1e-6):
        return Nlop(self.lib, self.lib.so.mdnn_nlop_inverse(self.h, max_iter, tol))

    def checkpoint(self):
        """checkpoint(f) (nlop.hpp:516-522): recompute-for-memory container."""
        return Nlop(self.lib, self.lib.checkp(self.lib.so.mdnn_nlop_checkpoint(self.h)))

    def reexecutions(self):
        return self.lib.so.mdnn_nlop_checkpoint_reexecutions(self.h)


def sense_dims(x, y, coils=1, maps=1, batch=1):
    return mdnn_sense_dims(x, y, coils, maps, batch)


def modl_cfg(lib, **kw):
    c = mdnn_modl_cfg()
    lib.so.mdnn_modl_cfg_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def varnet_cfg(lib, **kw):
    c = mdnn_varnet_cfg()
    lib.so.mdnn_varnet_cfg_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class Model:
    def __init__(self, lib: Lib, h):
        self.lib = lib
        self.h = lib.checkp(h)

    def __del__(self):
        try:
            self.lib.so.mdnn_model_free(self.h)
        except Exception:
            pass

    @property
    def nlop(self):
        return Nlop(self.lib, self.lib.so.mdnn_model_nlop(self.h))

    @property
    def args(self):
        so = self.lib.so
        return [(so.mdnn_model_arg_name(self.h, i).decode(), so.mdnn_model_arg_kind(self.h, i),
                 bool(so.mdnn_model_arg_real(self.h, i))) for i in range(so.mdnn_model_n_args(self.h))]

    @property
    def arg_names(self):
        return [a[0] for a in self.args]

    @property
    def out_names(self):
        so = self.lib.so
        return [so.mdnn_model_out_name(self.h, o).decode() for o in range(so.mdnn_model_n_outs(self.h))]

    def arg_index(self, name):
        i = self.lib.so.mdnn_model_arg_index(self.h, name.encode())
        if i < 0:
            raise MdnnError(4, self.lib.so.mdnn_last_error().decode())
        return i

    def output_index(self, name):
        i = self.lib.so.mdnn_model_output_index(self.h, name.encode())
        if i < 0:
            raise MdnnError(4, self.lib.so.mdnn_last_error().decode())
        return i

    def num_real_params(self):
        return self.lib.so.mdnn_model_num_real_params(self.h)

    def init_weight(self, seed, name):
        i = self.arg_index(name)
        out = cfl_zeros(self.nlop.in_dims(i))
        self.lib.check(self.lib.so.mdnn_model_init_weight(self.h, seed, name.encode(), C.byref(self.lib.arr(out))))
        return out

    def init_weights(self, seed):
        return {n: self.init_weight(seed, n) for n, k, _ in self.args if k != ARG_DATA}

    # constructors
    @staticmethod
    def modl(lib, **kw):
        return Model(lib, lib.so.mdnn_build_modl(C.byref(modl_cfg(lib, **kw))))

    @staticmethod
    def varnet(lib, **kw):
        return Model(lib, lib.so.mdnn_build_varnet(C.byref(varnet_cfg(lib, **kw))))

    @staticmethod
    def modl_denoiser(lib, **kw):
        """D_W(x) = x + CNN(x) of one MoDL unroll (recon.hpp:714-803)."""
        return Model(lib, lib.so.mdnn_modl_denoiser(C.byref(modl_cfg(lib, **kw))))

    @staticmethod
    def varnet_reg(lib, **kw):
        """sum_f K^T Phi'(Re K x) of VarNet stage it0 (recon.hpp:522-609)."""
        return Model(lib, lib.so.mdnn_varnet_reg(C.byref(varnet_cfg(lib, **kw))))

    @staticmethod
    def bn_block(lib, name, dims):
        """Train-mode BN -> gamma -> beta -> CReLU of one denoiser layer (recon.hpp:748-776)."""
        d = (C.c_long * len(dims))(*dims)
        return Model(lib, lib.so.mdnn_bn_block(name.encode(), len(dims), d))

    def rebatch(self, batch):
        """Model::rebatch (nn.hpp:82): the same network for `batch` items."""
        return Model(self.lib, self.lib.so.mdnn_model_rebatch(self.h, int(batch)))

    @staticmethod
    def conv_layer(lib, name, in_dims, kernel, out_channels, axes=(0, 1), chan_dim=2, pad_same=True,
                   transposed=False, bias=False):
        s = mdnn_conv_spec()
        s.rank = len(in_dims)
        for k, v in enumerate(in_dims):
            s.in_dims[k] = v
        s.n_axes = len(axes)
        for k, (a, kk) in enumerate(zip(axes, kernel)):
            s.axes[k] = a
            s.kernel[k] = kk
        s.chan_dim = chan_dim
        s.out_channels = out_channels
        s.pad_same = int(pad_same)
        s.transposed = int(transposed)
        return Model(lib, lib.so.mdnn_conv_layer(name.encode(), C.byref(s), int(bias)))

    @staticmethod
    def batchnorm_layer(lib, name, dims, flags, train=True, eps=1e-5, mom=0.1):
        return Model(lib, lib.so.mdnn_batchnorm_layer(name.encode(), len(dims), _longs(dims), flags, int(train),
                                                      eps, mom))

    @staticmethod
    def sense_normal_fragment(lib, sd):
        return Model(lib, lib.so.mdnn_sense_normal_fragment(C.byref(sd)))

    @staticmethod
    def sense_adjoint_fragment(lib, sd):
        return Model(lib, lib.so.mdnn_sense_adjoint_fragment(C.byref(sd)))

    @staticmethod
    def modl_normal_plus_lambda(lib, sd):
        return Model(lib, lib.so.mdnn_modl_normal_plus_lambda(C.byref(sd)))


class Trainer:
    """run_step (optim.hpp:314) over the C ABI; inputs are host or device arrays."""

    def __init__(self, lib: Lib, model: Model, seed=42, lr=1e-3, **kw):
        c = mdnn_train_cfg()
        lib.so.mdnn_train_cfg_default(C.byref(c))
        c.lr = lr
        for k, v in kw.items():
            setattr(c, k, v)
        self.lib = lib
        self.model = model
        self.h = lib.checkp(lib.so.mdnn_trainer_create(model.h, C.byref(c), seed))

    def __del__(self):
        try:
            self.lib.so.mdnn_trainer_free(self.h)
        except Exception:
            pass

    def set_data(self, name, a):
        if isinstance(a, np.ndarray):
            a = np.asfortranarray(a.astype(np.complex64))
        self._keep = a
        self.lib.check(self.lib.so.mdnn_trainer_set_data(self.h, name.encode(), C.byref(self.lib.arr(a))))

    def stage_data(self, name, a):
        """Queue a host batch for data argument `name` (asynchronous copy on the
        library's copy stream; the next forward pass takes the oldest queued
        batch).  `a` is kept alive until two further batches were queued."""
        if isinstance(a, np.ndarray):
            a = np.asfortranarray(a.astype(np.complex64))
        self._staged = (getattr(self, "_staged", []) + [a])[-3 * 8:]
        self.lib.check(self.lib.so.mdnn_trainer_stage_data(self.h, name.encode(), C.byref(self.lib.arr(a))))

    def set_weight(self, name, a):
        a = np.asfortranarray(np.asarray(a, dtype=np.complex64))
        self.lib.check(self.lib.so.mdnn_trainer_set_weight(self.h, name.encode(), C.byref(self.lib.arr(a))))

    def save_weights(self, directory, meta=None):
        """WeightsBundle::save of every weight (cfl.hpp:97-111)."""
        meta = dict(meta or {})
        keys = (C.c_char_p * max(1, len(meta)))(*[k.encode() for k in meta])
        vals = (C.c_char_p * max(1, len(meta)))(*[str(v).encode() for v in meta.values()])
        self.lib.check(self.lib.so.mdnn_weights_save(self.h, str(directory).encode(), len(meta), keys, vals))

    def load_weights(self, directory):
        """WeightsBundle::load into the weights by name (cfl.hpp:113-135)."""
        self.lib.check(self.lib.so.mdnn_weights_load(self.h, str(directory).encode()))

    def weight_names(self):
        so = self.lib.so
        return [so.mdnn_trainer_weight_name(self.h, k).decode() for k in range(so.mdnn_trainer_n_weights(self.h))]

    def _dims_of(self, name):
        return self.model.nlop.in_dims(self.model.arg_index(name))

    def get_weight(self, name):
        out = cfl_zeros(self._dims_of(name))
        self.lib.check(self.lib.so.mdnn_trainer_get_weight(self.h, name.encode(), C.byref(self.lib.arr(out))))
        return out

    def get_grad(self, name):
        out = cfl_zeros(self._dims_of(name))
        self.lib.check(self.lib.so.mdnn_trainer_get_grad(self.h, name.encode(), C.byref(self.lib.arr(out))))
        return out

    def forward_backward(self):
        loss = C.c_double()
        self.lib.check(self.lib.so.mdnn_trainer_forward_backward(self.h, C.byref(loss)))
        return loss.value

    def grad_buffer(self):
        p, n = C.POINTER(C.c_float)(), C.c_long()
        self.lib.check(self.lib.so.mdnn_trainer_grad_buffer(self.h, C.byref(p), C.byref(n)))
        return C.cast(p, C.c_void_p).value, n.value

    def update(self, scale=1.0):
        self.lib.check(self.lib.so.mdnn_trainer_update(self.h, scale))

    def sync_buffer(self):
        """(address, floats) of the data-parallel payload [gradients | moving statistics]."""
        p, n = C.POINTER(C.c_float)(), C.c_long()
        self.lib.check(self.lib.so.mdnn_trainer_sync_buffer(self.h, C.byref(p), C.byref(n)))
        return C.cast(p, C.c_void_p).value, n.value

    def update_dp(self, world):
        self.lib.check(self.lib.so.mdnn_trainer_update_dp(self.h, int(world)))

    def set_comm(self, unique_id: bytes, nranks, rank):
        """Attach an in-library NCCL communicator (id from nccl_unique_id on rank 0)."""
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        self.lib.check(self.lib.so.mdnn_trainer_set_comm(self.h, C.cast(buf, C.c_void_p), int(nranks), int(rank)))

    def moving_stat_names(self):
        return [a for a, k, _ in self.model.args if k == ARG_MOVING_STATS]

    def step(self):
        loss = C.c_double()
        self.lib.check(self.lib.so.mdnn_trainer_step(self.h, C.byref(loss)))
        return loss.value


def nccl_unique_id(lib: Lib) -> bytes:
    buf = (C.c_uint8 * 128)()
    lib.check(lib.so.mdnn_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


# ---- cfl files (cfl.hpp:19-88) ----------------------------------------------
def cfl_dims(lib: Lib, base):
    d = (C.c_long * 16)()
    lib.check(lib.so.mdnn_cfl_dims(str(base).encode(), d))
    return tuple(d[k] for k in range(16))


def cfl_read(lib: Lib, base, out=None):
    """Read <base>.cfl into `out` (host numpy F-order or device torch array) or a new host array."""
    if out is None:
        out = cfl_zeros(cfl_dims(lib, base))
    lib.check(lib.so.mdnn_cfl_read(str(base).encode(), C.byref(lib.arr(out))))
    return out


def cfl_write(lib: Lib, base, a):
    if isinstance(a, np.ndarray):
        a = np.asfortranarray(a.astype(np.complex64))
    lib.check(lib.so.mdnn_cfl_write(str(base).encode(), C.byref(lib.arr(a))))


def weights_meta(lib: Lib, directory, key, fallback=""):
    buf = C.create_string_buffer(4096)
    lib.check(lib.so.mdnn_weights_meta(str(directory).encode(), key.encode(), fallback.encode(), buf, 4096))
    return buf.value.decode()
