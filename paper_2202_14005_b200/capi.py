"""ctypes binding of the C ABI in include/mdnn.h.

The same binding drives the product library (csrc -> libmdnn_b200.so, device
arrays) and, in tests/bench only, the reference-backed oracle shim
(oracle/_ref/libmdnn_ref.so, host arrays).  Arrays cross the boundary as
`mdnn_array` structs: interleaved complex64, column-major (reference layout,
common.hpp:58-68), `device` -1 for host memory or a CUDA ordinal.

Host arrays are numpy complex64 arrays in Fortran order whose numpy shape is
the reference dims; device arrays are torch complex64 tensors whose torch
shape is the reversed dims (so torch's row-major storage is the same bytes).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

MAX_RANK = 16
ERR_NAMES = {1: "Error", 2: "ShapeError", 3: "IoError", 4: "ConfigError", 5: "SolverError",
             6: "BoundsError", 7: "AliasError", 8: "StaleDerivativeError", 9: "CudaError"}
ARG_DATA, ARG_WEIGHTS, ARG_MOVING_STATS = 0, 1, 2


class MdnnError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERR_NAMES.get(code, 'Error')}: {msg}")
        self.code = code
        self.kind = ERR_NAMES.get(code, "Error")


class mdnn_array(C.Structure):
    _fields_ = [("data", C.c_void_p), ("rank", C.c_int), ("device", C.c_int),
                ("dims", C.c_long * MAX_RANK), ("strides", C.c_long * MAX_RANK),
                ("has_strides", C.c_int)]


class mdnn_sense_dims(C.Structure):
    _fields_ = [("x", C.c_long), ("y", C.c_long), ("coils", C.c_long), ("maps", C.c_long), ("batch", C.c_long)]


class mdnn_conv_spec(C.Structure):
    _fields_ = [("rank", C.c_int), ("in_dims", C.c_long * MAX_RANK), ("n_axes", C.c_int),
                ("axes", C.c_int * 4), ("kernel", C.c_long * 4), ("chan_dim", C.c_int),
                ("out_channels", C.c_long), ("pad_same", C.c_int), ("transposed", C.c_int)]


class mdnn_modl_cfg(C.Structure):
    _fields_ = [("iterations", C.c_long), ("layers", C.c_long), ("filters", C.c_long), ("kernel", C.c_long),
                ("cg_iter", C.c_long), ("cg_tol", C.c_double), ("lambda_init", C.c_double),
                ("im_x", C.c_long), ("im_y", C.c_long), ("coils", C.c_long), ("maps", C.c_long),
                ("batch", C.c_long), ("train_mode", C.c_int)]


class mdnn_varnet_cfg(C.Structure):
    _fields_ = [("iterations", C.c_long), ("filters", C.c_long), ("kernel", C.c_long), ("rbf", C.c_long),
                ("im_x", C.c_long), ("im_y", C.c_long), ("coils", C.c_long), ("maps", C.c_long),
                ("batch", C.c_long)]


class mdnn_train_cfg(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("clip", C.c_double), ("algo", C.c_int), ("ipalm_alpha", C.c_double), ("ipalm_beta", C.c_double)]


ALGO_SGD, ALGO_ADAM, ALGO_IPALM = 0, 1, 2


class mdnn_reconet_opts(C.Structure):
    _fields_ = [("network", C.c_char_p), ("do_train", C.c_int), ("do_apply", C.c_int), ("normalize", C.c_int),
                ("pattern_file", C.c_char_p), ("init_weights", C.c_char_p),
                ("iterations", C.c_long), ("filters", C.c_long), ("kernel", C.c_long), ("rbf", C.c_long),
                ("layers", C.c_long), ("cg_iter", C.c_long), ("epochs", C.c_long), ("batch_size", C.c_long),
                ("lr", C.c_double), ("optimizer", C.c_char_p), ("seed", C.c_uint64), ("verbose", C.c_int),
                ("kspace_file", C.c_char_p), ("coils_file", C.c_char_p), ("weights_dir", C.c_char_p),
                ("target_file", C.c_char_p)]


P = C.c_void_p
L = C.POINTER(C.c_long)
_SIGS = {
    "mdnn_last_error": (C.c_char_p, []),
    "mdnn_backend": (C.c_char_p, []),
    "mdnn_set_device": (C.c_int, [C.c_int]),
    "mdnn_synchronize": (C.c_int, []),
    "mdnn_set_option": (C.c_int, [C.c_char_p, C.c_long]),
    "mdnn_stream": (C.c_void_p, []),
    "mdnn_profile_enable": (C.c_int, [C.c_int]),
    "mdnn_profile_read": (C.c_int, [C.c_char_p, C.POINTER(C.c_long), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]),
    "mdnn_profile_reset": (C.c_int, []),
    "mdnn_launch_count": (C.c_long, []),
    "mdnn_nlop_free": (None, [P]),
    "mdnn_nlop_ref": (P, [P]),
    "mdnn_nlop_n_in": (C.c_int, [P]),
    "mdnn_nlop_n_out": (C.c_int, [P]),
    "mdnn_nlop_in_dims": (C.c_int, [P, C.c_int, C.POINTER(C.c_int), L]),
    "mdnn_nlop_out_dims": (C.c_int, [P, C.c_int, C.POINTER(C.c_int), L]),
    "mdnn_nlop_apply": (C.c_int, [P, C.c_int, C.POINTER(mdnn_array), C.c_int, C.POINTER(mdnn_array)]),
    "mdnn_nlop_derivative": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(mdnn_array), C.POINTER(mdnn_array)]),
    "mdnn_nlop_adjoint": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(mdnn_array), C.POINTER(mdnn_array)]),
    "mdnn_nlop_adjoint_all": (C.c_int, [P, C.c_int, C.POINTER(mdnn_array), C.c_int, C.POINTER(mdnn_array),
                                        C.POINTER(C.c_uint8)]),
    "mdnn_nlop_combine": (P, [P, P]),
    "mdnn_nlop_link": (P, [P, C.c_int, C.c_int]),
    "mdnn_nlop_duplicate": (P, [P, C.c_int, C.c_int]),
    "mdnn_nlop_chain": (P, [P, P]),
    "mdnn_nlop_dft": (P, [C.c_int, L, C.c_ulong, C.c_int]),
    "mdnn_nlop_tenmul": (P, [C.c_int, L, L, L, L, L, L, L]),
    "mdnn_nlop_add": (P, [C.c_int, L, C.c_int]),
    "mdnn_nlop_bcast_add": (P, [C.c_int, L, L]),
    "mdnn_nlop_fork": (P, [C.c_int, L, C.c_int]),
    "mdnn_nlop_zconj": (P, [C.c_int, L]),
    "mdnn_nlop_zreal": (P, [C.c_int, L]),
    "mdnn_nlop_real_chan": (P, [C.c_int, L, C.c_int]),
    "mdnn_nlop_chan_cplx": (P, [C.c_int, L, C.c_int]),
    "mdnn_nlop_crelu": (P, [C.c_int, L]),
    "mdnn_nlop_exp_real": (P, [C.c_int, L]),
    "mdnn_nlop_mse": (P, [C.c_int, L]),
    "mdnn_nlop_batchnorm": (P, [C.c_int, L, C.c_ulong, C.c_int, C.c_double, C.c_double]),
    "mdnn_nlop_rbf": (P, [C.c_int, L, C.c_int, C.c_int, C.POINTER(C.c_float), C.c_float]),
    "mdnn_nlop_pad": (P, [C.c_int, L, L, L]),
    "mdnn_nlop_inverse": (P, [P, C.c_long, C.c_double]),
    "mdnn_nlop_checkpoint": (P, [P]),
    "mdnn_nlop_checkpoint_reexecutions": (C.c_long, [P]),
    "mdnn_nlop_cg_status": (C.c_int, [P, L, C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    "mdnn_sense_forward": (C.c_int, [C.POINTER(mdnn_array)] * 4),
    "mdnn_sense_adjoint": (C.c_int, [C.POINTER(mdnn_array)] * 4),
    "mdnn_sense_normal": (C.c_int, [C.POINTER(mdnn_array), C.POINTER(mdnn_array), C.c_float,
                                    C.POINTER(mdnn_array), C.POINTER(mdnn_array)]),
    "mdnn_cg_normal_solve": (C.c_int, [C.POINTER(mdnn_array), C.POINTER(mdnn_array), C.c_float,
                                       C.POINTER(mdnn_array), C.c_long, C.c_double, C.POINTER(mdnn_array),
                                       L, C.POINTER(C.c_double)]),
    "mdnn_dft": (C.c_int, [C.POINTER(mdnn_array), C.c_ulong, C.c_int, C.POINTER(mdnn_array)]),
    "mdnn_model_free": (None, [P]),
    "mdnn_model_nlop": (P, [P]),
    "mdnn_model_n_args": (C.c_int, [P]),
    "mdnn_model_arg_name": (C.c_char_p, [P, C.c_int]),
    "mdnn_model_arg_kind": (C.c_int, [P, C.c_int]),
    "mdnn_model_arg_real": (C.c_int, [P, C.c_int]),
    "mdnn_model_n_outs": (C.c_int, [P]),
    "mdnn_model_out_name": (C.c_char_p, [P, C.c_int]),
    "mdnn_model_arg_index": (C.c_int, [P, C.c_char_p]),
    "mdnn_model_output_index": (C.c_int, [P, C.c_char_p]),
    "mdnn_model_num_real_params": (C.c_long, [P]),
    "mdnn_model_init_weight": (C.c_int, [P, C.c_uint64, C.c_char_p, C.POINTER(mdnn_array)]),
    "mdnn_model_chain": (P, [P, P, C.c_char_p, C.c_int]),
    "mdnn_model_link": (P, [P, C.c_int, C.c_char_p]),
    "mdnn_model_combine": (P, [P, P]),
    "mdnn_model_dedupe": (P, [P]),
    "mdnn_conv_layer": (P, [C.c_char_p, C.POINTER(mdnn_conv_spec), C.c_int]),
    "mdnn_batchnorm_layer": (P, [C.c_char_p, C.c_int, L, C.c_ulong, C.c_int, C.c_double, C.c_double]),
    "mdnn_modl_cfg_default": (None, [C.POINTER(mdnn_modl_cfg)]),
    "mdnn_varnet_cfg_default": (None, [C.POINTER(mdnn_varnet_cfg)]),
    "mdnn_build_modl": (P, [C.POINTER(mdnn_modl_cfg)]),
    "mdnn_build_varnet": (P, [C.POINTER(mdnn_varnet_cfg)]),
    "mdnn_sense_normal_fragment": (P, [C.POINTER(mdnn_sense_dims)]),
    "mdnn_sense_adjoint_fragment": (P, [C.POINTER(mdnn_sense_dims)]),
    "mdnn_modl_normal_plus_lambda": (P, [C.POINTER(mdnn_sense_dims)]),
    "mdnn_model_rebatch": (P, [P, L]),
    "mdnn_modl_denoiser": (P, [C.POINTER(mdnn_modl_cfg)]),
    "mdnn_bn_block": (P, [C.c_char_p, C.c_int, L]),
    "mdnn_varnet_reg": (P, [C.POINTER(mdnn_varnet_cfg)]),
    "mdnn_loss_model_mse": (P, [C.c_int, L]),
    "mdnn_sim_item": (C.c_int, [C.c_uint64, C.c_long, C.c_long, C.c_long, C.c_long, P, P]),
    "mdnn_sim_pattern": (C.c_int, [C.c_long, C.c_long, C.c_long, P]),
    "mdnn_train_cfg_default": (None, [C.POINTER(mdnn_train_cfg)]),
    "mdnn_trainer_create": (P, [P, C.POINTER(mdnn_train_cfg), C.c_uint64]),
    "mdnn_trainer_free": (None, [P]),
    "mdnn_trainer_set_data": (C.c_int, [P, C.c_char_p, C.POINTER(mdnn_array)]),
    "mdnn_trainer_stage_data": (C.c_int, [P, C.c_char_p, C.POINTER(mdnn_array)]),
    "mdnn_trainer_set_weight": (C.c_int, [P, C.c_char_p, C.POINTER(mdnn_array)]),
    "mdnn_trainer_get_weight": (C.c_int, [P, C.c_char_p, C.POINTER(mdnn_array)]),
    "mdnn_trainer_get_grad": (C.c_int, [P, C.c_char_p, C.POINTER(mdnn_array)]),
    "mdnn_trainer_forward_backward": (C.c_int, [P, C.POINTER(C.c_double)]),
    "mdnn_trainer_grad_buffer": (C.c_int, [P, C.POINTER(C.POINTER(C.c_float)), L]),
    "mdnn_trainer_update": (C.c_int, [P, C.c_float]),
    "mdnn_trainer_step": (C.c_int, [P, C.POINTER(C.c_double)]),
    "mdnn_trainer_sync_buffer": (C.c_int, [P, C.POINTER(C.POINTER(C.c_float)), L]),
    "mdnn_trainer_update_dp": (C.c_int, [P, C.c_int]),
    "mdnn_nccl_unique_id": (C.c_int, [P]),
    "mdnn_trainer_set_comm": (C.c_int, [P, P, C.c_int, C.c_int]),
    "mdnn_trainer_n_weights": (C.c_int, [P]),
    "mdnn_trainer_weight_name": (C.c_char_p, [P, C.c_int]),
    "mdnn_reconet_opts_default": (None, [C.POINTER(mdnn_reconet_opts)]),
    "mdnn_reconet": (C.c_int, [C.POINTER(mdnn_reconet_opts)]),
    "mdnn_estimate_pattern": (C.c_int, [C.POINTER(mdnn_array), C.POINTER(mdnn_array)]),
    "mdnn_cfl_dims": (C.c_int, [C.c_char_p, L]),
    "mdnn_cfl_read": (C.c_int, [C.c_char_p, C.POINTER(mdnn_array)]),
    "mdnn_cfl_write": (C.c_int, [C.c_char_p, C.POINTER(mdnn_array)]),
    "mdnn_weights_save": (C.c_int, [P, C.c_char_p, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p)]),
    "mdnn_weights_load": (C.c_int, [P, C.c_char_p]),
    "mdnn_weights_meta": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_long]),
}
EXPORTED_SYMBOLS = tuple(_SIGS)


def _longs(seq):
    arr = (C.c_long * MAX_RANK)()
    for k, v in enumerate(seq):
        arr[k] = int(v)
    return arr


def dims16(*head):
    d = [1] * MAX_RANK
    for k, v in enumerate(head):
        d[k] = int(v)
    return d


class Lib:
    """One loaded implementation of include/mdnn.h."""

    def __init__(self, path):
        self.path = os.path.abspath(path)
        self.so = C.CDLL(self.path, mode=C.RTLD_LOCAL)
        for name, (res, args) in _SIGS.items():
            fn = getattr(self.so, name)
            fn.restype = res
            fn.argtypes = args
        self.backend = self.so.mdnn_backend().decode()
        self.is_device = self.backend.startswith("b200")

    # -- errors -------------------------------------------------------------
    def check(self, code):
        if code != 0:
            raise MdnnError(code, self.so.mdnn_last_error().decode())

    def checkp(self, ptr):
        if not ptr:
            msg = self.so.mdnn_last_error().decode()
            raise MdnnError(self._code_from_msg(msg), msg)
        return ptr

    @staticmethod
    def _code_from_msg(msg):
        return 1

    def __getattr__(self, name):
        return getattr(self.so, name)

    # -- arrays -------------------------------------------------------------
    def arr(self, a, dims=None):
        """mdnn_array view of a numpy (host) or torch (device) complex64 array."""
        s = mdnn_array()
        if isinstance(a, np.ndarray):
            assert a.dtype == np.complex64, a.dtype
            if dims is None:
                dims = a.shape
            assert a.flags.f_contiguous or a.size <= 1 or a.ndim <= 1
            s.data = a.ctypes.data
            s.device = -1
        else:  # torch tensor, reversed shape
            import torch
            assert a.dtype == torch.complex64 and a.is_contiguous()
            if dims is None:
                dims = tuple(reversed(a.shape))
            s.data = a.data_ptr()
            s.device = a.device.index if a.is_cuda else -1
        s.rank = len(dims)
        for k, v in enumerate(dims):
            s.dims[k] = int(v)
        s.has_strides = 0
        return s

    def zeros(self, dims, device=None):
        if device is None:
            return np.zeros(tuple(dims), dtype=np.complex64, order="F")
        import torch
        return torch.zeros(tuple(reversed(dims)), dtype=torch.complex64, device=device)

    # -- nlop helpers -------------------------------------------------------
    def nlop_dims(self, h, i, out=False):
        r = C.c_int()
        d = (C.c_long * MAX_RANK)()
        self.check((self.so.mdnn_nlop_out_dims if out else self.so.mdnn_nlop_in_dims)(h, i, C.byref(r), d))
        return tuple(d[k] for k in range(r.value))


def to_host(x):
    """numpy complex64 F-order array from a torch device tensor (reversed shape)."""
    if isinstance(x, np.ndarray):
        return x
    return np.asfortranarray(x.detach().cpu().numpy().transpose())


def to_device(a, device="cuda"):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a.transpose()))
    return t.to(device)
