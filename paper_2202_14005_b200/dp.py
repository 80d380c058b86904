"""Data-parallel training step (BART batch stacking).

One process per GPU.  Each rank runs forward + backward on its batch shard
through the C ABI, the flat fp32 weight-gradient buffer is summed across ranks
with torch.distributed (NCCL over NVLink on B200, ordered on the library's own
CUDA stream; gloo on host memory for the CPU tests), and every rank applies the
identical Adam update with gradient scale 1/world — so replicas stay bitwise
identical.  Per-shard semantics: CG scalars and train-mode BN statistics span
the rank's shard, exactly as if the reference ran on that shard.
"""
from __future__ import annotations

import ctypes as C

import numpy as np


class _DevBuf:
    def __init__(self, ptr, n, stream):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                         "stream": stream or 1}


class DataParallelTrainer:
    def __init__(self, trainer, world: int = 1, group=None, device=None):
        import torch
        self.tr = trainer
        self.world = world
        self.group = group
        lib = trainer.lib
        ptr, n = trainer.grad_buffer()
        self.is_device = lib.is_device
        if self.is_device:
            stream_ptr = lib.so.mdnn_stream()
            self.stream = torch.cuda.ExternalStream(stream_ptr, device=device)
            self.grads = torch.as_tensor(_DevBuf(ptr, n, stream_ptr), device=device)
        else:
            self.stream = None
            buf = (C.c_float * n).from_address(ptr)
            self.grads = torch.from_numpy(np.frombuffer(buf, dtype=np.float32))

    def allreduce(self):
        if self.world <= 1:
            return
        import torch
        import torch.distributed as dist
        if self.stream is not None:
            with torch.cuda.stream(self.stream):
                dist.all_reduce(self.grads, group=self.group)
        else:
            dist.all_reduce(self.grads, group=self.group)

    def step(self) -> float:
        loss = self.tr.forward_backward()
        self.allreduce()
        self.tr.update(1.0 / self.world)
        return loss
