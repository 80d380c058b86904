"""Data-parallel training step (BART batch stacking).

One process per GPU.  Each rank runs forward + backward on its batch shard
through the C ABI; the sync buffer [weight gradients | BN moving statistics]
is summed across ranks, and every rank applies the identical Adam update with
gradient scale 1/world and takes the replica mean of the moving statistics
(mdnn_trainer_update_dp) -- so replicas, including the BN running statistics
that eval-mode inference uses, stay bitwise identical.  Per-shard semantics:
CG scalars and train-mode BN batch statistics span the rank's shard, exactly
as if the reference ran on that shard.

Two exchange paths:
  * ``comm="library"`` (GPU product): an NCCL communicator inside the library
    (mdnn_trainer_set_comm); the trainer all-reduces gradient buckets on its
    comm stream while the reverse sweep is still running.  A C++ caller of the
    C ABI gets the same path without Python.
  * ``comm="torch"``: torch.distributed all-reduce of the whole sync buffer
    (gloo on host memory for the CPU tests; NCCL on the library stream).
"""
from __future__ import annotations

import ctypes as C

import numpy as np


class _DevBuf:
    def __init__(self, ptr, n, stream):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                         "stream": stream or 1}


class DataParallelTrainer:
    def __init__(self, trainer, world: int = 1, group=None, device=None, comm: str = "torch", rank: int = 0):
        import torch
        self.tr = trainer
        self.world = world
        self.group = group
        self.comm = comm if world > 1 else "none"
        lib = trainer.lib
        self.is_device = lib.is_device
        if self.comm == "library":
            import torch.distributed as dist
            from .mdnn import nccl_unique_id
            obj = [nccl_unique_id(lib) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            trainer.set_comm(obj[0], world, rank)
            return
        ptr, n = trainer.sync_buffer()
        if self.is_device:
            stream_ptr = lib.so.mdnn_stream()
            self.stream = torch.cuda.ExternalStream(stream_ptr, device=device)
            self.buf = torch.as_tensor(_DevBuf(ptr, n, stream_ptr), device=device)
        else:
            self.stream = None
            self.buf = torch.from_numpy(np.frombuffer((C.c_float * n).from_address(ptr), dtype=np.float32))

    def allreduce(self):
        if self.comm != "torch":
            return
        import torch
        import torch.distributed as dist
        if self.stream is not None:
            with torch.cuda.stream(self.stream):
                dist.all_reduce(self.buf, group=self.group)
        else:
            dist.all_reduce(self.buf, group=self.group)

    def step(self) -> float:
        if self.comm == "library":
            return self.tr.step()  # bucketed NCCL all-reduce inside the library + update_dp
        loss = self.tr.forward_backward()
        self.allreduce()
        if self.world > 1:
            self.tr.update_dp(self.world)
        else:
            self.tr.update(1.0)
        return loss
