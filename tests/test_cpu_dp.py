"""Multi-process data parallelism on CPU (gloo, world_size 2) through the same
C ABI and the product's DataParallelTrainer, driving the reference-backed
library (the GPU library needs a device).  Checks that (1) replicas stay
bitwise identical -- trainable weights and the BN moving statistics that
eval-mode inference reads -- and (2) the result equals one process that
averages the two shards' gradients and moving statistics before the same
Adam update."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import REPO

CFG = dict(iterations=1, layers=2, filters=3, cg_iter=3, im_x=10, im_y=8, coils=2, batch=1)


def _data(lib, item):
    import sys
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import ctypes as C
    from util import kspace_dims, sim_data
    ph, cm, pat = sim_data(lib, 10, 8, 2, 1, accel=3, acl=2, seed=1 + item)
    ks = np.zeros(kspace_dims(10, 8, 2), dtype=np.complex64, order="F")
    lib.check(lib.so.mdnn_sense_forward(C.byref(lib.arr(cm)), C.byref(lib.arr(pat)), C.byref(lib.arr(ph)),
                                        C.byref(lib.arr(ks))))
    return {"kspace": ks, "coils": cm, "pattern": pat, "reference": ph}


def _worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, REPO)
    import torch.distributed as dist
    from paper_2202_14005_b200.capi import Lib
    from paper_2202_14005_b200.dp import DataParallelTrainer
    from paper_2202_14005_b200.mdnn import Model, Trainer
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = Lib(os.path.join(REPO, "oracle", "_ref", "libmdnn_ref.so"))
    tr = Trainer(lib, Model.modl(lib, **CFG), seed=42)
    for k, v in _data(lib, rank).items():
        tr.set_data(k, v)
    dp = DataParallelTrainer(tr, world=world)
    losses = [dp.step() for _ in range(2)]
    names = tr.weight_names() + tr.moving_stat_names()
    out_q.put((rank, losses, {n: tr.get_weight(n) for n in names}))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_matches_averaged_single_process(ref):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (l, w)) for r, l, w in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w0, w1 = res[0][1], res[1][1]
    assert any("bn_mean" in k for k in w0) and any("bn_var" in k for k in w0)
    for k in w0:
        assert np.array_equal(w0[k], w1[k]), k  # replicas bitwise identical, moving statistics included

    # single process: average the two shards' gradients, same update
    from paper_2202_14005_b200.mdnn import Model, Trainer
    trs = []
    for item in range(2):
        t = Trainer(ref, Model.modl(ref, **CFG), seed=42)
        for k, v in _data(ref, item).items():
            t.set_data(k, v)
        trs.append(t)
    import ctypes as C
    for _ in range(2):
        bufs = []
        for t in trs:
            t.forward_backward()
            p, n = t.sync_buffer()
            bufs.append(np.frombuffer((C.c_float * n).from_address(p), dtype=np.float32))
        s = bufs[0] + bufs[1]
        for b in bufs:
            b[:] = s
        for t in trs:
            t.update_dp(2)
    for k in w0:
        np.testing.assert_allclose(w0[k], trs[0].get_weight(k), rtol=1e-6, atol=1e-7)
