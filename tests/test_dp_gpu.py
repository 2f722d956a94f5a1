"""The data-parallel mapping step's device path with two ranks (GPU).

Only one GPU per run: both ranks place their engines on cuda:0 and exchange
through gloo (a host-side all-reduce), so neither rank's kernels wait on the
other's -- the device work is the real DP step (graph replays of fwd -> loss
-> bwd, gradient all-reduce of the slab, replicated Adam) and the check is
that both replicas see both keyframes' losses and stay bit-identical.
(World-1 equality with the single-GPU step: test_mapping_gpu.py.)
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, root: str, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2511_23030_b200.workloads import build_c1
        eng = build_c1(n=20_000, keyframes=10, budget=100_000, store_dir=os.path.join(root, f"r{rank}"))
        losses = []
        for s in range(6):
            rows = eng.optimization_step_dp(0, s, world, rank)
            losses.append([r.loss for r in rows])
        torch.cuda.synchronize()
        hw = eng.store.slab.high_water()
        q.put((rank, losses, eng.store.slab.params[:hw].cpu().numpy(), eng.store.slab.adam_m[:hw].cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_dp_world2_device_step_replicas_identical(cuda, tmp_path):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, str(tmp_path), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, losses, params, m = q.get(timeout=600)
        res[rank] = (losses, params, m)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (l0, p0, m0), (l1, p1, m1) = res[0], res[1]
    assert l0 == l1                       # both ranks saw both keyframes' losses
    assert np.array_equal(p0, p1) and np.array_equal(m0, m1)   # replicas identical
    assert np.all(np.isfinite(l0)) and len(l0[0]) == 2
    assert float(np.abs(m0[:, :14]).max()) > 0.0   # Adam moved something
