"""World-size-2 tests of the data-parallel mapping step's host logic (gloo, CPU).

Only one GPU is available to this build, so the N>1 path is covered here:
every rank must draw the same keyframes (dp_select), the gradient exchange
(allreduce_step) must sum the ranks' slabs, and the replicated Adam update
that follows must leave identical parameters on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_23030_b200.mapping import allreduce_step, dp_select
        from paper_2511_23030_b200.select import KeyframeIndex, SelectConfig, record_loss
        idx = KeyframeIndex(config=SelectConfig(grid_resolution_m=100.0))
        rng = np.random.default_rng(0)          # same host state on every rank
        for k in range(10):
            idx.add(k, rng.uniform(-50, 50, 3))
        picks, params = [], torch.zeros(64, 16)
        m = torch.zeros_like(params)
        v = torch.zeros_like(params)
        for step in range(20):
            sel = dp_select(idx, 9, 7, step, world)
            picks.append(sel)
            # rank r "renders" keyframe sel[r]: a deterministic fake gradient
            g = torch.zeros_like(params)
            gen = torch.Generator().manual_seed(1000 * step + sel[rank])
            g[:, :14] = torch.randn(64, 14, generator=gen)
            buf = torch.zeros(world + 1)
            buf[rank] = float(sel[rank]) * 0.1 + step * 1e-3
            allreduce_step(g, buf, None)
            # the summed gradient must equal the sum of every rank's fake gradient
            ref = torch.zeros_like(g)
            for r in range(world):
                gr = torch.Generator().manual_seed(1000 * step + sel[r])
                ref[:, :14] += torch.randn(64, 14, generator=gr)
            assert torch.allclose(g, ref, atol=1e-6)
            # replicated Adam (same math on every rank)
            m.mul_(0.9).add_(g, alpha=0.1)
            v.mul_(0.999).addcmul_(g, g, value=0.001)
            params -= 1e-3 * m / (v.sqrt() + 1e-8)
            for r in range(world):   # every rank records every keyframe's loss, in order
                record_loss(sel[r], float(buf[r]), idx)
        out = [torch.zeros_like(params) for _ in range(world)]
        dist.all_gather(out, params)
        q.put((rank, picks, all(torch.equal(out[0], o) for o in out)))
    finally:
        dist.destroy_process_group()


def test_dp_step_host_logic_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == res[1][1]                 # identical keyframe plans on both ranks
    assert all(len(set(s)) >= 1 for s in res[0][1])
    assert res[0][2] and res[1][2]                # replicas stay bit-identical
