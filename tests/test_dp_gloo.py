"""World-size-2 tests of the data-parallel mapping step's host logic (gloo, CPU).

Only one GPU is available to this build, so the N>1 path is covered here with
C3's shape (K = 8 keyframes per step over G = 2 ranks): every rank must draw
the same K keyframes (dp_select), own keyframes r, r + G, ...
(owned_keyframes), and the exchange (allreduce_step) must turn the ranks'
partial gradient sums and loss slots into exactly what one rank
accumulating all K keyframes holds; the replicated Adam that follows must
leave identical parameters on every rank.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

K = 8


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_grad(step: int, j: int, kf: int) -> torch.Tensor:
    """Keyframe j's gradient records of one step (integers: exact sums)."""
    gen = torch.Generator().manual_seed(1000 * step + 31 * j + kf)
    g = torch.zeros(64, 16)
    g[:, :14] = torch.randint(-1000, 1000, (64, 14), generator=gen).float()
    return g


def _worker(rank: int, world: int, port: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_23030_b200.mapping import allreduce_step, dp_select, owned_keyframes
        from paper_2511_23030_b200.select import KeyframeIndex, SelectConfig, record_loss
        idx = KeyframeIndex(config=SelectConfig(grid_resolution_m=100.0))
        rng = np.random.default_rng(0)          # same host state on every rank
        for k in range(10):
            idx.add(k, rng.uniform(-50, 50, 3))
        picks, params = [], torch.zeros(64, 16)
        m = torch.zeros_like(params)
        v = torch.zeros_like(params)
        owned = []
        for step in range(20):
            sel = dp_select(idx, 9, 7, step, K)
            picks.append(sel)
            mine = owned_keyframes(K, world, rank)
            owned.append(mine)
            packed = torch.zeros(64, 16)
            buf = torch.zeros(K + 1)
            for j in mine:   # rank r renders keyframes r, r+G, ...: gradients accumulate
                packed += _fake_grad(step, j, sel[j])
                buf[j] = float(sel[j]) * 0.1 + step * 1e-3
            allreduce_step(packed, buf, None)
            ref = sum(_fake_grad(step, j, sel[j]) for j in range(K))   # one rank, all K keyframes
            assert torch.equal(packed, ref)
            assert torch.equal(buf[:K], torch.tensor([float(sel[j]) * 0.1 + step * 1e-3 for j in range(K)]))
            assert float(buf[K]) == 0.0
            # replicated Adam (same math on every rank)
            m.mul_(0.9).add_(packed, alpha=0.1)
            v.mul_(0.999).addcmul_(packed, packed, value=0.001)
            params -= 1e-3 * m / (v.sqrt() + 1e-8)
            for j in range(K):   # every rank records every keyframe's loss, in order
                record_loss(sel[j], float(buf[j]), idx)
        out = [torch.zeros_like(params) for _ in range(world)]
        dist.all_gather(out, params)
        q.put((rank, picks, owned, all(torch.equal(out[0], o) for o in out)))
    finally:
        dist.destroy_process_group()


def test_dp_step_host_logic_world2_k8():
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
    assert all(len(s) == K for s in res[0][1])
    assert res[0][2][0] == [0, 2, 4, 6] and res[1][2][0] == [1, 3, 5, 7]
    assert res[0][3] and res[1][3]                # replicas stay bit-identical


def test_dp_select_k1_is_the_single_step_draw():
    """K = 1 draws exactly what optimization_step draws (derive_seed(seed, 2, step))."""
    from paper_2511_23030_b200.mapping import derive_seed, dp_select
    from paper_2511_23030_b200.select import KeyframeIndex, SelectConfig, candidate_set, select_keyframe
    idx = KeyframeIndex(config=SelectConfig(grid_resolution_m=100.0))
    rng = np.random.default_rng(1)
    for k in range(6):
        idx.add(k, rng.uniform(-30, 30, 3))
    for step in range(30):
        cands = candidate_set(idx.position_of(5), idx)
        assert dp_select(idx, 5, 7, step, 1) == [select_keyframe(cands, idx, derive_seed(7, 2, step))]
