"""CPU tests of the host-side policy and formats against reference fixtures.

Everything here runs without a GPU: chunk ids (grid.py), frustum planes
(culling.py:80-101), keyframe selection (select.py), the .dcg/.dkf codecs
(diskformat.py), and the mapping-step metrics format (sim.py:66-87).
"""
import json

import numpy as np
import pytest

from paper_2511_23030_b200 import diskformat, grid, select
from paper_2511_23030_b200.core import CameraIntrinsics, Gaussian, Keyframe, Pose, quat_normalize
from paper_2511_23030_b200.culling import extract_frustum
from paper_2511_23030_b200.errors import CorruptChunk, Malformed, OutOfRange
from tests.conftest import GOLDEN


def test_encode_positions_bit_exact(golden):
    g = golden("grid.npz")
    for k in range(3):
        ids = grid.encode_positions(g[f"s{k}_positions"], float(g[f"s{k}_size"]))
        assert np.array_equal(ids, g[f"s{k}_ids"])


def test_grid_known_answers():
    # test_grid.py / test_acceptance.py criterion 1
    assert grid.encode_id(grid.ChunkCoord(0, 0, 0)) == 4611688217451692032
    assert grid.encode_id(grid.ChunkCoord(grid.COORD_MIN, grid.COORD_MIN, grid.COORD_MIN)) == 0
    c = grid.ChunkCoord(123, -456, 789)
    assert grid.decode_id(grid.encode_id(c)) == c
    assert grid.chunk_coord([4.999, -5.0, 5.0], 10.0) == grid.ChunkCoord(0, 0, 1)
    with pytest.raises(OutOfRange):
        grid.encode_id(grid.ChunkCoord(grid.COORD_MAX + 1, 0, 0))
    with pytest.raises(Malformed):
        grid.decode_id(1 << 63)
    rng = np.random.default_rng(1)
    coords = rng.integers(grid.COORD_MIN, grid.COORD_MAX + 1, size=(2000, 3))
    ids = np.array([grid.encode_id(grid.ChunkCoord(*map(int, c))) for c in coords], dtype=np.uint64)
    assert np.array_equal(grid.decode_ids(ids), coords)


def test_frustum_planes_bit_exact(golden):
    g = golden("grid.npz")
    it = g["intr"]
    intr = CameraIntrinsics(fx=it[0], fy=it[1], cx=it[2], cy=it[3], near=it[4], far=it[5],
                            width=int(it[6]), height=int(it[7]))
    for t in range(int(g["vis_count"])):
        pose = Pose(rotation=g[f"v{t}_pose_q"], translation=g[f"v{t}_pose_t"])
        assert np.array_equal(extract_frustum(pose, intr).planes, g[f"v{t}_planes"])


def test_keyframe_selection_trace():
    ops = json.loads((GOLDEN / "select_trace.json").read_text())
    idx = select.KeyframeIndex(config=select.SelectConfig(grid_resolution_m=50.0))
    from paper_2511_23030_b200.mapping import derive_seed
    for op in ops:
        if op["op"] == "add":
            idx.add(op["id"], op["pos"])
            continue
        latest = op["latest"]
        try:
            cands = select.candidate_set(idx.position_of(latest), idx)
        except Exception:
            cands = [latest]
        assert cands == op["cands"]
        seed = derive_seed(7, 2, ops.index(op) - 12)
        assert seed == op["seed"]
        chosen = select.select_keyframe(cands, idx, seed)
        assert chosen == op["chosen"]
        select.record_loss(chosen, op["loss"], idx)
        assert [idx.usage_of(i) for i in range(12)] == op["usage"]


def test_fast_selection_and_quantile_match_numpy():
    """The precomputed-uniform draw and the pure-Python quantile are the
    NumPy computations the reference uses (select.py:144-166), bit for bit."""
    rng = np.random.default_rng(5)
    for trial in range(3000):
        k = int(rng.integers(1, 20))
        w = rng.uniform(0, 3, k) * (rng.random(k) > 0.2) + (rng.random(k) < 0.1) * 1e-7
        w = np.maximum(w, 1e-6)
        p = w / w.sum()
        seed = int(rng.integers(0, 2**63))
        ref = int(np.random.default_rng(seed).choice(k, p=p))
        u = select.draw_uniform(seed)
        cdf = p.cumsum()
        cdf /= cdf[-1]
        assert int(cdf.searchsorted(u, side="right")) == ref
        vals = list(rng.uniform(0, 2, int(rng.integers(1, 30))))
        for q in (0.5, 0.25, 0.9, 1.0, 0.0):
            assert select.quantile_linear(vals, q) == float(np.quantile(vals, q))


def test_chunk_codec_matches_reference_bytes(golden):
    g = golden("diskformat.npz")
    gs = [Gaussian(position=g["positions"][i], rotation=g["rotations"][i], scale=g["scales"][i],
                   opacity=float(g["opacities"][i]), sh=g["sh"][i]) for i in range(len(g["positions"]))]
    plain = diskformat.pack_chunk(0x123456789A, gs)
    assert plain == g["chunk_plain"].tobytes()
    blob, off = g["opt_blob"].tobytes(), 0
    for gg, n in zip(gs, g["opt_lens"]):
        gg.opt_state = blob[off:off + int(n)]
        off += int(n)
    assert diskformat.pack_chunk(0xABCDEF, gs) == g["chunk_opt"].tobytes()
    cid, back = diskformat.unpack_chunk(g["chunk_opt"].tobytes())
    assert cid == 0xABCDEF and [x.opt_state for x in back] == [x.opt_state for x in gs]
    # uniform-stride zero-copy view used by the device codec
    cid, count, recs, stride = diskformat.parse_chunk_records(plain)
    assert (cid, count, stride) == (0x123456789A, len(gs), 240)
    assert np.array_equal(recs["position"].astype(np.float64), g["positions"])
    assert diskformat.parse_chunk_records(g["chunk_opt"].tobytes())[2] is None   # foreign tails
    assert diskformat.build_chunk_file(0x123456789A, recs) == plain


def test_keyframe_codec_matches_reference_bytes(golden):
    g = golden("diskformat.npz")
    kf = Keyframe(id=42, pose=Pose(rotation=g["kf_pose_q"], translation=g["kf_pose_t"]),
                  intrinsics=CameraIntrinsics(fx=20.0, fy=21.0, cx=6.0, cy=5.0, width=12, height=9,
                                              near=0.1, far=60.0),
                  rgb=g["kf_rgb"], depth=g["kf_depth"], last_loss=0.25, usage_remaining=3)
    data = diskformat.pack_keyframe(kf)
    assert data == g["keyframe"].tobytes()
    back = diskformat.unpack_keyframe(data)
    assert np.array_equal(back.rgb, kf.rgb) and np.array_equal(back.depth, kf.depth)


def test_corrupt_files_rejected():
    data = diskformat.pack_chunk(7, [Gaussian(position=[1, 2, 3])])
    with pytest.raises(CorruptChunk):
        diskformat.unpack_chunk(b"BAD!" + data[4:])
    with pytest.raises(CorruptChunk):
        diskformat.unpack_chunk(data[:-3])
    with pytest.raises(CorruptChunk):
        diskformat.read_chunk_header(data[:10])


def test_persistence_roundtrip_randomized():
    """test_acceptance.py criterion 9 (chunk half) on this codec."""
    rng = np.random.default_rng(109)
    for _ in range(200):
        gs = []
        for _ in range(int(rng.integers(0, 6))):
            opt = rng.bytes(int(rng.integers(1, 24))) if rng.random() < 0.5 else b""
            gs.append(diskformat.storage_canonical(Gaussian(
                position=rng.uniform(-500, 500, size=3), rotation=quat_normalize(rng.normal(size=4)),
                scale=rng.uniform(0.01, 2.0, size=3), opacity=float(rng.uniform(0, 1)),
                sh=rng.normal(size=48), opt_state=opt)))
        cid = int(rng.integers(0, 2**63))
        out_id, out = diskformat.unpack_chunk(diskformat.pack_chunk(cid, gs))
        assert out_id == cid and len(out) == len(gs)
        for a, b in zip(out, gs):
            assert np.array_equal(a.position, b.position) and np.array_equal(a.sh, b.sh)
            assert a.opacity == b.opacity and a.opt_state == b.opt_state


def test_metrics_row_format():
    from paper_2511_23030_b200.mapping import METRICS_HEADER, FrameMetrics
    assert METRICS_HEADER.count(",") == 11
    row = FrameMetrics(1, 2, 3, 4, 5, 6, 7, 8, 9, 10, None, 0.125).csv_row()
    assert row == "1,2,3,4,5,6,7,8,9,10,,0.125"


def test_synthetic_workloads_are_canonical():
    from paper_2511_23030_b200.synthetic import room_poses, room_scene
    s = room_scene(20000, seed=3)
    for a in (s.positions, s.rotations, s.scales, s.opacities, s.sh):
        assert np.array_equal(a, a.astype(np.float32).astype(np.float64))
    assert np.abs(np.linalg.norm(s.rotations, axis=1) - 1).max() <= 1e-6
    ids = grid.encode_positions(s.positions, 1.0)
    assert len(np.unique(ids)) == 128        # the 8x8x2 chunk grid
    assert len(room_poses(16)) == 16


def test_select_keyframe_fast_path_equals_generator_path():
    """select_keyframe with the precomputed uniform (plain-Python pairwise sum,
    cumsum, searchsorted) picks what NumPy's Generator.choice picks, for
    candidate lists below and above NumPy's 8-element pairwise block."""
    rng = np.random.default_rng(11)
    for trial in range(400):
        k = int(rng.integers(1, 40))
        pos = rng.uniform(-1, 1, (k, 3))
        ia = select.KeyframeIndex(config=select.SelectConfig(grid_resolution_m=1e6))
        ib = select.KeyframeIndex(config=select.SelectConfig(grid_resolution_m=1e6))
        for i in range(k):
            ia.add(i, pos[i])
            ib.add(i, pos[i])
        for i in range(k):
            loss = float(rng.uniform(0, 3) * (rng.random() > 0.2))
            select.record_loss(i, loss, ia)
            select.record_loss(i, loss, ib)
        seed = int(rng.integers(0, 2**63))
        a = select.select_keyframe(list(range(k)), ia, seed)
        b = select.select_keyframe(list(range(k)), ib, seed, uniform=select.draw_uniform(seed))
        assert a == b, trial


def test_visibility_cache_fast_scan_equals_vectorised_scan():
    """VisibilityCache.query's plain-float newest-first scan returns the same
    entry (result, hit flag, LRU order) as the vectorised prefilter it replaced
    (the reference's most-recent-match scan, culling.py:213-229)."""
    from paper_2511_23030_b200.core import CameraIntrinsics, Pose, quat_normalize
    from paper_2511_23030_b200.culling import ChunkExtent, CullConfig, VisibilityCache, _CacheEntry
    from paper_2511_23030_b200.grid import ChunkCoord

    class Old(VisibilityCache):   # the replaced implementation
        def query(self, pose, intr, extent, existing, generation, s, candidates=None):
            if self._entries:
                tr = np.array([e.translation for e in self._entries])
                d = np.sqrt(((tr - pose.translation) ** 2).sum(axis=1))
                for i in np.flatnonzero(d < self.cfg.pose_quantum_m * (1 + 1e-9) + 1e-300)[::-1]:
                    e = self._entries[int(i)]
                    if self._match(e, pose, intr, generation, s):
                        self._entries.append(self._entries.pop(int(i)))
                        return set(e.result), True
            res = frozenset({len(self._entries)})   # a marker per miss
            self._entries.append(_CacheEntry(pose.translation.copy(), pose.rotation.copy(), intr, s,
                                             generation, res, tuple(float(v) for v in pose.translation)))
            if len(self._entries) > self.cfg.cache_capacity:
                del self._entries[: len(self._entries) - self.cfg.cache_capacity]
            return set(res), False

    import paper_2511_23030_b200.culling as C
    rng = np.random.default_rng(3)
    intr = CameraIntrinsics(fx=100.0, fy=100.0, cx=50.0, cy=40.0, width=100, height=80, near=0.05)
    ext = ChunkExtent(ChunkCoord(0, 0, 0), ChunkCoord(1, 1, 1))
    cfg = CullConfig()
    new, old = VisibilityCache(cfg), Old(cfg)
    base = [rng.uniform(-1, 1, 3) for _ in range(20)]
    real = C.visible_chunks
    try:   # the same marker results on both sides
        for t in range(3000):
            b = base[int(rng.integers(0, len(base)))]
            tr = b + rng.normal(scale=cfg.pose_quantum_m * rng.choice([0.2, 0.7, 1.0, 3.0]), size=3)
            q = quat_normalize(np.array([1.0, 0, 0, 0]) + rng.normal(scale=1e-3, size=4))
            pose = Pose(rotation=q, translation=tr)
            gen = int(rng.integers(0, 2))
            C.visible_chunks = lambda *a, **k: {len(new._entries)}
            ra = new.query(pose, intr, ext, lambda c: True, gen, 10.0, candidates=lambda: [])
            rb = old.query(pose, intr, ext, lambda c: True, gen, 10.0)
            assert ra == rb, t
            assert [e.t3 for e in new._entries] == [e.t3 for e in old._entries]
    finally:
        C.visible_chunks = real


def test_slab_allocator_cap_and_compaction_cpu():
    """GaussianSlab's allocator on CPU tensors: first fit with coalescing;
    under a row cap (C5's HBM cap) it never grows, packs live segments to the
    front when no extent fits (rows and Adam state move with them, spare rows
    get zero gradients) and raises HbmCapExceeded past the cap."""
    import torch

    from paper_2511_23030_b200.errors import HbmCapExceeded
    from paper_2511_23030_b200.slab import GaussianSlab
    slab = GaussianSlab(0, device="cpu", max_rows=1000)
    assert slab.capacity == 1000 and slab.hbm_bytes() == 1000 * GaussianSlab.bytes_per_gaussian()
    segs = {}

    def pack_hook():
        keys = sorted(segs)
        new = slab.pack([segs[k] for k in keys])
        for k, off in zip(keys, new):
            segs[k] = (off, segs[k][1], segs[k][2])
    slab.compact_hook = pack_hook
    for k, size in enumerate([300, 200, 300, 150]):
        off = slab.alloc(size)
        segs[k] = (off, size, size - 10)
        slab.params[off:off + size - 10, 0] = float(k)
        slab.adam_m[off:off + size - 10, 14] = float(10 + k)
    slab.free(segs[0][0], 300)   # holes: [0, 300) and [950, 1000)
    slab.free(segs[2][0], 300)   # [500, 800) coalesces nothing with [0, 300)
    del segs[0], segs[2]
    assert slab.used() == 350
    off = slab.alloc(500)   # no 500-row extent: compaction, then fits
    assert slab.compactions == 1 and slab.capacity == 1000
    assert sorted(v[0] for v in segs.values()) == [0, 200]   # packed in offset order
    for k, (o, size, used) in segs.items():
        assert torch.all(slab.params[o:o + used, 0] == float(k))
        assert torch.all(slab.adam_m[o:o + used, 14] == float(10 + k))
        assert torch.all(slab.grads[o + used:o + size] == 0)
    assert off == 350
    with pytest.raises(HbmCapExceeded):
        slab.alloc(200)   # 150 rows free: past the cap
    uncapped = GaussianSlab(1024, device="cpu")
    a = uncapped.alloc(1000)
    b = uncapped.alloc(1000)   # grows
    assert uncapped.capacity >= 2000 and b == a + 1000


def test_sample_pixels_host_draw_matches_reference(golden):
    """sample.py:87-101: the draw stays on the host (NumPy Generator.choice
    without replacement); fed the reference's probability map it returns the
    reference's pixels (tests/golden/sample.npz)."""
    from paper_2511_23030_b200.sample import log_kernel, sample_pixels
    g = golden("sample.npz")
    for n, seed in ((50, 3), (500, 4), (5000, 5)):
        draw = np.array(sample_pixels(g["ps"], n, seed), dtype=np.int64).reshape(-1, 2)
        assert np.array_equal(draw, g[f"draw_{n}_{seed}"])
    assert sample_pixels(np.zeros((4, 5)), 10, 1) == []
    k = log_kernel(1.0, 2)
    assert k.shape == (5, 5) and abs(k.sum()) < 1e-12 and k[2, 2] == k.min()
