"""ChunkStore (HBM slab + GPU codec) against the reference store's own trace.

tests/golden/store_trace.json was recorded by running the reference
ChunkStore (store.py) through 120 seeded insert / ensure_resident /
evict_lru / mark_chunk_mutated operations: every LoadReport, eviction list,
stats vector (loads, evictions, writes, io_ns, bytes), resident set and the
final flushed map must be identical here.
"""
import json

import numpy as np
import pytest

from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _stats(st):
    s = st.stats
    return [s.active_gaussians, s.active_chunks, s.chunk_loads, s.chunk_evictions, s.chunk_writes,
            s.io_nanos, s.bytes_read, s.bytes_written, s.budget_overshoot, st.generation,
            s.total_gaussians_ever]


def test_store_policy_trace_matches_reference(cuda, tmp_path):
    from paper_2511_23030_b200.core import Gaussian
    from paper_2511_23030_b200.errors import InsufficientEvictable
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    trace = json.loads((GOLDEN / "store_trace.json").read_text())
    st = ChunkStore(StoreConfig(disk_root=tmp_path, chunk_size_m=10.0, gaussian_budget=60,
                                keyframe_budget=4, io_ns_per_byte=1.0))
    for k, op in enumerate(trace["ops"]):
        if op["op"] == "insert":
            gs = [Gaussian(position=p, opacity=o, scale=s, rotation=r, sh=sh)
                  for p, o, s, r, sh in zip(op["positions"], op["opacity"], op["scale"],
                                            op["rotation"], op["sh"])]
            assert st.insert_gaussians(gs) == op["ret"], k
        elif op["op"] == "ensure":
            rep = st.ensure_resident([int(i) for i in op["ids"]])
            assert (rep.loaded, rep.already_resident) == (op["loaded"], op["already"]), k
            assert [str(e) for e in rep.evicted] == op["evicted"], k
        elif op["op"] == "evict":
            prot = {int(p) for p in op["protected"]}
            if op["error"]:
                with pytest.raises(InsufficientEvictable):
                    st.evict_lru(op["required"], protected=prot)
            else:
                assert [str(e) for e in st.evict_lru(op["required"], protected=prot)] == op["evicted"], k
        else:
            st.mark_chunk_mutated(int(op["id"]))
        assert _stats(st) == op["stats"], (k, op["op"])
        assert [str(r) for r in sorted(st.resident_chunk_ids())] == [str(r) for r in op["resident"]], k
    st.flush()
    assert _stats(st) == trace["final_stats"]
    content = []
    for cid, gs in st.iter_map():
        for g in gs:
            content.append([str(cid)] + g.position.tolist() + [g.opacity])
    assert content == trace["final_map"]


@pytest.mark.parametrize("write_behind", [False, True])
def test_policy_trace_sync_and_write_behind(cuda, tmp_path, write_behind):
    """Same trace with synchronous and write-behind eviction: identical policy,
    stats and flushed files (the streamer never changes a decision)."""
    from paper_2511_23030_b200.core import Gaussian
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    trace = json.loads((GOLDEN / "store_trace.json").read_text())
    st = ChunkStore(StoreConfig(disk_root=tmp_path, chunk_size_m=10.0, gaussian_budget=60,
                                io_ns_per_byte=1.0, write_behind=write_behind))
    for op in trace["ops"]:
        if op["op"] == "insert":
            st.insert_gaussians([Gaussian(position=p, opacity=o, scale=s, rotation=r, sh=sh)
                                 for p, o, s, r, sh in zip(op["positions"], op["opacity"], op["scale"],
                                                           op["rotation"], op["sh"])])
        elif op["op"] == "ensure":
            st.ensure_resident([int(i) for i in op["ids"]])
        elif op["op"] == "evict" and not op["error"]:
            st.evict_lru(op["required"], protected={int(p) for p in op["protected"]})
        elif op["op"] == "mutate":
            st.mark_chunk_mutated(int(op["id"]))
        assert _stats(st) == op["stats"]
    st.flush()
    assert _stats(st) == trace["final_stats"]
    if write_behind:
        assert st.streamer.stats["async_writes"] > 0


def test_evict_reload_bit_exact_with_adam_state(cuda, tmp_path):
    """Chunks written with the 120-byte Adam tail reload params + moments exactly."""
    import torch

    from paper_2511_23030_b200.core import Gaussian, quat_normalize
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    rng = np.random.default_rng(4)
    st = ChunkStore(StoreConfig(disk_root=tmp_path, chunk_size_m=10.0, gaussian_budget=10_000,
                                io_ns_per_byte=1.0))
    gs = [Gaussian(position=rng.uniform(-4, 4, 3), rotation=quat_normalize(rng.normal(size=4)),
                   scale=rng.uniform(0.01, 0.2, 3), opacity=float(rng.uniform(0, 1)),
                   sh=rng.normal(size=48)) for _ in range(300)]
    st.insert_gaussians(gs)
    (cid,) = st.resident_chunk_ids()
    ch = st.chunk(cid)
    rows = slice(ch.offset, ch.offset + ch.count)
    st.slab.adam_m[rows] = torch.randn_like(st.slab.adam_m[rows])
    st.slab.adam_m[rows, 14] = 5.0
    st.slab.adam_v[rows] = torch.rand_like(st.slab.adam_v[rows])
    st.slab.adam_v[rows, 14:] = 0.0
    st.slab.adam_m[rows, 15] = 0.0
    st.mark_trained([cid])
    before = [t[rows].clone() for t in (st.slab.params, st.slab.adam_m, st.slab.adam_v, st.slab.sh_rest)]
    assert st.evict_lru(1) == [cid]
    st.ensure_resident([cid])
    ch = st.chunk(cid)
    rows = slice(ch.offset, ch.offset + ch.count)
    after = [t[rows] for t in (st.slab.params, st.slab.adam_m, st.slab.adam_v, st.slab.sh_rest)]
    for a, b in zip(before, after):
        assert torch.equal(a, b)
    st.streamer.drain()   # the write-behind file lands asynchronously
    data = (tmp_path / "chunks" / f"{cid:016x}.dcg").read_bytes()
    assert len(data) == 32 + 300 * 360


def test_foreign_opt_state_roundtrips(cuda, tmp_path):
    """Opaque opt_state payloads of untrained splats survive paging (store.py contract)."""
    from paper_2511_23030_b200.core import Gaussian
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    st = ChunkStore(StoreConfig(disk_root=tmp_path, gaussian_budget=100, io_ns_per_byte=1.0))
    gs = [Gaussian(position=[1.0 + i * 0.01, 2.0, 3.0], opt_state=bytes([i, i + 1, i + 2]) * (i % 3))
          for i in range(5)]
    st.insert_gaussians(gs)
    (cid,) = st.resident_chunk_ids()
    st.evict_lru(1)
    st.ensure_resident([cid])
    assert [g.opt_state for g in st.chunk(cid).gaussians] == [g.opt_state for g in gs]


def test_corrupt_chunk_detected_on_device(cuda, tmp_path):
    from paper_2511_23030_b200.core import Gaussian
    from paper_2511_23030_b200.errors import CorruptChunk
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    st = ChunkStore(StoreConfig(disk_root=tmp_path, gaussian_budget=100, io_ns_per_byte=1.0))
    st.insert_gaussians([Gaussian(position=[1.0, 2.0, 3.0]) for _ in range(3)])
    st.flush()
    (cid,) = st.resident_chunk_ids()
    st.evict_lru(1)
    p = tmp_path / "chunks" / f"{cid:016x}.dcg"
    data = bytearray(p.read_bytes())
    data[32 + 40:32 + 44] = np.float32(-1.0).tobytes()   # opacity of record 0 -> -1
    p.write_bytes(bytes(data))
    used = st.slab.used()
    with pytest.raises(CorruptChunk):
        st.ensure_resident([cid])
    assert st.slab.used() == used   # the rows reserved for the corrupt chunk were released
    assert cid not in st.resident_chunk_ids()


def test_write_behind_failure_keeps_data_and_retries(cuda, tmp_path, monkeypatch):
    """A write-behind that fails (ENOSPC) must not lose the chunk: the error
    surfaces at the next paging call, a reload is served from the kept packed
    bytes (not from the stale file), and the next flush writes the file."""
    import builtins
    import errno

    import torch

    from paper_2511_23030_b200 import streamer as S
    from paper_2511_23030_b200.core import Gaussian
    from paper_2511_23030_b200.errors import IoFailure
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    st = ChunkStore(StoreConfig(disk_root=tmp_path, chunk_size_m=10.0, gaussian_budget=100, io_ns_per_byte=1.0))
    st.insert_gaussians([Gaussian(position=[1.0 + 0.1 * i, 2.0, 3.0]) for i in range(5)])
    st.insert_gaussians([Gaussian(position=[31.0, 2.0 + 0.1 * i, 3.0]) for i in range(4)])
    st.flush()
    a = min(st.resident_chunk_ids())
    ch = st.chunk(a)
    st.slab.params[ch.offset:ch.offset + ch.count, 0] += 0.5   # new content, chunk dirty
    st.mark_chunk_mutated(a)
    want = st.slab.params[ch.offset:ch.offset + ch.count].clone()
    path = tmp_path / "chunks" / f"{a:016x}.dcg"
    stale = path.read_bytes()
    fail = {"n": 1}

    def fake_open(p, *args, **kw):
        if fail["n"] and str(p).startswith(str(path)):
            fail["n"] -= 1
            raise OSError(errno.ENOSPC, "No space left on device")
        return builtins.open(p, *args, **kw)
    monkeypatch.setattr(S, "open", fake_open, raising=False)
    st.evict_lru(ch.count, protected=set(st.resident_chunk_ids()) - {a})
    st.streamer._queue.join()   # the write-behind ran (and failed)
    assert path.read_bytes() == stale
    with pytest.raises(IoFailure):   # surfaces at the next paging operation
        st.ensure_resident([a])
    st.ensure_resident([a])          # served from the kept packed bytes
    ch = st.chunk(a)
    assert torch.equal(st.slab.params[ch.offset:ch.offset + ch.count], want)
    st.evict_lru(ch.count, protected=set(st.resident_chunk_ids()) - {a})
    st.flush()                       # the retried / newer write lands
    assert path.read_bytes() != stale
    st2 = ChunkStore(StoreConfig(disk_root=tmp_path, chunk_size_m=10.0, gaussian_budget=100, io_ns_per_byte=1.0))
    st2.ensure_resident([a])
    c2 = st2.chunk(a)
    assert torch.equal(st2.slab.params[c2.offset:c2.offset + c2.count], want)


def test_device_encode_positions_bit_exact(cuda, golden):
    import torch

    from paper_2511_23030_b200 import _lib
    g = golden("grid.npz")
    lib = _lib.load()
    for k in range(3):
        pos = g[f"s{k}_positions"]
        rec = np.zeros((len(pos), 16), np.float32)
        rec[:, :3] = pos
        t = torch.as_tensor(rec, device="cuda")
        ids = torch.empty(len(pos), dtype=torch.int64, device="cuda")
        err = torch.empty(1, dtype=torch.int64, device="cuda")
        _lib.check(lib.sm_encode_positions(_lib.ptr(t), len(pos), float(g[f"s{k}_size"]), _lib.ptr(ids),
                                           _lib.ptr(err), _lib.stream_handle()))
        assert int(err.item()) == -1
        assert np.array_equal(ids.cpu().numpy().view(np.uint64), g[f"s{k}_ids"])


def test_visible_chunks_bit_exact(cuda, golden):
    """K1 over the chunk table == the reference's visible_chunks sets (culling.py:134)."""
    from paper_2511_23030_b200.core import CameraIntrinsics, Pose
    from paper_2511_23030_b200.culling import ChunkExtent, CullConfig, visible_chunks
    from paper_2511_23030_b200.grid import ChunkCoord, encode_id
    g = golden("grid.npz")
    it = g["intr"]
    intr = CameraIntrinsics(fx=it[0], fy=it[1], cx=it[2], cy=it[3], near=it[4], far=it[5],
                            width=int(it[6]), height=int(it[7]))
    coords = g["coords"]
    ext = ChunkExtent(ChunkCoord(*map(int, coords.min(0))), ChunkCoord(*map(int, coords.max(0))))
    cfg = CullConfig(max_distance_m=float(g["max_distance"]))
    for t in range(int(g["vis_count"])):
        occ = {encode_id(ChunkCoord(*map(int, c))) for c in coords[g[f"v{t}_occ"]]}
        pose = Pose(rotation=g[f"v{t}_pose_q"], translation=g[f"v{t}_pose_t"])
        got = visible_chunks(pose, intr, ext, occ.__contains__, cfg, 10.0)
        assert sorted(got) == g[f"v{t}_visible"].tolist(), t


def test_streamer_device_reload_paths_bit_exact(cuda, tmp_path):
    """Write-behind eviction, then reloads served from every tier -- a pending
    write (device buffer), the HBM victim cache, the prefetch tier and the disk
    -- bring back exactly the rows (params, SH rest, Adam moments) that left."""
    import torch

    from paper_2511_23030_b200.core import Gaussian, quat_normalize
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    rng = np.random.default_rng(8)
    st = ChunkStore(StoreConfig(disk_root=tmp_path, chunk_size_m=10.0, gaussian_budget=10_000,
                                io_ns_per_byte=1.0, write_behind=True))
    gs = []
    for cx in range(4):   # four chunks of 500
        for _ in range(500):
            gs.append(Gaussian(position=[cx * 10.0 + rng.uniform(-4, 4), rng.uniform(-4, 4), rng.uniform(-4, 4)],
                               rotation=quat_normalize(rng.normal(size=4)), scale=rng.uniform(0.01, 0.2, 3),
                               opacity=float(rng.uniform(0, 1)), sh=rng.normal(size=48)))
    st.insert_gaussians(gs)
    ids = sorted(st.resident_chunk_ids())
    expect = {}
    for cid in ids:   # train-like edits + Adam state, then remember the rows
        ch = st.chunk(cid)
        rows = slice(ch.offset, ch.offset + ch.count)
        st.slab.params[rows, 0:3] += torch.randn_like(st.slab.params[rows, 0:3]) * 1e-3
        st.slab.adam_m[rows, :14] = torch.randn_like(st.slab.adam_m[rows, :14])
        st.slab.adam_m[rows, 14] = 3.0
        st.slab.adam_v[rows, :14] = torch.rand_like(st.slab.adam_v[rows, :14])
        st.mark_trained([cid])
        expect[cid] = [t[rows].clone() for t in (st.slab.params, st.slab.adam_m, st.slab.adam_v, st.slab.sh_rest)]

    def check(cid):
        ch = st.chunk(cid)
        rows = slice(ch.offset, ch.offset + ch.count)
        got = [t[rows] for t in (st.slab.params, st.slab.adam_m, st.slab.adam_v, st.slab.sh_rest)]
        for a, b in zip(expect[cid], got):
            assert torch.equal(a, b), cid

    st.evict_lru(st.stats.active_gaussians)         # all four out, writes pending
    st.ensure_resident([ids[0]])                    # pending or victim hit
    check(ids[0])
    st.streamer.drain()                             # writes landed: victim tier
    st.ensure_resident([ids[1]])
    check(ids[1])
    st.streamer.victim_limit = 0                    # no victims for what is evicted next
    st.streamer._victims.clear()
    st.prefetch([ids[2]])                           # prefetch tier
    st.ensure_resident([ids[2]])
    check(ids[2])
    st.ensure_resident([ids[3]])                    # plain disk read
    check(ids[3])
    s = st.streamer.stats
    assert s["victim_hits"] + s["pending_hits"] >= 2 and s["prefetch_hits"] >= 1, s
    st.flush()


def test_hbm_cap_compaction_bit_exact(cuda, tmp_path):
    """A slab under a hard HBM cap (C5's 8 GB, scaled down) never grows:
    when no free extent fits a chunk it packs the resident segments to the
    front (compaction).  Against an uncapped store driven by the same
    operations (inserts in slices with flush + evict, paging, training-like
    updates with Adam state): identical policy stats, identical resident rows
    after every step and byte-identical files; the cap holds and a working
    set that cannot fit raises HbmCapExceeded."""
    import torch

    from paper_2511_23030_b200.errors import HbmCapExceeded
    from paper_2511_23030_b200.slab import GaussianSlab
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    from paper_2511_23030_b200.workloads import c1_scene
    from paper_2511_23030_b200.grid import encode_positions
    scene = c1_scene(20_000)
    # the map is built slice by slice like C5: whole chunks per slice (<= 2500 rows)
    cid = encode_positions(scene.positions, 5.0)
    order = np.argsort(cid, kind="stable")
    starts = np.r_[0, np.flatnonzero(np.diff(cid[order])) + 1, len(order)]
    slices, a = [], 0
    for b0, b1 in zip(starts[:-1], starts[1:]):
        if b1 - a > 2_500:
            slices.append(order[a:b0])
            a = b0
    slices.append(order[a:])
    # the reference policy loads a working set before it evicts down to the
    # budget: the cap must hold budget + working set (+ segment slack)
    cap_rows = 5_200
    # the cap also covers the streamer's device buffers (1/8 of it, store.py)
    cap_bytes = -(-cap_rows * GaussianSlab.bytes_per_gaussian() * 8 // 7)
    cap_rows = (cap_bytes - cap_bytes // 8) // GaussianSlab.bytes_per_gaussian()
    stores = []
    for name, cap in (("free", None), ("capped", cap_bytes)):
        st = ChunkStore(StoreConfig(disk_root=tmp_path / name, chunk_size_m=5.0, gaussian_budget=2_500,
                                    io_ns_per_byte=1.0, hbm_cap_bytes=cap))
        for idx in slices:
            st.insert_arrays(scene.positions[idx], scene.rotations[idx], scene.scales[idx],
                             scene.opacities[idx], scene.sh[idx])
            st.flush()
            st.evict_lru(st.stats.active_gaussians, protected=set())
        stores.append(st)
    free, capped = stores
    assert capped.slab.capacity == cap_rows
    ids = sorted(free.known_chunk_ids())
    rng = np.random.default_rng(8)
    for step in range(120):
        want = []
        for c in rng.permutation(ids):   # a random working set that fits the budget
            if sum(free.chunk_gaussian_count(x) for x in want) + free.chunk_gaussian_count(c) <= 2_000:
                want.append(int(c))
            if len(want) >= rng.integers(2, 7):
                break
        reps = [st.ensure_resident(want) for st in stores]
        assert reps[0] == reps[1]
        for st in stores:   # "training": rows and Adam state change, chunks go dirty
            for c in want:
                ch = st.chunk(c)
                rows = slice(ch.offset, ch.offset + ch.count)
                st.slab.params[rows, 0:3] += 1e-3 * (step + 1)
                st.slab.adam_m[rows, 0:14] += 1.0
                st.slab.adam_m[rows, 14] += 1.0
                st.slab.adam_v[rows, 0:14] += 0.5
            st.mark_trained(want)
        assert _stats(free) == _stats(capped)
        assert free.resident_chunk_ids() == capped.resident_chunk_ids()
        for c in want:
            a, b = free.chunk(c), capped.chunk(c)
            for name in ("params", "adam_m", "adam_v", "sh_rest"):
                ta, tb = getattr(free.slab, name), getattr(capped.slab, name)
                assert torch.equal(ta[a.offset:a.offset + a.count], tb[b.offset:b.offset + b.count]), (step, c)
        assert capped.slab.capacity == cap_rows   # never grew
    assert capped.slab.compactions > 0
    for st in stores:
        st.flush()
        st.streamer.drain()
    for c in ids:
        name = f"{c:016x}.dcg"
        assert (tmp_path / "free" / "chunks" / name).read_bytes() == \
               (tmp_path / "capped" / "chunks" / name).read_bytes()
    with pytest.raises(HbmCapExceeded):   # a working set larger than the cap
        capped.ensure_resident(ids)


def test_streamer_under_pool_pressure_matches_sync(cuda, tmp_path):
    """Staging pools of two buffers each: evictions wait for landed writes
    (pinned) or take victim-cache buffers back (device) instead of
    allocating; the paging sequence still ends in byte-identical files and
    identical resident rows compared with synchronous I/O."""
    import torch

    from paper_2511_23030_b200.core import Gaussian, quat_normalize
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    rng = np.random.default_rng(21)
    gs = []
    for cx in range(8):   # eight chunks of 300
        for _ in range(300):
            gs.append(Gaussian(position=[cx * 10.0 + rng.uniform(-4, 4), rng.uniform(-4, 4), rng.uniform(-4, 4)],
                               rotation=quat_normalize(rng.normal(size=4)), scale=rng.uniform(0.01, 0.2, 3),
                               opacity=float(rng.uniform(0, 1)), sh=rng.normal(size=48)))
    stores = []
    for name, wb in (("sync", False), ("tight", True)):
        st = ChunkStore(StoreConfig(disk_root=tmp_path / name, chunk_size_m=10.0, gaussian_budget=900,
                                    io_ns_per_byte=1.0, write_behind=wb))
        if wb:
            st.streamer.PINNED_SLOTS = 2
            st.streamer.DEVICE_SLOTS = 2
            st.streamer.victim_limit = 1 << 20
        st.insert_gaussians(gs)
        stores.append(st)
    ids = sorted(stores[0].known_chunk_ids())
    order = np.random.default_rng(3).integers(0, len(ids), size=(40, 3))
    for step, pick in enumerate(order):
        want = sorted({ids[int(k)] for k in pick})
        for st in stores:
            st.ensure_resident(want)
            for c in want:   # training-like edit, chunk goes dirty
                ch = st.chunk(c)
                st.slab.params[ch.offset:ch.offset + ch.count, 0] += 1e-3 * (step + 1)
            st.mark_trained(want)
        assert _stats(stores[0]) == _stats(stores[1])
        for c in want:
            a, b = stores[0].chunk(c), stores[1].chunk(c)
            assert torch.equal(stores[0].slab.params[a.offset:a.offset + a.count],
                               stores[1].slab.params[b.offset:b.offset + b.count])
    for st in stores:
        st.flush()
    tight = stores[1].streamer.stats
    assert tight["async_writes"] > 0 and tight["alloc_pinned"] == 0 and tight["alloc_device"] == 0
    for c in ids:
        name = f"{c:016x}.dcg"
        assert (tmp_path / "sync" / "chunks" / name).read_bytes() == (tmp_path / "tight" / "chunks" / name).read_bytes()


def test_streamer_prefetch_tier_and_oversize_buffers(cuda, tmp_path):
    """The speculative tier under pressure: prefetches of chunks that are
    never loaded are dropped oldest-first (FIFO) or taken back by real I/O,
    chunks bigger than a pool slot get a buffer without waiting, and the
    paging sequence still matches synchronous I/O row for row and, after
    flush, byte for byte."""
    import torch

    from paper_2511_23030_b200.core import Gaussian, quat_normalize
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    rng = np.random.default_rng(31)
    gs = []
    for cx in range(12):   # twelve chunks, every third ten times denser
        for _ in range(3000 if cx % 3 == 0 else 300):
            gs.append(Gaussian(position=[cx * 10.0 + rng.uniform(-4, 4), rng.uniform(-4, 4), rng.uniform(-4, 4)],
                               rotation=quat_normalize(rng.normal(size=4)), scale=rng.uniform(0.01, 0.2, 3),
                               opacity=float(rng.uniform(0, 1)), sh=rng.normal(size=48)))
    stores = []
    for name, wb in (("sync", False), ("spec", True)):
        st = ChunkStore(StoreConfig(disk_root=tmp_path / name, chunk_size_m=10.0, gaussian_budget=4000,
                                    io_ns_per_byte=1.0, write_behind=wb))
        if wb:   # small slots: the dense chunks (~0.9 MB) exceed two of them
            sm = st.streamer
            sm.PINNED_SLOT_BYTES = 256 << 10
            sm.PINNED_SLOTS = 12
            sm.DEVICE_SLOTS = 6
            sm._largest = {True: 2 * sm.PINNED_SLOT_BYTES, False: 2 * sm.PINNED_SLOT_BYTES}
        st.insert_gaussians(gs)
        stores.append(st)
    ids = sorted(stores[0].known_chunk_ids())
    order = np.random.default_rng(4).integers(0, len(ids), size=(40, 4))
    for step, pick in enumerate(order):
        want = sorted({ids[int(k)] for k in pick[:2]})
        stores[1].prefetch([ids[int(k)] for k in pick[2:]])   # speculation, often never used
        for st in stores:
            st.ensure_resident(want)
            for c in want:
                ch = st.chunk(c)
                st.slab.params[ch.offset:ch.offset + ch.count, 0] += 1e-3 * (step + 1)
            st.mark_trained(want)
        assert _stats(stores[0]) == _stats(stores[1])
        for c in want:
            a, b = stores[0].chunk(c), stores[1].chunk(c)
            assert torch.equal(stores[0].slab.params[a.offset:a.offset + a.count],
                               stores[1].slab.params[b.offset:b.offset + b.count])
    stats = stores[1].streamer.stats
    assert stats["prefetch_issued"] > 0 and stats["prefetch_dropped"] > 0, stats
    assert stats["alloc_pinned"] + stats["alloc_device"] > 0, stats   # oversize chunks: no waiting
    assert stats["pool_wait_s"] < 1.0, stats
    for st in stores:
        st.flush()
    for c in ids:
        name = f"{c:016x}.dcg"
        assert (tmp_path / "sync" / "chunks" / name).read_bytes() == (tmp_path / "spec" / "chunks" / name).read_bytes()


def test_capped_write_behind_backlog_in_pinned_memory(cuda, tmp_path):
    """Under a hard HBM cap the eviction D2H is issued at eviction and the
    device buffer goes back to the small pool once it completed; a chunk
    reloaded while its write is still queued is served from the pinned copy.
    With the writers held back (every write pending), the paging sequence
    still matches synchronous I/O row for row and, once the writers run,
    byte for byte on disk."""
    import threading

    import torch

    from paper_2511_23030_b200.core import Gaussian, quat_normalize
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    rng = np.random.default_rng(23)
    gs = []
    for cx in range(8):   # eight chunks of 300
        for _ in range(300):
            gs.append(Gaussian(position=[cx * 10.0 + rng.uniform(-4, 4), rng.uniform(-4, 4), rng.uniform(-4, 4)],
                               rotation=quat_normalize(rng.normal(size=4)), scale=rng.uniform(0.01, 0.2, 3),
                               opacity=float(rng.uniform(0, 1)), sh=rng.normal(size=48)))
    sync = ChunkStore(StoreConfig(disk_root=tmp_path / "sync", chunk_size_m=10.0, gaussian_budget=900,
                                  io_ns_per_byte=1.0, write_behind=False))
    capped = ChunkStore(StoreConfig(disk_root=tmp_path / "capped", chunk_size_m=10.0, gaussian_budget=900,
                                    io_ns_per_byte=1.0, hbm_cap_bytes=1 << 30))
    gate = threading.Event()
    orig = capped.streamer._write_one

    def held(pw):
        gate.wait()
        return orig(pw)
    capped.streamer._write_one = held
    stores = (sync, capped)
    try:
        for st in stores:
            st.insert_gaussians(gs)
        ids = sorted(sync.known_chunk_ids())
        order = np.random.default_rng(5).integers(0, len(ids), size=(30, 3))
        for step, pick in enumerate(order):
            want = sorted({ids[int(k)] for k in pick})
            for st in stores:
                st.ensure_resident(want)
                for c in want:
                    ch = st.chunk(c)
                    st.slab.params[ch.offset:ch.offset + ch.count, 0] += 1e-3 * (step + 1)
                st.mark_trained(want)
            assert _stats(sync) == _stats(capped)
            for c in want:
                a, b = sync.chunk(c), capped.chunk(c)
                assert torch.equal(sync.slab.params[a.offset:a.offset + a.count],
                                   capped.slab.params[b.offset:b.offset + b.count])
        stats = capped.streamer.stats
        assert stats["pending_pinned_hits"] > 0, stats
    finally:
        gate.set()
    for st in stores:
        st.flush()
    for c in ids:
        name = f"{c:016x}.dcg"
        assert (tmp_path / "sync" / "chunks" / name).read_bytes() == \
               (tmp_path / "capped" / "chunks" / name).read_bytes()


def test_write_through_views_match_reference_bytes(cuda, tmp_path):
    """chunk.gaussians / gather_visible are live views (store.py:361-379): the
    reference's refine_reset loop (loopclose.py:236-242), nudge-style in-place
    sh0 / opacity edits (sim.py:309-317) and scale edits through GaussianRefs,
    interleaved with paging, flush byte-identical files
    (tests/golden/view_edits.json was recorded on the reference store)."""
    import hashlib

    from paper_2511_23030_b200.core import Gaussian
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    rec = json.loads((GOLDEN / "view_edits.json").read_text())
    st = ChunkStore(StoreConfig(disk_root=tmp_path, chunk_size_m=10.0, gaussian_budget=70,
                                keyframe_budget=4, io_ns_per_byte=1.0))
    for batch in rec["inserts"]:
        st.insert_gaussians([Gaussian(position=g["position"], opacity=g["opacity"], scale=g["scale"],
                                      rotation=g["rotation"], sh=g["sh"], opt_state=bytes.fromhex(g["opt"]))
                             for g in batch])
    for op in rec["ops"]:
        if op["op"] == "ensure":
            st.ensure_resident([int(i) for i in op["ids"]])
            continue
        cid = int(op["id"])
        if op["op"] == "reset":
            for g in st.chunk(cid).gaussians:
                g.opacity = op["opacity"]
                g.opt_state = b""
            st.mark_chunk_mutated(cid)
        elif op["op"] == "nudge":
            for e in op["edits"]:
                g = st.chunk(cid).gaussians[e["index"]]
                g.sh[[0, 16, 32]] = e["sh0"]
                if e["opacity"] is not None:
                    g.opacity = e["opacity"]
            st.mark_chunk_mutated(cid)
        else:
            refs = st.gather_visible([cid])
            for k in op["picks"]:
                g = refs[k].gaussian
                g.scale[:] = np.float32(g.scale * 1.25).astype(np.float64)
    st.flush()
    got = {p.name: hashlib.sha256(p.read_bytes()).hexdigest()
           for p in sorted((tmp_path / "chunks").glob("*.dcg"))}
    assert got == rec["files"]


def test_opt_state_reset_gives_fresh_adam(cuda, tmp_path):
    """opt_state = b"" through a view resets the row's Adam state (the
    loopclose.py:241 contract): a trained chunk's reset rows get zero moments
    and step 0 and are written with opt_len 0, untouched rows keep their
    Adam tail; a view whose rows moved on (training) fails loudly."""
    from paper_2511_23030_b200 import diskformat
    from paper_2511_23030_b200.errors import NotResident
    from paper_2511_23030_b200.workloads import build_c1
    eng = build_c1(n=4000, keyframes=3, budget=100_000, store_dir=tmp_path)
    for s in range(4):
        eng.optimization_step(0, s)
    st = eng.store
    cid = max((c for c in st.resident_chunk_ids() if st.chunk(c).trained), key=lambda c: len(st.chunk(c)))
    ch = st.chunk(cid)
    views = ch.gaussians
    assert all(len(g.opt_state) == diskformat.ADAM_TAIL for g in views)
    reset = set(range(0, len(views), 2))
    for i in reset:
        views[i].opt_state = b""
    st.mark_chunk_mutated(cid)
    lo = ch.offset
    m = st.slab.adam_m[lo:lo + len(ch)].cpu().numpy()
    assert np.all(m[sorted(reset)] == 0.0) and np.all(m[1::2, 14] > 0)
    st.flush()
    _, gs = diskformat.unpack_chunk((tmp_path / "chunks" / f"{cid:016x}.dcg").read_bytes())
    assert [len(g.opt_state) for g in gs] == [0 if i in reset else diskformat.ADAM_TAIL for i in range(len(gs))]
    st.mark_trained([cid])   # the device rows moved on (what a training step does)
    with pytest.raises(NotResident):
        views[1].opacity = 0.5


def test_keyframe_tier_trace_matches_reference(cuda, tmp_path):
    """Keyframe tier (store.py:427-489) against the reference's own trace
    (tests/golden/keyframe_trace.json): add / get / dirty / pose update /
    flush under a budget of 3 -- LRU order, loads, evictions, write-backs,
    io_ns and bytes after every op, and the flushed .dkf files byte for byte."""
    import hashlib

    from paper_2511_23030_b200.core import CameraIntrinsics, Keyframe, Pose
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    rec = json.loads((GOLDEN / "keyframe_trace.json").read_text())
    intr = CameraIntrinsics(fx=10.0, fy=10.0, cx=4.0, cy=3.0, width=8, height=6, near=0.1, far=50.0)
    st = ChunkStore(StoreConfig(disk_root=tmp_path, keyframe_budget=3, io_ns_per_byte=1.0))
    for k, op in enumerate(rec["ops"]):
        if op["op"] == "add":
            st.keyframe_add(Keyframe(id=op["id"], pose=Pose(rotation=op["q"], translation=op["t"]), intrinsics=intr,
                                     rgb=np.array(op["rgb"]), depth=np.array(op["depth"], dtype=np.float32),
                                     last_loss=op["loss"], usage_remaining=op["usage"]))
        elif op["op"] == "get":
            st.keyframe_get(op["id"])
        elif op["op"] == "dirty":
            st.mark_keyframe_dirty(op["id"])
        elif op["op"] == "pose":
            st.update_keyframe_pose(op["id"], Pose(rotation=op["q"], translation=op["t"]))
        else:
            st.flush()
        s = st.stats
        assert list(st._keyframes) == op["resident"], k
        assert [s.keyframe_loads, s.keyframe_evictions, s.keyframe_writes, s.io_nanos, s.bytes_read,
                s.bytes_written, s.active_keyframes] == op["stats"], (k, op["op"])
    st.flush()
    got = {p.name: hashlib.sha256(p.read_bytes()).hexdigest() for p in sorted((tmp_path / "keyframes").glob("*.dkf"))}
    assert got == rec["files"]


def test_keyframe_device_pack_byte_identical(cuda, tmp_path):
    """The .dkf of an evicted keyframe assembled on the device from the HBM
    keyframe tier (sm_keyframe_pack) equals diskformat.pack_keyframe, and
    the write-behind path the store takes with it produces that file."""
    from paper_2511_23030_b200 import diskformat
    from paper_2511_23030_b200.workloads import build_c1
    eng = build_c1(n=4000, keyframes=6, budget=100_000, store_dir=tmp_path / "s", keyframe_budget=3)
    for s in range(6):
        eng.optimization_step(0, s)
    st = eng.store
    kid = sorted(eng.device_keyframe_ids())[0]
    kf = st.keyframe_get(kid)
    kf.last_loss = 0.25
    out = tmp_path / "probe.dkf"
    assert eng._pack_device_keyframe(kid, kf, out)
    st.streamer.drain()
    assert out.read_bytes() == diskformat.pack_keyframe(kf)
    writes0 = st.stats.keyframe_writes
    for k in sorted(st.known_keyframe_ids()):   # cycle the tier: device-packed write-backs
        st.keyframe_get(k)
        st.mark_keyframe_dirty(k)
        eng._device_keyframe(st.keyframe_get(k))
    st.flush()
    assert st.stats.keyframe_writes > writes0
    for p in sorted((tmp_path / "s" / "keyframes").glob("*.dkf")):
        k2 = diskformat.unpack_keyframe(p.read_bytes())
        assert p.read_bytes() == diskformat.pack_keyframe(k2)
