"""C5 stress run: a 100M-splat map under a hard 8 GB HBM cap.

    python tools/stress_bench.py [--n 100000000] [--length 5000] [--cap-gb 8]

The C4 street corridor generator at five times the length (5 km, 20k splats
per metre, s = 10 m chunks, KITTI 1241x376).  The map is built slice by slice
(each slice inserted, flushed to disk and evicted, so HBM never holds more
than the cap), then a car drives the whole corridor: a keyframe every
`--spacing` metres joins the map and is followed by `--steps` mapping
iterations (keyframe draw, visibility, residency, fwd + loss + bwd + Adam),
with write-behind eviction and prefetch.  The slab is allocated once at the
cap (StoreConfig.hbm_cap_bytes) and never grows; fragmentation is handled by
compaction.  A compute-only rate is measured first on the corridor's first
`--resident-keyframes` keyframes with their chunks all resident (no paging),
so overlap = streamed steps/s / resident steps/s.

Prints one JSON line (also written to --out when given).
"""

import argparse
import json
import shutil
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


class Slices:
    """The corridor generated slice by slice (seeded per slice).  The ground
    truth ("perturbed") splats of the last two slices stay on the device as
    one x-sorted packed-param tensor, so a view's window is a row range."""

    def __init__(self, n, length, n_slices, device, seed=7):
        self.n, self.length, self.k = n, length, n_slices
        self.len_s = length / n_slices
        self.seed = seed
        self.device = device
        self.parts = []   # [(slice, x (host, sorted), packed params (device))]

    def scene(self, i):
        from paper_2511_23030_b200.synthetic import SceneData, corridor_scene
        s = corridor_scene(self.n // self.k, length=self.len_s, seed=self.seed + 1000 * i)
        pos = s.positions.copy()
        pos[:, 0] += i * self.len_s
        return SceneData(pos, s.rotations, s.scales, s.opacities, s.sh)

    def add_target(self, i, scene):
        import torch

        from paper_2511_23030_b200.renderloss import SceneArrays, pack_params
        from paper_2511_23030_b200.synthetic import perturbed
        t = perturbed(scene, 49 + i)
        o = np.argsort(t.positions[:, 0], kind="stable")
        sa = SceneArrays(t.positions[o], t.rotations[o], t.scales[o], t.opacities[o], t.sh0[o])
        self.parts = [p for p in self.parts if p[0] >= i - 1]
        self.parts.append((i, t.positions[o, 0].copy(), torch.from_numpy(pack_params(sa)).to(self.device)))
        self.x = np.concatenate([p[1] for p in self.parts])
        self.params = torch.cat([p[2] for p in self.parts])

    def near(self, x0, x1):
        a, b = np.searchsorted(self.x, [x0, x1])
        return self.params[a:b]


def gt_frame(params, pose, intr, eng):
    from paper_2511_23030_b200.renderloss import render_device
    rgb, depth, _ = render_device(params, None, params.shape[0], pose, intr, eng)
    return rgb.cpu().numpy(), depth.cpu().numpy()


def disk_bandwidth(root: Path, nbytes: int = 2 << 30) -> dict:
    """This box's disk, in the same job: sequential write with fsync, then a
    read with the page cache dropped for the file (posix_fadvise DONTNEED)."""
    import os
    path = root / "_bw.bin"
    buf = np.random.default_rng(0).integers(0, 255, 64 << 20, dtype=np.uint8).tobytes()
    t0 = time.perf_counter()
    with open(path, "wb", buffering=0) as f:
        for _ in range(nbytes // len(buf)):
            f.write(buf)
        os.fsync(f.fileno())
    w = time.perf_counter() - t0
    fd = os.open(path, os.O_RDONLY)
    os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
    os.close(fd)
    t0 = time.perf_counter()
    with open(path, "rb", buffering=0) as f:
        while f.read(64 << 20):
            pass
    r = time.perf_counter() - t0
    path.unlink()
    return {"write_gbs": nbytes / w / 1e9, "read_gbs": nbytes / r / 1e9, "bytes": nbytes}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--length", type=float, default=5000.0)
    ap.add_argument("--slices", type=int, default=20)
    ap.add_argument("--cap-gb", type=float, default=8.0)
    ap.add_argument("--pinned-gb", type=float, default=8.0, help="host staging (write-behind + prefetch)")
    ap.add_argument("--budget", type=int, default=0, help="Gaussian budget (default: 85%% of the cap's rows)")
    ap.add_argument("--spacing", type=float, default=2.0)
    ap.add_argument("--keyframes", type=int, default=0, help="limit (default: the whole corridor)")
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--resident-keyframes", type=int, default=0, help="limit (default: the same trajectory)")
    ap.add_argument("--max-distance", type=float, default=50.0)
    ap.add_argument("--out", default="")
    ap.add_argument("--profile", action="store_true", help="cProfile the streamed run (host hot spots)")
    args = ap.parse_args()
    import torch

    from paper_2511_23030_b200.core import Keyframe
    from paper_2511_23030_b200.culling import CullConfig
    from paper_2511_23030_b200.mapping import MappingEngine
    from paper_2511_23030_b200.renderloss import default_engine
    from paper_2511_23030_b200.slab import GaussianSlab
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    from paper_2511_23030_b200.synthetic import C4_INTR, corridor_poses

    device = torch.device("cuda")
    cap_bytes = int(args.cap_gb * (1 << 30))
    pool = min(6 << 30, cap_bytes // 8)   # the streamer's share of the cap (store.py)
    cap_rows = (cap_bytes - pool) // GaussianSlab.bytes_per_gaussian()
    budget = args.budget or int(0.85 * cap_rows)
    n_kf = int(args.length / args.spacing)
    if args.keyframes:
        n_kf = min(n_kf, args.keyframes)
    poses = corridor_poses(n_kf, spacing=args.spacing)
    root = Path(tempfile.mkdtemp(prefix="c5_"))
    t_build = time.perf_counter()
    store = ChunkStore(StoreConfig(disk_root=root, chunk_size_m=10.0, gaussian_budget=budget,
                                   keyframe_budget=400, io_ns_per_byte=1.0, hbm_cap_bytes=cap_bytes,
                                   pinned_pool_bytes=int(args.pinned_gb * (1 << 30))))
    sl = Slices(args.n, args.length, args.slices, device)
    frames = [None] * n_kf
    eng_r = default_engine(device)
    # the compute-only reference: the SAME scene and trajectory with every
    # chunk resident (uncapped store, 100M x 436 B = 44 GB of HBM)
    rroot = Path(tempfile.mkdtemp(prefix="c5_resident_"))
    rstore = ChunkStore(StoreConfig(disk_root=rroot, chunk_size_m=10.0, gaussian_budget=args.n + 1,
                                    keyframe_budget=400, io_ns_per_byte=1.0,
                                    slab_capacity=int(args.n * 1.02) + 4096))
    next_pose = 0
    for i in range(args.slices):
        sc = sl.scene(i)
        store.insert_arrays(sc.positions, sc.rotations, sc.scales, sc.opacities, sc.sh)
        store.flush()
        store.evict_lru(store.stats.active_gaussians, protected=set())
        store.flush()
        rstore.insert_arrays(sc.positions, sc.rotations, sc.scales, sc.opacities, sc.sh)
        sl.add_target(i, sc)
        del sc
        # GT of every pose whose view window lies in the generated slices
        covered = (i + 1) * sl.len_s
        while next_pose < n_kf:
            x = poses[next_pose].translation[0]
            if x + args.max_distance + 10.0 > covered and i + 1 < args.slices:
                break
            frames[next_pose] = gt_frame(sl.near(x - 2.0, x + args.max_distance + 10.0), poses[next_pose],
                                         C4_INTR, eng_r)
            next_pose += 1
    store.streamer.drain()
    del sl
    torch.cuda.empty_cache()
    build_s = time.perf_counter() - t_build
    disk_bytes = sum(p.stat().st_size for p in (root / "chunks").glob("*.dcg"))
    print(json.dumps({"built": True, "seconds": build_s, "chunks": len(store.known_chunk_ids()),
                      "disk_bytes": disk_bytes}), file=sys.stderr, flush=True)

    disk = disk_bandwidth(root)
    print(json.dumps({"disk": disk}), file=sys.stderr, flush=True)
    res = {}
    k_res = min(args.resident_keyframes, n_kf) if args.resident_keyframes else n_kf
    for mode, st, k in (("resident", rstore, k_res), ("streamed", store, n_kf)):
        eng = MappingEngine(st, C4_INTR, seed=7, cull=CullConfig(max_distance_m=args.max_distance))
        blocked = [0.0]
        ensure = st.ensure_resident

        def timed(ids, ensure=ensure, blocked=blocked):
            t = time.perf_counter()
            try:
                return ensure(ids)
            finally:
                blocked[0] += time.perf_counter() - t
        st.ensure_resident = timed
        st.streamer.warm()
        sstats0 = dict(st.streamer.stats)   # (the build phase's paging is not the run's)
        s0 = st.stats
        base = (s0.chunk_loads, s0.chunk_evictions, s0.chunk_writes, s0.bytes_read, s0.bytes_written,
                s0.keyframe_writes, s0.keyframe_loads)
        # the keyframes arrive as Keyframe objects (their 8-bit quantisation
        # is ingest, core.py:266, not mapping): built before the clock starts
        kfs = [Keyframe(id=i, pose=poses[i], intrinsics=C4_INTR, rgb=frames[i][0], depth=frames[i][1])
               for i in range(k)]
        torch.cuda.synchronize()
        prof = None
        if args.profile and mode == "streamed":
            import cProfile
            prof = cProfile.Profile()
            prof.enable()
        t0 = time.perf_counter()
        steps = 0
        add_s = 0.0
        for kf_i in range(k):
            pose = poses[kf_i]
            ta = time.perf_counter()
            eng.add_keyframe(kfs[kf_i])   # the engine prefetches itself (look-ahead); no harness prefetch
            add_s += time.perf_counter() - ta
            for s in range(args.steps):
                eng.optimization_step(kf_i, s)
                steps += 1
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if prof is not None:
            import io
            import pstats
            prof.disable()
            buf = io.StringIO()
            pstats.Stats(prof, stream=buf).sort_stats("tottime").print_stats(30)
            print(buf.getvalue(), file=sys.stderr)
        s1 = st.stats
        now = (s1.chunk_loads, s1.chunk_evictions, s1.chunk_writes, s1.bytes_read, s1.bytes_written,
               s1.keyframe_writes, s1.keyframe_loads)
        d = [a - b for a, b in zip(now, base)]
        res[mode] = {"keyframes": k, "steps": steps, "seconds": dt, "steps_per_s": steps / dt,
                     "chunk_loads": d[0], "chunk_evictions": d[1], "chunk_writes": d[2],
                     "bytes_read": d[3], "bytes_written": d[4], "keyframe_writes": d[5],
                     "keyframe_loads": d[6], "ensure_resident_s": blocked[0], "add_keyframe_s": add_s,
                     "mean_visible": eng.counter_gaussians / max(eng.counter_steps, 1),
                     "slab_bytes": st.slab.hbm_bytes(), "slab_compactions": st.slab.compactions,
                     "hbm_bytes_store": st.slab.hbm_bytes() + st.streamer.device_bytes,
                     "graph_replays": eng.counter_replays, "eager_steps": eng.counter_eager}
        if st.streamer is not None:
            res[mode].update({f"streamer_{a}": (b - sstats0.get(a, 0) if a != "arena_s" else b)
                              for a, b in st.streamer.stats.items()})
        print(json.dumps({mode: res[mode]}), file=sys.stderr, flush=True)
        st.flush()
        st.streamer.drain()
        del eng
    rs_, ss_ = res["resident"], res["streamed"]
    floor_s = max(rs_["seconds"] * ss_["steps"] / max(rs_["steps"], 1),
                  ss_["bytes_written"] / disk["write_gbs"] / 1e9)
    line = {"disk": disk, "disk_floor_seconds": floor_s, "vs_disk_floor": floor_s / ss_["seconds"],
            "workload": f"C5: {args.n} splats over {args.length:.0f} m (s = 10 m), 1241x376, HBM cap "
                        f"{args.cap_gb:g} GB ({cap_rows} slab rows), budget {budget}, {n_kf} keyframes x "
                        f"{args.steps} steps",
            "build_seconds": build_s, "disk_bytes": disk_bytes, "runs": res,
            "overlap": res["streamed"]["steps_per_s"] / res["resident"]["steps_per_s"],
            "cap_held": res["streamed"]["hbm_bytes_store"] <= cap_bytes}
    print(json.dumps(line))
    if args.out:
        Path(args.out).write_text(json.dumps(line) + "\n")
    shutil.rmtree(root, ignore_errors=True)
    shutil.rmtree(rroot, ignore_errors=True)


if __name__ == "__main__":
    main()
