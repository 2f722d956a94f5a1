"""Out-of-core mapping run (C4-lite): is chunk streaming hidden behind rendering?

    python tools/stream_bench.py [--n 4000000] [--keyframes 100] [--steps 8]

A car drives a 200 m street corridor (C4 density: 20k splats per metre,
s = 10 m chunks, KITTI 1241x376); a keyframe every 2 m joins the map and is
followed by `--steps` mapping iterations (keyframe draw, visibility,
residency, fwd + loss + bwd + Adam).  With a 1.5M-splat HBM budget the store
pages chunks in ahead of the car and evicts (writes back) the ones behind it.
Three runs of the identical trajectory:

* resident  -- budget >= n: no paging at all (the compute-only reference),
* sync      -- budget 1.5M, blocking reads and write-back,
* streamed  -- budget 1.5M, write-behind eviction (copy stream + writer
  thread); the engine's own look-ahead prefetch (the newest keyframe's and
  the next draw's candidate views' chunks, on reader threads) -- nothing is
  prefetched by this harness.

Prints one JSON line: steps/s of each run, paging volume, and
overlap = t_resident / t_streamed (1.0 = streaming fully hidden).
"""

import argparse
import json
import shutil
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def run(mode: str, scene, poses, frames, args, prof=None):
    import torch

    from paper_2511_23030_b200.core import Keyframe
    from paper_2511_23030_b200.culling import CullConfig
    from paper_2511_23030_b200.mapping import MappingEngine
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    from paper_2511_23030_b200.synthetic import C4_INTR
    root = Path(tempfile.mkdtemp(prefix=f"c4lite_{mode}_"))
    budget = len(scene) + 1 if mode == "resident" else args.budget
    store = ChunkStore(StoreConfig(disk_root=root, chunk_size_m=10.0, gaussian_budget=budget,
                                   keyframe_budget=400, io_ns_per_byte=1.0,
                                   write_behind=(mode == "streamed"), writer_threads=args.writers))
    store.insert_arrays(scene.positions, scene.rotations, scene.scales, scene.opacities, scene.sh)
    store.flush()
    if mode != "resident":   # cold start: the map is on disk, HBM empty
        store.evict_lru(store.stats.active_gaussians, protected=set())
        store.flush()
    blocked = [0.0]
    ensure = store.ensure_resident

    def timed_ensure(ids):
        t = time.perf_counter()
        try:
            return ensure(ids)
        finally:
            blocked[0] += time.perf_counter() - t
    store.ensure_resident = timed_ensure
    store.streamer.warm()   # staging pools are allocated once, at startup
    eng = MappingEngine(store, C4_INTR, seed=7, cull=CullConfig(max_distance_m=args.max_distance))
    eng.prefetch_lookahead = mode == "streamed"
    eng.use_graphs = not args.no_graphs
    st0 = store.stats
    loads0, ev0, wr0, rb0, wb0 = st0.chunk_loads, st0.chunk_evictions, st0.chunk_writes, st0.bytes_read, st0.bytes_written
    # keyframes arrive as Keyframe objects (their 8-bit quantisation is
    # ingest, core.py:266, not mapping): built before the clock starts
    kfs = [Keyframe(id=k, pose=pose, intrinsics=C4_INTR, rgb=rgb, depth=depth)
           for k, (pose, (rgb, depth)) in enumerate(zip(poses, frames))]
    torch.cuda.synchronize()
    if prof is not None:   # the timed loop only
        prof.enable()
    import gc
    gc_t = [0.0, 0, 0.0]   # total, collections, longest

    def gc_cb(phase, info, _t=[0.0]):
        if phase == "start":
            _t[0] = time.perf_counter()
        else:
            d = time.perf_counter() - _t[0]
            gc_t[0] += d
            gc_t[1] += 1
            gc_t[2] = max(gc_t[2], d)
    gc.callbacks.append(gc_cb)
    t0 = time.perf_counter()
    steps = 0
    step_t = []   # host wall time of every step (where streaming costs show up)
    eager_at = []
    add_t = 0.0
    for k, (pose, kf) in enumerate(zip(poses, kfs)):
        ta = time.perf_counter()
        eng.add_keyframe(kf)   # the engine itself prefetches (new keyframe, next draw's candidates)
        tb = time.perf_counter()
        add_t += tb - ta
        for s in range(args.steps):
            e0 = eng.counter_eager
            eng.optimization_step(k, s)
            eager_at.append(eng.counter_eager - e0)
            tc = time.perf_counter()
            step_t.append(tc - tb)
            tb = tc
            steps += 1
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if prof is not None:
        prof.disable()
    gc.callbacks.remove(gc_cb)
    import numpy as np
    st_ = np.sort(np.asarray(step_t))
    step_stats = {"add_keyframe_s": add_t, "step_ms_p50": 1e3 * float(np.median(st_)),
                  "step_ms_p90": 1e3 * float(st_[int(0.9 * len(st_))]),
                  "step_ms_p99": 1e3 * float(st_[int(0.99 * len(st_))]), "step_ms_max": 1e3 * float(st_[-1]),
                  "slowest_5pct_s": float(st_[int(0.95 * len(st_)):].sum()),
                  "slowest_steps": [(int(i), round(1e3 * step_t[i], 2), eager_at[i])
                                    for i in np.argsort(step_t)[::-1][:6]],
                  "gc_s": gc_t[0], "gc_collections": gc_t[1], "gc_longest_ms": 1e3 * gc_t[2]}
    st = store.stats
    out = {"mode": mode, "seconds": dt, "steps": steps, "steps_per_s": steps / dt,
           "chunk_loads": st.chunk_loads - loads0, "chunk_evictions": st.chunk_evictions - ev0,
           "chunk_writes": st.chunk_writes - wr0, "bytes_read": st.bytes_read - rb0,
           "bytes_written": st.bytes_written - wb0, "active_gaussians_end": st.active_gaussians,
           "mean_visible": eng.counter_gaussians / max(eng.counter_steps, 1),
           "ensure_resident_s": blocked[0], "graph_replays": eng.counter_replays,
           "eager_steps": eng.counter_eager, **step_stats,
           # the training itself must not depend on the paging: the (keyframe,
           # loss) sequence of every mode is compared in main()
           "trace": [(r.selected_kf, r.loss) for r in eng.rows]}
    if store.streamer is not None:
        out.update({k: v for k, v in store.streamer.stats.items()})
    store.flush()
    del eng, store
    torch.cuda.empty_cache()
    shutil.rmtree(root, ignore_errors=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4_000_000)
    ap.add_argument("--length", type=float, default=200.0)
    ap.add_argument("--keyframes", type=int, default=100)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--budget", type=int, default=1_500_000)
    ap.add_argument("--max-distance", type=float, default=50.0)
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--writers", type=int, default=4, help="write-behind threads")
    ap.add_argument("--modes", default="resident,sync,streamed")
    ap.add_argument("--profile", action="store_true", help="cProfile each run (host hot spots to stderr)")
    ap.add_argument("--repeat", type=int, default=1,
                    help="run the modes this many times, interleaved; each mode reports its median run")
    args = ap.parse_args()
    import torch

    from paper_2511_23030_b200.synthetic import C4_INTR, corridor_poses, corridor_scene, perturbed
    from paper_2511_23030_b200.workloads import _gt_frames
    scene = corridor_scene(args.n, length=args.length, seed=7)
    poses = corridor_poses(args.keyframes, spacing=args.length / args.keyframes)
    # ground truth: each keyframe renders the perturbed scene near it (the
    # renderer packs (tile, depth rank) into 32 bits: <= 2M splats per view)
    target = perturbed(scene, 49)
    frames = []
    for pose in poses:
        x = pose.translation[0]
        near = (target.positions[:, 0] > x - 2.0) & (target.positions[:, 0] < x + args.max_distance + 10.0)
        frames += _gt_frames(target.subset(near), [pose], C4_INTR, torch.device("cuda"))
    res = {}
    # warm-up (library init, kernels, allocator): a short resident run, discarded
    warm = argparse.Namespace(**{**vars(args), "steps": 2})
    run("resident", scene, poses[:5], frames[:5], warm)
    runs: dict[str, list] = {}
    for mode in [m for _ in range(args.repeat) for m in args.modes.split(",")]:
        pr = None
        if args.profile:
            import cProfile
            import io
            import pstats
            pr = cProfile.Profile()
        out = run(mode, scene, poses, frames, args, pr)
        runs.setdefault(mode, []).append(out)
        if args.profile:
            for key in ("tottime", "cumulative"):
                buf = io.StringIO()
                pstats.Stats(pr, stream=buf).sort_stats(key).print_stats(30)
                print(f"==== {mode} ({key})\n" + buf.getvalue(), file=sys.stderr)
        print(json.dumps({k: v for k, v in out.items() if k != "trace"}), file=sys.stderr, flush=True)
    for mode, rs in runs.items():
        rs = sorted(rs, key=lambda r: r["seconds"])
        res[mode] = rs[len(rs) // 2]
        res[mode]["seconds_all"] = [r["seconds"] for r in rs]
        if any(r["trace"] != rs[0]["trace"] for r in rs):
            res[mode]["repeat_diverged"] = True
    from stress_bench import disk_bandwidth
    bw_root = Path(tempfile.mkdtemp(prefix="c4_bw_"))
    disk = disk_bandwidth(bw_root)
    shutil.rmtree(bw_root, ignore_errors=True)
    name = "C4" if args.n >= 20_000_000 else "C4-lite"
    line = {"disk": disk, "workload": f"{name}: {args.n} splats over {args.length:.0f} m (s = 10 m), 1241x376, "
                        f"budget {args.budget}, {args.keyframes} keyframes x {args.steps} steps",
            "runs": res}
    if "resident" in res and "streamed" in res:
        line["overlap"] = res["resident"]["seconds"] / res["streamed"]["seconds"]
        # what the disk alone forces: every write-back has to reach it (reads
        # of recently written chunks may come from the page cache: not counted)
        floor = max(res["resident"]["seconds"], res["streamed"]["bytes_written"] / disk["write_gbs"] / 1e9)
        line["disk_floor_seconds"] = floor
        line["vs_disk_floor"] = floor / res["streamed"]["seconds"]
    traces = {m: r.pop("trace") for m, r in res.items()}
    base = next(iter(traces.values()))
    line["same_training"] = {m: t == base for m, t in traces.items()}
    for m, t in traces.items():
        if t != base:
            k = next(i for i, (a, b) in enumerate(zip(t, base)) if a != b)
            line.setdefault("first_divergence", {})[m] = [k, t[k], base[k]]
    if "resident" in res and "sync" in res:
        line["sync_vs_resident"] = res["resident"]["seconds"] / res["sync"]["seconds"]
    print(json.dumps(line))


if __name__ == "__main__":
    main()
