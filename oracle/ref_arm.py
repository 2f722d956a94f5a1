"""CPU arms of bench.py (BENCH / TEST INFRASTRUCTURE ONLY -- never imported by
the product package).

Two CPU timings of the C2 mapping loop, on the box's host cores:

* ``OracleMappingLoop`` -- the like-for-like arm.  The reference's own host
  policy, imported unmodified from ``baseline/_ref/splatmap`` (a ``pip
  --target`` install of /root/reference; select.py candidate set and
  loss-weighted draw with sim._derive_seed seeds, culling.VisibilityCache /
  visible_chunks), drives the same sequence the GPU arm runs -- one training
  iteration per keyframe (the GPU arm's graph warm-up), W warm-up steps, K
  timed steps -- and the device work of a step (render, loss + gradient,
  backward, Adam over the active set in sorted-chunk-id order, sim.py:236-253)
  is the fp64 oracle (oracle/render_oracle.c or_train_step).  The reference
  itself has no backward or Adam (pkg/README.md:125-129), so that part is the
  restatement; everything else is the reference's code.
* ``reference_replay_leg`` -- context: the unmodified reference
  ``sim._Replay.optimization_step`` (sim.py:319-370: cull, page, SoA build,
  render_arrays, total_loss, nudge) on the same C2 scene, its chunks written
  as reference .dcg files (diskformat.py:51-66 layout) and paged in by the
  reference ChunkStore.
"""

from __future__ import annotations

import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

from oracle import oracle as O

ROOT = Path(__file__).resolve().parents[1]


def load_reference():
    """The unmodified reference package from baseline/_ref (+ the scikit-image
    shim restating structural_similarity: scikit-image is absent offline)."""
    for p in (ROOT / "tests" / "golden" / "shim", ROOT / "baseline" / "_ref"):
        if str(p) not in sys.path:
            sys.path.insert(0, str(p))
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_ref_"))
    import splatmap  # noqa: F401
    from splatmap import core, culling, grid, select, sim, store
    return dict(core=core, culling=culling, grid=grid, select=select, sim=sim, store=store)


class OracleMappingLoop:
    """The C2 mapping loop on the CPU: reference policy + fp64 oracle step."""

    def __init__(self, scene, target, poses, intr, chunk_size=1.0, max_distance=200.0, seed=7,
                 threads=None, lr=None, betas=(0.9, 0.999), eps=1e-15, min_scale=1e-5,
                 weights=(0.2, 0.5)):
        ref = load_reference()
        self.ref = ref
        self.intr = intr
        self.seed = seed
        self.threads = threads or os.cpu_count() or 1
        self.lr = lr if lr is not None else [1e-4] * 3 + [1e-3] * 4 + [5e-5] * 3 + [1e-2] + [2.5e-3] * 3
        self.betas, self.eps, self.min_scale, self.weights = betas, eps, min_scale, weights
        self.state = O.TrainState(scene.positions, scene.rotations, scene.scales, scene.opacities, scene.sh0)
        # chunk membership (grid.encode_positions) in sorted-chunk-id order
        ids = O.chunk_ids(scene.positions, chunk_size)
        order = np.argsort(ids, kind="stable")
        sids = ids[order]
        cuts = np.flatnonzero(np.diff(sids)) + 1
        self.members = {int(sids[a]): order[a:b] for a, b in zip(np.r_[0, cuts], np.r_[cuts, len(ids)])}
        coords = [ref["grid"].decode_id(c) for c in self.members]
        lo = ref["grid"].ChunkCoord(min(c.cx for c in coords), min(c.cy for c in coords), min(c.cz for c in coords))
        hi = ref["grid"].ChunkCoord(max(c.cx for c in coords), max(c.cy for c in coords), max(c.cz for c in coords))
        self.extent = ref["culling"].ChunkExtent(lo, hi)
        self.chunk_size = chunk_size
        self.cache = ref["culling"].VisibilityCache(cfg=ref["culling"].CullConfig(max_distance_m=max_distance))
        self.index = ref["select"].KeyframeIndex(config=ref["select"].SelectConfig())
        self.poses = list(poses)
        self.gt = []
        for k, pose in enumerate(self.poses):
            rgb, depth, _ = O.render_arrays(target.positions, target.rotations, target.scales, target.opacities,
                                            target.sh0, pose.rotation, pose.translation, intr.fx, intr.fy,
                                            intr.cx, intr.cy, intr.near, intr.width, intr.height,
                                            threads=self.threads)
            # Keyframe quantisation (core.py:262-267): k/255 in float32
            q = (np.round(np.clip(rgb, 0.0, 1.0) * 255.0).astype(np.float32) / np.float32(255.0)).astype(np.float64)
            self.gt.append((q, depth.astype(np.float32).astype(np.float64)))
            self.index.add(k, np.asarray(pose.translation, dtype=np.float64),
                           usage_remaining=self.index.config.initial_usage)
        self.latest = len(self.poses) - 1
        self.step_counter = 0
        self.selected: list[int] = []
        self.n_active: list[int] = []

    def _subset(self, pose) -> np.ndarray:
        vis, _ = self.cache.query(pose, self.intr, self.extent, lambda c: c in self.members, 0, self.chunk_size)
        ids = sorted(vis)
        return np.concatenate([self.members[c] for c in ids]) if ids else np.zeros(0, dtype=np.int64)

    def train(self, kid: int, threads=None) -> float:
        """One mapping iteration on keyframe kid's active set; returns the loss."""
        pose = self.poses[kid]
        sub = self._subset(pose)
        self.n_active.append(len(sub))
        gt, gd = self.gt[kid]
        return self.state.step(pose.rotation, pose.translation, self.intr, gt, gd, self.weights[0],
                               self.weights[1], self.lr, self.betas[0], self.betas[1], self.eps,
                               self.min_scale, threads=threads or self.threads, subset=sub)

    def warm(self) -> None:
        """The GPU arm's graph warm-up: one iteration per keyframe, sorted ids."""
        for kid in range(len(self.poses)):
            self.train(kid)

    def step(self, threads=None) -> float:
        """sim._Replay.optimization_step's policy with the oracle as the device."""
        sel, sim = self.ref["select"], self.ref["sim"]
        try:
            cands = sel.candidate_set(self.index.position_of(self.latest), self.index)
        except Exception:   # EmptyCandidates
            cands = [self.latest]
        kid = sel.select_keyframe(cands, self.index, sim._derive_seed(self.seed, 2, self.step_counter))
        loss = self.train(kid, threads)
        sel.record_loss(kid, loss, self.index)
        self.selected.append(int(kid))
        self.step_counter += 1
        return loss


def _write_reference_chunks(scene, chunk_size: float, root: Path) -> None:
    """The scene as reference .dcg files (diskformat.py:51-66: header <4sIQQQ,
    records <3f4f3ff48fI, opt_len 0), one per chunk, in the store's path
    layout (store.py:130-131)."""
    rec_t = np.dtype([("pos", "<f4", 3), ("rot", "<f4", 4), ("scale", "<f4", 3), ("op", "<f4"),
                      ("sh", "<f4", 48), ("opt", "<u4")])
    ids = O.chunk_ids(scene.positions, chunk_size)
    order = np.argsort(ids, kind="stable")
    sids = ids[order]
    cuts = np.flatnonzero(np.diff(sids)) + 1
    (root / "chunks").mkdir(parents=True, exist_ok=True)
    for a, b in zip(np.r_[0, cuts], np.r_[cuts, len(ids)]):
        idx = order[a:b]
        rec = np.zeros(len(idx), dtype=rec_t)
        rec["pos"], rec["rot"], rec["scale"] = scene.positions[idx], scene.rotations[idx], scene.scales[idx]
        rec["op"], rec["sh"] = scene.opacities[idx], scene.sh[idx]
        cid = int(sids[a])
        head = np.zeros(1, dtype=[("m", "S4"), ("v", "<u4"), ("id", "<u8"), ("n", "<u8"), ("r", "<u8")])
        head["m"], head["v"], head["id"], head["n"] = b"DCG1", 1, cid, len(idx)
        (root / "chunks" / f"{cid:016x}.dcg").write_bytes(head.tobytes() + rec.tobytes())


def reference_replay_leg(scene, target, poses, intr, chunk_size=1.0, max_distance=200.0,
                         steps=3, warmup=1, budget=1_500_000, gts=None):
    """Time the unmodified reference _Replay.optimization_step (single
    process; its numba compositor is serial) on the C2 scene."""
    ref = load_reference()
    sim, store_m, core = ref["sim"], ref["store"], ref["core"]
    d = Path(tempfile.mkdtemp(prefix="ref_replay_"))
    cfg = sim.ReplayConfig(trajectory=d / "traj.txt", images_dir=d / "img", depth_dir=d / "depth",
                           out=d / "metrics.csv", store_dir=d / "store", chunk_size=chunk_size,
                           gaussian_budget=budget, keyframe_budget=400, max_distance=max_distance, seed=7)
    rep = sim._Replay(cfg, core.CameraIntrinsics(fx=intr.fx, fy=intr.fy, cx=intr.cx, cy=intr.cy,
                                                   width=intr.width, height=intr.height, near=intr.near))
    _write_reference_chunks(scene, chunk_size, cfg.store_dir)
    rep.store = store_m.ChunkStore(store_m.StoreConfig(disk_root=cfg.store_dir, chunk_size_m=chunk_size,
                                                       gaussian_budget=budget, keyframe_budget=400,
                                                       io_ns_per_byte=1.0))
    for k, pose in enumerate(poses):
        if gts is not None:
            rgb, depth = gts[k]
        else:
            rgb, depth, _ = O.render_arrays(target.positions, target.rotations, target.scales,
                                            target.opacities, target.sh0, pose.rotation, pose.translation,
                                            intr.fx, intr.fy, intr.cx, intr.cy, intr.near, intr.width,
                                            intr.height)
        kf = core.Keyframe(id=k, pose=core.Pose(rotation=pose.rotation, translation=pose.translation),
                           intrinsics=rep.intr, rgb=np.clip(rgb, 0, 1), depth=depth.astype(np.float32),
                           usage_remaining=rep.select_cfg.initial_usage)
        rep.store.keyframe_add(kf)
        rep.index.add(k, kf.position, usage_remaining=rep.select_cfg.initial_usage)
        rep.latest_kf = k
    times, active = [], []
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        row = rep.optimization_step(0, s)
        dt = time.perf_counter() - t0
        if s >= warmup:
            times.append(dt)
            active.append(row.active_gaussians)
    per = sum(times) / len(times)
    return {"value": 1.0 / per, "unit": "it/s", "ms_per_step": per * 1e3, "steps": steps, "warmup": warmup,
            "cores": 1, "kind": "reference",
            "sample": (f"unmodified reference sim._Replay.optimization_step (baseline/_ref/splatmap: cull, page "
                       f"from .dcg, SoA build, numba render_arrays, total_loss, nudge; forward only) on the C2 "
                       f"1M room, 640x480, {steps} steps after {warmup} warm-up, ~{int(np.mean(active))} "
                       f"resident Gaussians; serial compositor")}
