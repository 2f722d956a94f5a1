"""Generate golden fixtures by running the REFERENCE splatmap package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the read-only reference from /root/reference/pkg/src with the
test-only scikit-image shim in tests/golden/shim (scikit-image is absent and
not installable offline; the shim restates its structural_similarity).  The
fixtures it writes are small .npz / .json files committed next to this
script; nothing at test or bench time reads /root/reference.

Fixtures:
  render_small.npz  reference render_arrays outputs on seeded scenes
  render_fd.npz     central finite differences of the reference forward
                    (linear functional of rgb/depth/alpha and total_loss)
  loss.npz          reference total_loss / image_loss / ssim / depth_loss
  grid.npz          encode_positions, chunk coords, frustum planes, visible sets
  diskformat.npz    pack_chunk / pack_keyframe bytes
  store_trace.json  ChunkStore policy trace (loads, evictions, stats)
  sample.npz        log_norm / sampling_probability / sample_pixels / lift / ingest_keyframe
  keyframe_trace.json keyframe-tier LRU / write-back trace + .dkf hashes
  loopclose.json    run_correction (batch / sequential): reports, stats, flushed map
  view_edits.json   in-place edits through chunk.gaussians / gather_visible + flushed file hashes
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path(os.environ.get("SPLATMAP_REF_SRC", "/root/reference/pkg/src"))
sys.path.insert(0, str(HERE / "shim"))
sys.path.insert(0, str(REF_SRC))
os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))

import splatmap  # noqa: E402
from splatmap import core, culling, diskformat, grid, renderloss, store  # noqa: E402

SH_C0 = core.SH_C0


def _scene(rng, n, span=2.0, depth=(2.0, 8.0), scale=(0.05, 0.3)):
    """Seeded SoA scene shaped like test_renderloss.random_scene (fp32-canonical)."""
    pos = np.stack([rng.uniform(-span, span, n), rng.uniform(-span, span, n),
                    rng.uniform(*depth, n)], axis=1)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sc = rng.uniform(*scale, size=(n, 3))
    op = rng.uniform(0.3, 0.95, n)
    col = rng.uniform(0.05, 0.95, size=(n, 3))
    sh0 = (col - 0.5) / SH_C0
    f = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    return renderloss.SceneArrays(positions=f(pos), rotations=f(q), scales=f(sc),
                                  opacities=f(op), sh0=f(sh0))


def _pose(rng, jitter=0.2, rotate=False):
    rot = core.quat_normalize(rng.normal(size=4) * 0.05 + np.array([1.0, 0, 0, 0])) if rotate \
        else np.array([1.0, 0.0, 0.0, 0.0])
    return core.Pose(rotation=rot, translation=rng.normal(size=3) * jitter)


def make_render_small():
    rng = np.random.default_rng(2024)
    cases = []
    intr64 = core.CameraIntrinsics(fx=50.0, fy=50.0, cx=32.0, cy=32.0, width=64, height=64,
                                   near=0.2, far=100.0)
    for i in range(4):
        cases.append((_scene(rng, 150), _pose(rng, rotate=i % 2 == 1), intr64))
    # behind-near-plane and straddling Gaussians
    sc = _scene(rng, 120, depth=(-1.0, 4.0))
    cases.append((sc, core.Pose(), intr64))
    # large footprints that clamp at the borders, non-square, odd principal point
    intr_odd = core.CameraIntrinsics(fx=37.0, fy=41.0, cx=20.3, cy=15.7, width=48, height=33,
                                     near=0.1, far=50.0)
    cases.append((_scene(rng, 90, span=3.0, depth=(0.5, 3.0), scale=(0.1, 0.8)), _pose(rng), intr_odd))
    # C1-shaped mini: 2000 splats at 160x120
    intr_c1 = core.CameraIntrinsics(fx=120.0, fy=120.0, cx=80.0, cy=60.0, width=160, height=120,
                                    near=0.05, far=1000.0)
    cases.append((_scene(rng, 2000, span=4.0, depth=(1.0, 12.0), scale=(0.02, 0.25)),
                  _pose(rng, rotate=True), intr_c1))
    # single opaque on-axis Gaussian (test_renderloss known answer)
    one = renderloss.SceneArrays(positions=np.array([[0.0, 0.0, 2.0]]),
                                 rotations=np.array([[1.0, 0, 0, 0]]),
                                 scales=np.full((1, 3), 0.1), opacities=np.array([0.999]),
                                 sh0=((np.array([[0.9, 0.3, 0.6]]) - 0.5) / SH_C0))
    intr32 = core.CameraIntrinsics(fx=40.0, fy=40.0, cx=16.0, cy=16.0, width=32, height=32,
                                   near=0.1, far=200.0)
    cases.append((one, core.Pose(), intr32))
    out = {"count": len(cases)}
    for k, (sc, pose, intr) in enumerate(cases):
        fr = renderloss.render_arrays(sc, pose, intr)
        out[f"c{k}_positions"] = sc.positions
        out[f"c{k}_rotations"] = sc.rotations
        out[f"c{k}_scales"] = sc.scales
        out[f"c{k}_opacities"] = sc.opacities
        out[f"c{k}_sh0"] = sc.sh0
        out[f"c{k}_pose_q"] = pose.rotation
        out[f"c{k}_pose_t"] = pose.translation
        out[f"c{k}_intr"] = np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.near, intr.far,
                                      intr.width, intr.height], dtype=np.float64)
        out[f"c{k}_rgb"] = fr.rgb
        out[f"c{k}_depth"] = fr.depth
        out[f"c{k}_alpha"] = fr.alpha
    np.savez_compressed(HERE / "render_small.npz", **out)


def make_render_fd():
    """Central differences of the reference forward (fp64), h = 1e-6."""
    rng = np.random.default_rng(77)
    intr = core.CameraIntrinsics(fx=30.0, fy=30.0, cx=16.0, cy=16.0, width=32, height=32,
                                 near=0.2, far=100.0)
    sc = _scene(rng, 40, span=1.5, depth=(2.0, 5.0), scale=(0.08, 0.35))
    pose = _pose(rng, rotate=True)
    wr = rng.normal(size=(32, 32, 3))
    wd = rng.normal(size=(32, 32))
    wa = rng.normal(size=(32, 32))
    gt_rgb = np.round(rng.uniform(0, 1, size=(32, 32, 3)) * 255) / 255
    gt_depth = rng.uniform(1.0, 6.0, size=(32, 32)).astype(np.float32)
    gt_depth[rng.random((32, 32)) < 0.2] = 0.0
    kf = core.Keyframe(id=0, pose=pose, intrinsics=intr, rgb=gt_rgb, depth=gt_depth)
    w = renderloss.LossWeights()

    def lin(s):
        fr = renderloss.render_arrays(s, pose, intr)
        return float((fr.rgb * wr).sum() + (fr.depth * wd).sum() + (fr.alpha * wa).sum())

    def tl(s):
        return renderloss.total_loss(renderloss.render_arrays(s, pose, intr), kf, w)

    fields = ["positions", "rotations", "scales", "opacities", "sh0"]
    picks = rng.choice(len(sc.positions), size=12, replace=False)
    h = 1e-6
    res = {f"lin_{f}": [] for f in fields}
    res.update({f"loss_{f}": [] for f in fields})
    for i in picks:
        for f in fields:
            arr = getattr(sc, f)
            ncomp = 1 if arr.ndim == 1 else arr.shape[1]
            gl, gt = [], []
            for c in range(ncomp):
                vals = []
                for sgn in (1.0, -1.0):
                    s2 = renderloss.SceneArrays(**{k: getattr(sc, k).copy() for k in fields})
                    a2 = getattr(s2, f)
                    if a2.ndim == 1:
                        a2[i] += sgn * h
                    else:
                        a2[i, c] += sgn * h
                    vals.append((lin(s2), tl(s2)))
                gl.append((vals[0][0] - vals[1][0]) / (2 * h))
                gt.append((vals[0][1] - vals[1][1]) / (2 * h))
            res[f"lin_{f}"].append(gl)
            res[f"loss_{f}"].append(gt)
    fr = renderloss.render_arrays(sc, pose, intr)
    out = {k: np.array(v) for k, v in res.items()}
    out.update(picks=picks, positions=sc.positions, rotations=sc.rotations, scales=sc.scales,
               opacities=sc.opacities, sh0=sc.sh0, pose_q=pose.rotation, pose_t=pose.translation,
               intr=np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.near, intr.far, 32, 32.0]),
               w_rgb=wr, w_depth=wd, w_alpha=wa, gt_rgb=kf.rgb, gt_depth=kf.depth,
               loss=tl(sc), rgb=fr.rgb, depth=fr.depth, alpha=fr.alpha, h=h)
    np.savez_compressed(HERE / "render_fd.npz", **out)


def make_loss():
    rng = np.random.default_rng(3)
    out = {}
    shapes = [(16, 16), (24, 31), (48, 64), (120, 160)]
    for k, (h, w) in enumerate(shapes):
        rgb = rng.uniform(0, 1, size=(h, w, 3))
        if k == 3:
            rgb = np.clip(rgb * 0.3 + 0.5 + 0.2 * np.sin(np.arange(w) / 5.0)[None, :, None], 0, 1)
        depth = rng.uniform(0.5, 9.0, size=(h, w))
        kf = core.Keyframe(id=k, pose=core.Pose(),
                           intrinsics=core.CameraIntrinsics(fx=30.0, fy=30.0, cx=w / 2, cy=h / 2,
                                                            width=w, height=h),
                           rgb=rng.uniform(0, 1, size=(h, w, 3)),
                           depth=(rng.uniform(0.5, 9.0, size=(h, w))
                                  * (rng.random((h, w)) > 0.25)).astype(np.float32))
        fr = renderloss.RenderedFrame(rgb=rgb, depth=depth, alpha=np.ones((h, w)))
        out[f"c{k}_rgb"] = rgb
        out[f"c{k}_depth"] = depth
        out[f"c{k}_gt_rgb"] = kf.rgb
        out[f"c{k}_gt_depth"] = kf.depth
        for j, (ls, ld) in enumerate([(0.2, 0.5), (0.0, 0.0), (1.0, 2.0)]):
            out[f"c{k}_total_{j}"] = np.array(
                [ls, ld, renderloss.total_loss(fr, kf, renderloss.LossWeights(ls, ld))])
        out[f"c{k}_ssim"] = np.array(renderloss.ssim(rgb, kf.rgb))
        out[f"c{k}_depth_loss"] = np.array(renderloss.depth_loss(depth, kf.depth))
    out["count"] = len(shapes)
    np.savez_compressed(HERE / "loss.npz", **out)


def make_grid():
    rng = np.random.default_rng(5)
    out = {}
    for k, s in enumerate([10.0, 1.0, 0.37]):
        pos = rng.uniform(-1e3, 1e3, size=(2000, 3)) * (s / 10.0)
        # exact cell boundaries and negative-zero cases
        pos[:6] = np.array([[s / 2, -s / 2, 0.0], [-0.0, s * 1.5, -s * 1.5],
                            [s / 2 - 1e-12, s / 2 + 1e-12, -s / 2 + 1e-12],
                            [0.0, 0.0, 0.0], [1e-300, -1e-300, s], [-s, s * 2.5, -s * 2.5]])
        pos = pos.astype(np.float32).astype(np.float64)
        out[f"s{k}_size"] = np.array(s)
        out[f"s{k}_positions"] = pos
        out[f"s{k}_ids"] = grid.encode_positions(pos, s)
    # frustum planes + visibility sets over a 12^3 extent (criterion-2 style)
    intr = core.CameraIntrinsics(fx=50.0, fy=45.0, cx=31.0, cy=33.0, width=64, height=64,
                                 near=0.5, far=120.0)
    cfg = culling.CullConfig(max_distance_m=70.0)
    lo, hi = -6, 5
    ext = culling.ChunkExtent(grid.ChunkCoord(lo, lo, lo), grid.ChunkCoord(hi, hi, hi))
    coords = np.array([[x, y, z] for x in range(lo, hi + 1) for y in range(lo, hi + 1)
                       for z in range(lo, hi + 1)])
    vis = []
    for t in range(40):
        occ = rng.random(len(coords)) < 0.4
        ids = {grid.encode_id(grid.ChunkCoord(*map(int, c))) for c in coords[occ]}
        pose = core.Pose(rotation=core.quat_normalize(rng.normal(size=4)),
                         translation=rng.uniform(-40, 40, size=3))
        res = culling.visible_chunks(pose, intr, ext, ids.__contains__, cfg, 10.0)
        fr = culling.extract_frustum(pose, intr)
        out[f"v{t}_occ"] = occ
        out[f"v{t}_pose_q"] = pose.rotation
        out[f"v{t}_pose_t"] = pose.translation
        out[f"v{t}_planes"] = fr.planes
        out[f"v{t}_visible"] = np.array(sorted(res), dtype=np.uint64)
        vis.append(len(res))
    out["coords"] = coords
    out["vis_count"] = np.array(len(vis))
    out["intr"] = np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.near, intr.far, 64, 64.0])
    out["max_distance"] = np.array(cfg.max_distance_m)
    np.savez_compressed(HERE / "grid.npz", **out)


def make_diskformat():
    rng = np.random.default_rng(9)
    gs = []
    for i in range(7):
        gs.append(diskformat.storage_canonical(core.Gaussian(
            position=rng.uniform(-50, 50, size=3), rotation=core.quat_normalize(rng.normal(size=4)),
            scale=rng.uniform(0.01, 2.0, size=3), opacity=float(rng.uniform(0, 1)),
            sh=rng.normal(size=48), opt_state=b"")))
    plain = diskformat.pack_chunk(0x123456789A, gs)
    gs_opt = [g.copy() for g in gs]
    for i, g in enumerate(gs_opt):
        g.opt_state = bytes(rng.integers(0, 256, size=(i * 5) % 13, dtype=np.uint8))
    with_opt = diskformat.pack_chunk(0xABCDEF, gs_opt)
    kf = core.Keyframe(id=42, pose=core.Pose(rotation=core.quat_normalize(rng.normal(size=4)),
                                             translation=rng.normal(size=3)),
                       intrinsics=core.CameraIntrinsics(fx=20.0, fy=21.0, cx=6.0, cy=5.0,
                                                        width=12, height=9, near=0.1, far=60.0),
                       rgb=rng.random((9, 12, 3)),
                       depth=rng.uniform(0, 5, size=(9, 12)).astype(np.float32),
                       last_loss=0.25, usage_remaining=3)
    out = dict(
        chunk_plain=np.frombuffer(plain, dtype=np.uint8),
        chunk_opt=np.frombuffer(with_opt, dtype=np.uint8),
        keyframe=np.frombuffer(diskformat.pack_keyframe(kf), dtype=np.uint8),
        positions=np.array([g.position for g in gs]), rotations=np.array([g.rotation for g in gs]),
        scales=np.array([g.scale for g in gs]), opacities=np.array([g.opacity for g in gs]),
        sh=np.array([g.sh for g in gs]),
        opt_lens=np.array([len(g.opt_state) for g in gs_opt]),
        opt_blob=np.frombuffer(b"".join(g.opt_state for g in gs_opt), dtype=np.uint8),
        kf_rgb=kf.rgb, kf_depth=kf.depth, kf_pose_q=kf.pose.rotation, kf_pose_t=kf.pose.translation,
    )
    np.savez_compressed(HERE / "diskformat.npz", **out)


def make_store_trace():
    """Scripted ChunkStore workload; records every policy-visible outcome."""
    rng = np.random.default_rng(11)
    trace = {"ops": []}
    with tempfile.TemporaryDirectory() as d:
        st = store.ChunkStore(store.StoreConfig(disk_root=d, chunk_size_m=10.0,
                                                gaussian_budget=60, keyframe_budget=4,
                                                io_ns_per_byte=1.0))
        cells = [(x, y, 0) for x in range(-2, 3) for y in range(-1, 2)]

        def stats():
            s = st.stats
            return [s.active_gaussians, s.active_chunks, s.chunk_loads, s.chunk_evictions,
                    s.chunk_writes, s.io_nanos, s.bytes_read, s.bytes_written,
                    s.budget_overshoot, st.generation, s.total_gaussians_ever]

        for step in range(120):
            kind = rng.choice(["insert", "ensure", "evict", "mutate"], p=[0.35, 0.45, 0.1, 0.1])
            if kind == "insert":
                k = int(rng.integers(1, 18))
                pos = []
                for _ in range(k):
                    cx, cy, cz = cells[int(rng.integers(len(cells)))]
                    pos.append([cx * 10 + rng.uniform(-4.9, 4.9), cy * 10 + rng.uniform(-4.9, 4.9),
                                rng.uniform(-4.9, 4.9)])
                gs = [core.Gaussian(position=p, opacity=float(rng.uniform(0, 1)),
                                    scale=rng.uniform(0.01, 1, size=3),
                                    rotation=core.quat_normalize(rng.normal(size=4)),
                                    sh=rng.normal(size=48)) for p in pos]
                n = st.insert_gaussians(gs)
                trace["ops"].append({"op": "insert", "positions": np.array(pos).tolist(),
                                     "opacity": [g.opacity for g in gs],
                                     "scale": [g.scale.tolist() for g in gs],
                                     "rotation": [g.rotation.tolist() for g in gs],
                                     "sh": [g.sh.tolist() for g in gs],
                                     "ret": n, "stats": stats(),
                                     "resident": sorted(st.resident_chunk_ids())})
            elif kind == "ensure":
                k = int(rng.integers(1, 5))
                ids = sorted({grid.encode_id(grid.ChunkCoord(*cells[int(rng.integers(len(cells)))]))
                              for _ in range(k)})
                rep = st.ensure_resident(ids)
                trace["ops"].append({"op": "ensure", "ids": [str(i) for i in ids],
                                     "loaded": rep.loaded, "already": rep.already_resident,
                                     "evicted": [str(e) for e in rep.evicted], "stats": stats(),
                                     "resident": [str(r) for r in sorted(st.resident_chunk_ids())]})
            elif kind == "evict":
                res = sorted(st.resident_chunk_ids())
                prot = [c for c in res if rng.random() < 0.3]
                req = int(rng.integers(0, 40))
                try:
                    ev = st.evict_lru(req, protected=set(prot))
                    err = None
                except Exception as exc:  # InsufficientEvictable
                    ev, err = [], type(exc).__name__
                trace["ops"].append({"op": "evict", "required": req,
                                     "protected": [str(p) for p in prot],
                                     "evicted": [str(e) for e in ev], "error": err,
                                     "stats": stats(),
                                     "resident": [str(r) for r in sorted(st.resident_chunk_ids())]})
            else:
                res = sorted(st.resident_chunk_ids())
                if not res:
                    continue
                cid = res[int(rng.integers(len(res)))]
                st.mark_chunk_mutated(cid)
                trace["ops"].append({"op": "mutate", "id": str(cid), "stats": stats(),
                                     "resident": [str(r) for r in sorted(st.resident_chunk_ids())]})
        st.flush()
        trace["final_stats"] = stats()
        # final map content in canonical order (chunk id, then in-chunk index)
        content = []
        for cid, gs in st.iter_map():
            for g in gs:
                content.append([str(cid)] + g.position.tolist() + [g.opacity])
        trace["final_map"] = content
    for op in trace["ops"]:
        if op["op"] == "insert":
            op["resident"] = [str(r) for r in op["resident"]]
    (HERE / "store_trace.json").write_text(json.dumps(trace))


def make_view_edits():
    """Write-through view contract (store.py:361-379): the reference store
    edited in place through chunk.gaussians / gather_visible -- the
    refine_reset loop (loopclose.py:236-242: opacity + opt_state = b"" then
    mark_chunk_mutated), nudge-style sh0/opacity edits (sim.py:309-317) and
    scale edits through GaussianRefs -- interleaved with paging.  Records the
    declarative op list and the sha256 of every flushed chunk file."""
    import hashlib
    rng = np.random.default_rng(23)
    out = {"inserts": [], "ops": []}
    with tempfile.TemporaryDirectory() as d:
        st = store.ChunkStore(store.StoreConfig(disk_root=d, chunk_size_m=10.0, gaussian_budget=70,
                                                keyframe_budget=4, io_ns_per_byte=1.0))
        cells = [(x, y, 0) for x in range(-2, 2) for y in range(-1, 2)]
        gs = []
        for k in range(150):
            cx, cy, cz = cells[k % len(cells)]
            p = [cx * 10 + rng.uniform(-4.9, 4.9), cy * 10 + rng.uniform(-4.9, 4.9), rng.uniform(-4.9, 4.9)]
            opt = b"" if k % 5 else bytes(rng.integers(0, 256, int(rng.integers(1, 9))).astype(np.uint8))
            gs.append(core.Gaussian(position=p, opacity=float(rng.uniform(0, 1)),
                                    scale=rng.uniform(0.01, 1, size=3),
                                    rotation=core.quat_normalize(rng.normal(size=4)), sh=rng.normal(size=48),
                                    opt_state=opt))
        for a in range(0, 150, 50):
            batch = gs[a:a + 50]
            st.insert_gaussians(batch)
            out["inserts"].append([{"position": g.position.tolist(), "opacity": g.opacity,
                                    "scale": g.scale.tolist(), "rotation": g.rotation.tolist(),
                                    "sh": g.sh.tolist(), "opt": g.opt_state.hex()} for g in batch])
        all_ids = sorted(st.known_chunk_ids())
        f32 = lambda v: float(np.float32(v))  # noqa: E731
        for step in range(40):
            kind = rng.choice(["reset", "nudge", "scale", "ensure"], p=[0.2, 0.35, 0.2, 0.25])
            if kind == "ensure" or not st.resident_chunk_ids():
                ids = sorted({all_ids[int(rng.integers(len(all_ids)))] for _ in range(int(rng.integers(1, 4)))})
                st.ensure_resident(ids)
                out["ops"].append({"op": "ensure", "ids": [str(i) for i in ids]})
                continue
            res = sorted(st.resident_chunk_ids())
            cid = res[int(rng.integers(len(res)))]
            if kind == "reset":   # refine_reset's inner loop (loopclose.py:236-242)
                op = f32(rng.uniform(0.05, 0.2))
                for g in st.chunk(cid).gaussians:
                    g.opacity = op
                    g.opt_state = b""
                st.mark_chunk_mutated(cid)
                out["ops"].append({"op": "reset", "id": str(cid), "opacity": op})
            elif kind == "nudge":   # sim.py:309-317 style in-place edits
                n = len(st.chunk(cid))
                if not n:
                    continue
                edits = []
                for _ in range(int(rng.integers(1, 4))):
                    i = int(rng.integers(n))
                    g = st.chunk(cid).gaussians[i]
                    sh0 = np.float32(g.sh[[0, 16, 32]] + rng.normal(size=3) * 0.1).astype(np.float64)
                    g.sh[[0, 16, 32]] = sh0
                    newop = None
                    if rng.random() < 0.5:
                        newop = f32(min(1.0, g.opacity + 0.02))
                        g.opacity = newop
                    edits.append({"index": i, "sh0": sh0.tolist(), "opacity": newop})
                st.mark_chunk_mutated(cid)
                out["ops"].append({"op": "nudge", "id": str(cid), "edits": edits})
            else:   # in-place scale edits through gather_visible refs
                refs = st.gather_visible([cid])
                picks = sorted({int(rng.integers(len(refs))) for _ in range(3)}) if refs else []
                for k in picks:
                    g = refs[k].gaussian
                    g.scale[:] = np.float32(g.scale * 1.25).astype(np.float64)
                out["ops"].append({"op": "scale", "id": str(cid), "picks": picks})
        st.flush()
        out["files"] = {p.name: hashlib.sha256(p.read_bytes()).hexdigest()
                        for p in sorted((Path(d) / "chunks").glob("*.dcg"))}
    (HERE / "view_edits.json").write_text(json.dumps(out))


def make_sample():
    """Ingest path (sample.py:49-146, sim.py:264-278): log_norm of images
    (random, step edges, a rendered scene), sampling_probability,
    sample_pixels draws, lift_to_gaussians (rotated poses, invalid depth),
    and two reference _Replay.ingest_keyframe calls on a small scene."""
    from splatmap import sample, sim
    rng = np.random.default_rng(31)
    out = {}
    imgs = [rng.uniform(0, 1, (48, 64, 3)),
            np.repeat(np.repeat((rng.uniform(0, 1, (6, 8, 3)) > 0.5).astype(np.float64), 8, 0), 8, 1),
            np.zeros((20, 24, 3)), np.full((20, 24, 3), 0.6)]
    scene = _scene(rng, 300)
    intr = core.CameraIntrinsics(fx=50.0, fy=50.0, cx=31.5, cy=23.5, width=64, height=48, near=0.2, far=100.0)
    pose = core.Pose()
    imgs.append(renderloss.render_arrays(scene, pose, intr).rgb)
    for k, im in enumerate(imgs):
        out[f"img{k}"] = im
        for sig, rad in ((1.0, 2), (1.5, 3)):
            out[f"log{k}_{sig}_{rad}"] = sample.log_norm(im, sig, rad)
    out["n_img"] = np.array(len(imgs))
    a, b = out["log0_1.0_2"], out["log4_1.0_2"]
    ps = sample.sampling_probability(a, b)
    out["ps"] = ps
    for n, seed in ((50, 3), (500, 4), (5000, 5)):
        out[f"draw_{n}_{seed}"] = np.array(sample.sample_pixels(ps, n, seed), dtype=np.int64).reshape(-1, 2)
    # lift: rotated pose, some invalid depth, quantised rgb
    for k in range(3):
        q = core.quat_normalize(rng.normal(size=4))
        t = rng.normal(size=3) * 2
        depth = rng.uniform(0.5, 6.0, (48, 64)).astype(np.float32)
        depth[rng.random((48, 64)) < 0.2] = 0.0
        kf = core.Keyframe(id=k, pose=core.Pose(rotation=q, translation=t), intrinsics=intr,
                           rgb=rng.uniform(0, 1, (48, 64, 3)), depth=depth)
        pix = [(int(r), int(c)) for r, c in zip(rng.integers(0, 48, 200), rng.integers(0, 64, 200))]
        gs = sample.lift_to_gaussians(pix, kf, sample.SampleConfig(init_scale_factor=1.0 + 0.5 * k))
        out[f"lift{k}_q"], out[f"lift{k}_t"] = q, t
        out[f"lift{k}_rgb"], out[f"lift{k}_depth"] = kf.rgb, kf.depth
        out[f"lift{k}_pix"] = np.array(pix, dtype=np.int64)
        out[f"lift{k}_pos"] = np.array([g.position for g in gs])
        out[f"lift{k}_scale"] = np.array([g.scale for g in gs])
        out[f"lift{k}_sh0"] = np.array([g.sh[[0, 16, 32]] for g in gs])
    # two ingests through the reference replay (first: empty map, second: the
    # map the first inserted renders into the current view)
    with tempfile.TemporaryDirectory() as d:
        d = Path(d)
        cfg = sim.ReplayConfig(trajectory=d / "t", images_dir=d / "i", depth_dir=d / "d", out=d / "o.csv",
                               store_dir=d / "store", chunk_size=2.0, gaussian_budget=100_000, seed=7,
                               samples_per_keyframe=800)
        rep = sim._Replay(cfg, intr)
        for k in range(2):
            pose_k = core.Pose(translation=[0.1 * k, 0.0, 0.0])
            tgt = renderloss.render_arrays(scene, pose_k, intr)
            depth = np.where(tgt.alpha > 0.5, tgt.depth, 0.0).astype(np.float32)
            n_ins = rep.ingest_keyframe(k, pose_k, tgt.rgb, depth)
            out[f"ingest{k}_rgb"], out[f"ingest{k}_depth"] = tgt.rgb, depth
            out[f"ingest{k}_t"] = np.asarray(pose_k.translation)
            out[f"ingest{k}_n"] = np.array(n_ins)
        rows, cids = [], []
        for cid, gs in rep.store.iter_map():
            for g in gs:
                cids.append(cid)
                rows.append(list(g.position) + list(g.scale) + [g.opacity] + list(g.sh[[0, 16, 32]]))
        out["ingest_map"] = np.array(rows)
        out["ingest_cids"] = np.array(cids, dtype=np.uint64)
    np.savez_compressed(HERE / "sample.npz", **out)


def make_loopclose():
    """Loop-closure correction (loopclose.py:146-268) on the reference store:
    two clusters, two keyframes, a rotation + translation and a translation
    (each crossing chunk boundaries), keyframe 1 a junction, batch and
    sequential modes (budget 150 forces paging in sequential).  Records the
    outcome reports, stats and the flushed map."""
    from splatmap import loopclose
    out = {}
    intr = core.CameraIntrinsics(fx=20.0, fy=20.0, cx=8.0, cy=8.0, width=16, height=16, near=0.1, far=60.0)

    def cluster(rng, n, center, spread):
        gs = []
        for _ in range(n):
            sh = np.zeros(48)
            sh[[0, 16, 32]] = (rng.uniform(0.1, 0.9, 3) - 0.5) / 0.28209479177
            gs.append(core.Gaussian(position=np.asarray(center) + rng.uniform(-spread, spread, 3),
                                    rotation=core.quat_normalize(rng.normal(size=4)),
                                    scale=rng.uniform(0.08, 0.25, size=3), opacity=float(rng.uniform(0.4, 0.9)),
                                    sh=sh, opt_state=rng.bytes(4)))
        return gs

    def kf(kid, pose):
        r = np.random.default_rng(kid + 100)
        return core.Keyframe(id=kid, pose=pose, intrinsics=intr, rgb=r.integers(0, 256, size=(16, 16, 3)) / 255.0,
                             depth=r.uniform(1, 10, size=(16, 16)).astype(np.float32))

    cs = loopclose.CorrectionSet(entries=(
        (0, core.RigidTransform(rotation=core.quat_normalize([0.98, 0.0, 0.0, 0.2]), translation=[12.0, 0.0, 0.0])),
        (1, core.RigidTransform(translation=[0.0, 11.0, 0.0]))), junction_ids=frozenset({1}))
    cull = culling.CullConfig(max_distance_m=100.0)
    inserts = []
    rng = np.random.default_rng(13)
    for n_c, center in ((50, (0.0, 0.0, 4.0)), (50, (3.0, 0.0, 8.0)), (70, (60.0, 0.0, 4.0))):
        gs = cluster(rng, n_c, center, 2.0)
        inserts.append([[*g.position, *g.rotation, *g.scale, g.opacity, *g.sh[[0, 16, 32]]] for g in gs])
        out.setdefault("opts", []).extend(g.opt_state.hex() for g in gs)
    out["inserts"] = inserts
    for mode in (loopclose.CorrectionMode.BATCH, loopclose.CorrectionMode.SEQUENTIAL):
        with tempfile.TemporaryDirectory() as d:
            st = store.ChunkStore(store.StoreConfig(disk_root=Path(d), gaussian_budget=150, keyframe_budget=8,
                                                    io_ns_per_byte=1.0))
            r2 = np.random.default_rng(13)
            st.insert_gaussians(cluster(r2, 50, (0.0, 0.0, 4.0), 2.0))
            st.insert_gaussians(cluster(r2, 50, (3.0, 0.0, 8.0), 2.0))
            st.insert_gaussians(cluster(r2, 70, (60.0, 0.0, 4.0), 2.0))   # out of view: paging
            st.keyframe_add(kf(0, core.Pose()))
            st.keyframe_add(kf(1, core.Pose(translation=[2.0, 0.0, 0.0])))
            o = loopclose.run_correction(cs, st, cull, force_mode=mode)
            st.flush()
            m = []
            for cid, gs in st.iter_map():
                for g in gs:
                    m.append([str(cid), *g.position, *g.rotation, *g.scale, g.opacity, *g.sh[[0, 16, 32]],
                              g.opt_state.hex()])
            s_ = st.stats
            out[mode.value] = {
                "plan": [o.plan.mode.value, sorted(str(c) for c in o.plan.unique_chunks), o.plan.estimated_gaussians],
                "report": [o.report.transformed, o.report.skipped_duplicates,
                           sorted(str(c) for c in o.report.touched_chunks)],
                "moves": [o.moves.moved, sorted(str(c) for c in o.moves.created_chunks),
                          sorted(str(c) for c in o.moves.emptied_chunks)],
                "resets": o.reset_gaussians,
                "stats": [s_.chunk_loads, s_.chunk_evictions, s_.chunk_writes, s_.total_gaussians_ever],
                "poses": [[*st.keyframe_get(k).pose.rotation, *st.keyframe_get(k).pose.translation] for k in (0, 1)],
                "map": m}
    (HERE / "loopclose.json").write_text(json.dumps(out))


def make_keyframe_trace():
    """Keyframe tier policy (store.py:427-489): seeded add / get / dirty /
    update_keyframe_pose / flush operations under a budget of 3; after each
    op the resident ids in LRU order and the keyframe stats; at the end the
    sha256 of every .dkf file (diskformat.py:198-250)."""
    import hashlib
    rng = np.random.default_rng(29)
    intr = core.CameraIntrinsics(fx=10.0, fy=10.0, cx=4.0, cy=3.0, width=8, height=6, near=0.1, far=50.0)
    ops, added = [], []
    with tempfile.TemporaryDirectory() as d:
        st = store.ChunkStore(store.StoreConfig(disk_root=Path(d), keyframe_budget=3, io_ns_per_byte=1.0))
        for step in range(90):
            kind = rng.choice(["add", "get", "dirty", "pose", "flush"], p=[0.25, 0.45, 0.12, 0.12, 0.06])
            if kind == "add" or not added:
                kid = len(added)
                pose = core.Pose(rotation=core.quat_normalize(rng.normal(size=4)), translation=rng.normal(size=3))
                rgb = rng.uniform(0, 1, (6, 8, 3))
                depth = rng.uniform(0.5, 5.0, (6, 8)).astype(np.float32)
                kf = core.Keyframe(id=kid, pose=pose, intrinsics=intr, rgb=rgb, depth=depth,
                                   last_loss=float(rng.uniform(0, 1)), usage_remaining=int(rng.integers(0, 9)))
                st.keyframe_add(kf)
                added.append(kid)
                op = {"op": "add", "id": kid, "q": pose.rotation.tolist(), "t": pose.translation.tolist(),
                      "rgb": rgb.tolist(), "depth": depth.tolist(), "loss": kf.last_loss,
                      "usage": kf.usage_remaining}
            elif kind == "get":
                kid = int(added[int(rng.integers(len(added)))])
                st.keyframe_get(kid)
                op = {"op": "get", "id": kid}
            elif kind == "dirty":
                res = list(st._keyframes)
                kid = int(res[int(rng.integers(len(res)))])
                st.mark_keyframe_dirty(kid)
                op = {"op": "dirty", "id": kid}
            elif kind == "pose":
                kid = int(added[int(rng.integers(len(added)))])
                pose = core.Pose(rotation=core.quat_normalize(rng.normal(size=4)), translation=rng.normal(size=3))
                st.update_keyframe_pose(kid, pose)
                op = {"op": "pose", "id": kid, "q": pose.rotation.tolist(), "t": pose.translation.tolist()}
            else:
                st.flush()
                op = {"op": "flush"}
            s_ = st.stats
            op["resident"] = [int(k) for k in st._keyframes]
            op["stats"] = [s_.keyframe_loads, s_.keyframe_evictions, s_.keyframe_writes, s_.io_nanos,
                           s_.bytes_read, s_.bytes_written, s_.active_keyframes]
            ops.append(op)
        st.flush()
        files = {p.name: hashlib.sha256(p.read_bytes()).hexdigest()
                 for p in sorted((Path(d) / "keyframes").glob("*.dkf"))}
    (HERE / "keyframe_trace.json").write_text(json.dumps({"ops": ops, "files": files}))


def make_select_trace():
    """KeyframeIndex / select_keyframe / record_loss policy trace (select.py)."""
    from splatmap import select, sim
    rng = np.random.default_rng(21)
    idx = select.KeyframeIndex(config=select.SelectConfig(grid_resolution_m=50.0))
    ops = []
    for k in range(12):
        pos = rng.uniform(-80, 80, size=3)
        idx.add(k, pos)
        ops.append({"op": "add", "id": k, "pos": pos.tolist()})
    for step in range(200):
        latest = int(rng.integers(0, 12))
        try:
            cands = select.candidate_set(idx.position_of(latest), idx)
        except Exception:
            cands = [latest]
        seed = sim._derive_seed(7, 2, step)
        chosen = select.select_keyframe(cands, idx, seed)
        loss = float(rng.uniform(0, 2)) if step % 7 else 0.0
        select.record_loss(chosen, loss, idx)
        ops.append({"op": "step", "latest": latest, "cands": cands, "seed": seed, "chosen": chosen,
                    "loss": loss, "usage": [idx.usage_of(i) for i in range(12)]})
    (HERE / "select_trace.json").write_text(json.dumps(ops))


if __name__ == "__main__":
    make_select_trace()
    print("reference splatmap", splatmap.__version__, "from", splatmap.__file__)
    make_render_small()
    make_loss()
    make_grid()
    make_diskformat()
    make_store_trace()
    make_view_edits()
    make_sample()
    make_loopclose()
    make_keyframe_trace()
    make_render_fd()
    for p in sorted(HERE.glob("*.npz")) + sorted(HERE.glob("*.json")):
        print(f"{p.name:24s} {p.stat().st_size:>9d} bytes")
