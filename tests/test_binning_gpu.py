"""Bit-exact pin of the tile binning (K2/K3): the device's global depth order,
its tile-sorted (tile, depth rank) instance keys and its per-tile instance
ranges equal the CPU restatement oracle/bin_oracle.c element for element.

The reference composites every pixel of each Gaussian's clamped 3-sigma box
(renderloss.py:122-135) in np.argsort(z, kind="stable") order
(renderloss.py:202); binning is how the device splits that loop into 16x16
tiles, so it has no reference output to compare with -- the restatement of
the same arithmetic (one rounding per op, no FMA) is the oracle.  Cases: the
C1-shaped 20k scene, the edge-case scene (ragged image, near-plane
stragglers, off-screen boxes, needles, saturating stack), the C2 full-size
1M-splat view, and 64-bit keys (a workspace sized past 2M splats) -- each
with the ellipse tile cull on and off (off = exactly the reference's 3-sigma
box tiles).
"""
import ctypes

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_cases import edge_scene, f32

pytestmark = pytest.mark.gpu


def _device_binning(scene, pose, intr, min_gaussians=None):
    import torch

    from paper_2511_23030_b200 import _lib
    from paper_2511_23030_b200 import renderloss as rl
    lib = _lib.load()
    sa = rl.SceneArrays(**scene)
    params = torch.from_numpy(rl.pack_params(sa)).cuda()
    eng = rl.RenderEngine("cuda")
    if min_gaussians:
        eng.ensure(min_gaussians, intr.width, intr.height)
    rl.render_device(params, None, len(sa), pose, intr, eng)
    torch.cuda.synchronize()
    n_inst = eng.counters()["n_instances"]
    rb, kb = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(lib.sm_render_key_layout(ctypes.byref(eng.dims), ctypes.byref(rb), ctypes.byref(kb)))
    ws = eng.ws
    o = lib.sm_render_ws_offset(eng.dims, 4)
    raw = ws[o:o + n_inst * kb.value].cpu().numpy()
    keys = raw.view(np.uint64 if kb.value == 8 else np.uint32).astype(np.uint64)
    tiles = rl.RenderEngine.n_tiles(intr.width, intr.height)
    o = lib.sm_render_ws_offset(eng.dims, 0)
    ranges = ws[o:o + 8 * tiles].cpu().numpy().view(np.uint32).reshape(tiles, 2)
    o = lib.sm_render_ws_offset(eng.dims, 2)
    order = ws[o:o + 4 * len(sa)].cpu().numpy().view(np.uint32).astype(np.int64)
    return order, keys, ranges, rb.value, kb.value, params.cpu().numpy()


def _check(scene, pose, intr, tag, min_gaussians=None):
    from paper_2511_23030_b200 import _lib
    lib = _lib.load()
    counts = []
    try:
        for cull in (1, 0):
            lib.sm_set_ellipse_cull(cull)
            order, keys, ranges, rb, kb, params = _device_binning(scene, pose, intr, min_gaussians)
            o_order, o_keys, o_ranges = O.bin_tiles(params, pose.rotation, pose.translation, intr.fx, intr.fy,
                                                    intr.cx, intr.cy, intr.near, intr.width, intr.height,
                                                    ellipse_cull=bool(cull), rank_bits=rb)
            assert np.array_equal(order, o_order), (tag, cull, "depth order")
            assert len(keys) == len(o_keys), (tag, cull, len(keys), len(o_keys))
            assert np.array_equal(keys, o_keys), (tag, cull, "keys", int(np.flatnonzero(keys != o_keys)[0]))
            assert np.array_equal(ranges, o_ranges), (tag, cull, "ranges")
            counts.append(len(keys))
    finally:
        lib.sm_set_ellipse_cull(1)
    assert counts[0] <= counts[1], (tag, counts)   # the ellipse cull only drops tiles
    return rb, kb, counts


def test_binning_c1_scene_bit_exact(cuda):
    from paper_2511_23030_b200.core import CameraIntrinsics, Pose, quat_normalize
    rng = np.random.default_rng(7)
    n = 20000
    pos = np.stack([rng.uniform(-6, 6, n), rng.uniform(-4, 4, n), rng.uniform(-1.0, 14.0, n)], 1)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    scene = f32(dict(positions=pos, rotations=q, scales=np.exp(rng.uniform(np.log(0.01), np.log(0.2), (n, 3))),
                     opacities=rng.uniform(0.3, 0.95, n), sh0=rng.normal(size=(n, 3))))
    intr = CameraIntrinsics(fx=120.0, fy=120.0, cx=80.0, cy=60.0, width=160, height=120, near=0.05)
    pose = Pose(rotation=quat_normalize([1.0, 0.02, -0.03, 0.01]), translation=[0.1, -0.2, 0.3])
    rb, kb, counts = _check(scene, pose, intr, "c1")
    assert kb == 4 and counts[0] > n


def test_binning_edge_cases_bit_exact(cuda):
    scene, pose, intr, _ = edge_scene()
    _check(scene, pose, intr, "edge")


def test_binning_full_size_c2_view_bit_exact(cuda):
    from paper_2511_23030_b200.synthetic import C2_INTR, room_poses, room_scene
    sc = room_scene(1_000_000, seed=42)
    scene = dict(positions=sc.positions, rotations=sc.rotations, scales=sc.scales,
                 opacities=sc.opacities, sh0=sc.sh0)
    poses = room_poses(16, seed=42)
    _, kb, _ = _check(scene, poses[5], C2_INTR, "c2-view5")
    assert kb == 4
    # 64-bit keys: a workspace sized past 2M splats (22 rank bits + 11 tile bits)
    _, kb, _ = _check(scene, poses[11], C2_INTR, "c2-view11-wide", min_gaussians=3_000_000)
    assert kb == 8
