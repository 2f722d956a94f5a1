"""Benchmark / smoke workloads assembled from the synthetic generators.

``build_c2`` creates the BASELINE.json configs[1] case: a 1M-Gaussian
Replica-shaped room in a ChunkStore (s = 1 m -> 8x8x2 chunks, budget 1.5M,
everything resident), 640x480 keyframes whose ground truth is rendered from
a perturbed copy of the scene.  ``build_c1`` is the 20k / 160x120 config[0]
shape used by smoke() and the parity tests.
"""

from __future__ import annotations

import tempfile
from pathlib import Path

import numpy as np

from .core import Keyframe
from .culling import CullConfig
from .mapping import MappingEngine
from .renderloss import SceneArrays, default_engine, pack_params, render_device
from .store import ChunkStore, StoreConfig
from .synthetic import (C1_INTR, C2_INTR, C4_INTR, SceneData, corridor_poses, corridor_scene, perturbed,
                        room_poses, room_scene, uniform_scene)


def _gt_frames(target: SceneData, poses, intr, device):
    import torch
    sa = SceneArrays(target.positions, target.rotations, target.scales, target.opacities, target.sh0)
    params = torch.from_numpy(pack_params(sa)).to(device)
    eng = default_engine(device)
    out = []
    for pose in poses:
        rgb, depth, _ = render_device(params, None, len(sa), pose, intr, eng)
        out.append((rgb.cpu().numpy(), depth.cpu().numpy()))
    del params
    return out


def build_engine(scene: SceneData, poses, intr, chunk_size: float, budget: int,
                 store_dir: Path | None = None, device=None, seed: int = 7,
                 max_distance: float = 200.0, target_seed: int = 49,
                 keyframe_budget: int = 400) -> MappingEngine:
    import torch
    device = torch.device(device if device is not None else "cuda")
    store_dir = Path(store_dir or tempfile.mkdtemp(prefix="splatmap_b200_"))
    store = ChunkStore(StoreConfig(disk_root=store_dir, chunk_size_m=chunk_size,
                                   gaussian_budget=budget, keyframe_budget=keyframe_budget, io_ns_per_byte=1.0,
                                   device=str(device)))
    store.insert_arrays(scene.positions, scene.rotations, scene.scales, scene.opacities, scene.sh)
    eng = MappingEngine(store, intr, seed=seed, cull=CullConfig(max_distance_m=max_distance))
    frames = _gt_frames(perturbed(scene, target_seed), poses, intr, device)
    for k, (pose, (rgb, depth)) in enumerate(zip(poses, frames)):
        eng.add_keyframe(Keyframe(id=k, pose=pose, intrinsics=intr, rgb=rgb, depth=depth))
    return eng


def build_c2(n: int = 1_000_000, keyframes: int = 16, store_dir=None, device=None) -> MappingEngine:
    scene = room_scene(n, seed=42)
    return build_engine(scene, room_poses(keyframes, seed=42), C2_INTR, 1.0, 1_500_000,
                        store_dir, device)


def c1_scene(n: int = 20_000) -> SceneData:
    return uniform_scene(n, lo=[-5.0, -5.0, -5.0], hi=[15.0, 15.0, 5.0], seed=1)


def c1_poses(k: int = 10):
    from .core import Pose, quat_normalize
    base = quat_normalize(np.array([0.5, -0.5, 0.5, -0.5]))   # looking along +x
    return [Pose(rotation=base, translation=np.array([-12.0 + i * 1.5, 5.0 + 0.3 * i, 0.0]))
            for i in range(k)]


def build_c1(n: int = 20_000, keyframes: int = 10, budget: int = 12_000, store_dir=None,
             device=None, keyframe_budget: int = 400) -> MappingEngine:
    return build_engine(c1_scene(n), c1_poses(keyframes), C1_INTR, 10.0, budget, store_dir, device,
                        keyframe_budget=keyframe_budget)


def build_c4lite(n: int = 4_000_000, length: float = 200.0, keyframes: int = 100, budget: int = 1_500_000,
                 store_dir=None, device=None, max_distance: float = 50.0) -> MappingEngine:
    """Out-of-core C4 shape at 1/5 length: a street corridor
    with C4's density (20k splats/m, s = 10 m, 4 chunks across), KITTI
    intrinsics, a 1.5M-splat HBM budget, keyframes every 2 m."""
    scene = corridor_scene(n, length=length, seed=7)
    return build_engine(scene, corridor_poses(keyframes, spacing=length / keyframes), C4_INTR, 10.0, budget,
                        store_dir, device, max_distance=max_distance)
