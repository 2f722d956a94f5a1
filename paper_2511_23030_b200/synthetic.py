"""Seeded synthetic workloads for the BASELINE.json configurations.

All values are float32-canonical like the store.  Quaternions are normalised
N(0,1)^4, scales log-uniform per axis, opacity U(0.3, 0.95), colours
U(0.05, 0.95) encoded as sh0 = (c - 0.5) / SH_C0 with the other 45 SH zero.

* C1: 20k uniform in x,y in [-5,15), z in [-5,5) (s = 10 -> 2x2x1 chunks),
  160x120, fx = fy = 120.
* C2: "Replica-shaped" room: 1M Gaussians on the floor, ceiling and four
  walls of an 8 x 8 x 2 m room (s = 1 m -> 8x8x2 chunks) plus box clutter,
  scales 0.5-5 cm, 640x480, fx = fy = 525, cx = 319.5, cy = 239.5.
Keyframe poses look horizontally from inside the room (corridor camera
convention q = (0.5, -0.5, 0.5, -0.5) of sim.py:448, yawed).  Ground-truth
images are renders of a perturbed copy of the scene (held-out colour and
opacity edits), 8-bit quantised like Keyframe (core.py:262-267).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .core import SH_C0, CameraIntrinsics, Pose, quat_multiply, quat_normalize

__all__ = ["SceneData", "uniform_scene", "room_scene", "room_poses", "corridor_scene",
           "corridor_poses", "C1_INTR", "C2_INTR", "C4_INTR", "perturbed"]

C1_INTR = CameraIntrinsics(fx=120.0, fy=120.0, cx=80.0, cy=60.0, width=160, height=120, near=0.05)
C2_INTR = CameraIntrinsics(fx=525.0, fy=525.0, cx=319.5, cy=239.5, width=640, height=480, near=0.05)
# KITTI-00
C4_INTR = CameraIntrinsics(fx=718.856, fy=718.856, cx=607.19, cy=185.22, width=1241, height=376, near=0.05)
_BASE_Q = quat_normalize(np.array([0.5, -0.5, 0.5, -0.5]))   # cam z -> +x, cam y -> -z


@dataclass
class SceneData:
    positions: np.ndarray   # (N, 3) float64 (float32-canonical)
    rotations: np.ndarray   # (N, 4)
    scales: np.ndarray      # (N, 3)
    opacities: np.ndarray   # (N,)
    sh: np.ndarray          # (N, 48)

    def __len__(self):
        return self.positions.shape[0]

    @property
    def sh0(self) -> np.ndarray:
        return self.sh[:, [0, 16, 32]]

    def subset(self, idx) -> "SceneData":
        return SceneData(self.positions[idx], self.rotations[idx], self.scales[idx],
                         self.opacities[idx], self.sh[idx])


def _c(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def _attributes(rng, n, scale_lo, scale_hi):
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q = _c(q)
    # float32 rounding can push |q| off 1 by ~1e-7: renormalise in float32 space
    q = _c(q / np.linalg.norm(q, axis=1, keepdims=True))
    scales = np.exp(rng.uniform(math.log(scale_lo), math.log(scale_hi), size=(n, 3)))
    op = rng.uniform(0.3, 0.95, n)
    col = rng.uniform(0.05, 0.95, size=(n, 3))
    sh = np.zeros((n, 48))
    sh[:, [0, 16, 32]] = (col - 0.5) / SH_C0
    return q, _c(scales), _c(op), _c(sh)


def uniform_scene(n: int, lo, hi, seed: int, scale_lo=0.02, scale_hi=0.25) -> SceneData:
    rng = np.random.default_rng(seed)
    pos = rng.uniform(lo, hi, size=(n, 3))
    q, s, o, sh = _attributes(rng, n, scale_lo, scale_hi)
    return SceneData(_c(pos), q, s, o, sh)


def room_scene(n: int = 1_000_000, seed: int = 42, size=(8.0, 8.0, 2.0), chunk: float = 1.0,
               clutter_frac: float = 0.25, scale_lo=0.005, scale_hi=0.05) -> SceneData:
    """Surfaces + clutter of a size[0] x size[1] x size[2] room aligned to the chunk grid."""
    rng = np.random.default_rng(seed)
    lo = np.full(3, -chunk / 2.0)
    hi = lo + np.asarray(size)
    eps = 0.02   # keep splats strictly inside the room's chunks
    lo_in, hi_in = lo + eps, hi - eps
    n_clutter = int(n * clutter_frac)
    n_surf = n - n_clutter
    dx, dy, dz = hi_in - lo_in
    areas = np.array([dx * dy, dx * dy, dx * dz, dx * dz, dy * dz, dy * dz])
    face = rng.choice(6, size=n_surf, p=areas / areas.sum())
    u = rng.uniform(size=(n_surf, 3))
    pos = lo_in + u * (hi_in - lo_in)
    pos[face == 0, 2] = lo_in[2]
    pos[face == 1, 2] = hi_in[2]
    pos[face == 2, 1] = lo_in[1]
    pos[face == 3, 1] = hi_in[1]
    pos[face == 4, 0] = lo_in[0]
    pos[face == 5, 0] = hi_in[0]
    pos += rng.normal(scale=0.004, size=pos.shape)   # surface roughness
    # clutter: points on the faces of random boxes standing on the floor
    n_box = 24
    bc = rng.uniform(lo_in[:2] + 0.6, hi_in[:2] - 0.6, size=(n_box, 2))
    bs = rng.uniform([0.2, 0.2, 0.2], [0.9, 0.9, 1.2], size=(n_box, 3))
    which = rng.integers(0, n_box, n_clutter)
    cmin = np.concatenate([bc[which] - bs[which, :2] / 2, np.full((n_clutter, 1), lo_in[2])], 1)
    cext = bs[which]
    cu = rng.uniform(size=(n_clutter, 3))
    cface = rng.integers(0, 5, n_clutter)   # 4 sides + top
    cp = cmin + cu * cext
    axis = np.array([0, 0, 1, 1, 2])[cface]
    side = np.array([0, 1, 0, 1, 1])[cface]
    cp[np.arange(n_clutter), axis] = cmin[np.arange(n_clutter), axis] + side * cext[np.arange(n_clutter), axis]
    pos = np.concatenate([pos, cp], 0)
    pos = np.clip(pos, lo_in, hi_in)
    perm = rng.permutation(n)
    q, s, o, sh = _attributes(rng, n, scale_lo, scale_hi)
    return SceneData(_c(pos[perm]), q, s, o, sh)


def room_poses(k: int, seed: int = 42, size=(8.0, 8.0, 2.0), chunk: float = 1.0,
               height: float = 0.5) -> list[Pose]:
    """k horizontal-looking cameras inside the room (yaw spread, small jitter)."""
    rng = np.random.default_rng(seed + 1)
    lo = -chunk / 2.0
    poses = []
    for i in range(k):
        yaw = 2.0 * math.pi * i / k + rng.uniform(-0.2, 0.2)
        qz = np.array([math.cos(yaw / 2), 0.0, 0.0, math.sin(yaw / 2)])
        rot = quat_normalize(quat_multiply(qz, _BASE_Q))
        c = np.array([lo + size[0] / 2, lo + size[1] / 2, lo + height]) + \
            rng.uniform(-1.5, 1.5, 3) * np.array([1, 1, 0.2])
        # back the camera away from the wall it faces so the frustum sees the room
        fwd = np.array([math.cos(yaw), math.sin(yaw), 0.0])
        poses.append(Pose(rotation=rot, translation=c - 1.2 * fwd))
    return poses


def corridor_scene(n: int, length: float = 200.0, width: float = 40.0, seed: int = 7,
                   scale_lo=0.02, scale_hi=0.2) -> SceneData:
    """C4-shaped street corridor along +x (20k splats per metre,
    s = 10 m chunks, 4 chunks across): road surface, two building facades,
    and boxes (parked cars / street furniture) along the kerbs."""
    rng = np.random.default_rng(seed)
    half = width / 2.0 - 0.05
    n_road, n_wall = int(n * 0.35), int(n * 0.4)
    n_box = n - n_road - n_wall
    road = np.stack([rng.uniform(0.05, length - 0.05, n_road), rng.uniform(-half, half, n_road),
                     np.full(n_road, -1.6) + rng.normal(scale=0.01, size=n_road)], 1)
    side = rng.integers(0, 2, n_wall)
    wall = np.stack([rng.uniform(0.05, length - 0.05, n_wall),
                     np.where(side == 0, -12.0, 12.0) + rng.normal(scale=0.05, size=n_wall),
                     rng.uniform(-1.6, 4.9, n_wall)], 1)
    nb = max(1, int(length / 4))
    bx = rng.uniform(0.5, length - 0.5, nb)
    by = np.where(rng.integers(0, 2, nb) == 0, -6.0, 6.0) + rng.uniform(-1.0, 1.0, nb)
    bsz = rng.uniform([1.5, 0.8, 0.8], [4.5, 2.0, 1.8], size=(nb, 3))
    which = rng.integers(0, nb, n_box)
    cmin = np.stack([bx[which] - bsz[which, 0] / 2, by[which] - bsz[which, 1] / 2, np.full(n_box, -1.6)], 1)
    cp = cmin + rng.uniform(size=(n_box, 3)) * bsz[which]
    face = rng.integers(0, 5, n_box)
    axis = np.array([0, 0, 1, 1, 2])[face]
    top = np.array([0, 1, 0, 1, 1])[face]
    rows = np.arange(n_box)
    cp[rows, axis] = cmin[rows, axis] + top * bsz[which][rows, axis]
    pos = np.concatenate([road, wall, cp], 0)
    pos = np.clip(pos, [0.01, -half, -4.9], [length - 0.01, half, 4.9])
    pos = pos[rng.permutation(n)]
    q, sc, o, sh = _attributes(rng, n, scale_lo, scale_hi)
    return SceneData(_c(pos), q, sc, o, sh)


def corridor_poses(k: int, spacing: float = 2.0, seed: int = 7) -> list[Pose]:
    """A car driving along +x at 1.5 m above the road, slight lateral wander."""
    rng = np.random.default_rng(seed + 1)
    poses = []
    for i in range(k):
        yaw = rng.uniform(-0.05, 0.05)
        qz = np.array([math.cos(yaw / 2), 0.0, 0.0, math.sin(yaw / 2)])
        rot = quat_normalize(quat_multiply(qz, _BASE_Q))
        poses.append(Pose(rotation=rot, translation=np.array([1.0 + i * spacing, rng.uniform(-1.0, 1.0), 0.0])))
    return poses


def perturbed(scene: SceneData, seed: int, frac: float = 0.2) -> SceneData:
    """Held-out edit of the scene used to make ground-truth views."""
    rng = np.random.default_rng(seed)
    n = len(scene)
    sh = scene.sh.copy()
    op = scene.opacities.copy()
    pick = rng.random(n) < frac
    col = rng.uniform(0.05, 0.95, size=(int(pick.sum()), 3))
    sh[np.ix_(pick, [0, 16, 32])] = (col - 0.5) / SH_C0
    op[pick] = rng.uniform(0.3, 0.95, int(pick.sum()))
    return SceneData(scene.positions, scene.rotations, scene.scales, _c(op), _c(sh))
