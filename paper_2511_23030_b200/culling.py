"""Frustum extraction and per-chunk visibility (splatmap culling.py:1-246).

``extract_frustum`` evaluates the reference's NumPy expression sequence
(culling.py:80-101) so the six planes are bit-identical on the same host.
``visible_chunks`` replaces the octree-halving recursion with a brute-force
pass of kernel K1 (sm_cull_chunks) over the candidate chunk table: the
reference proves its recursion equal to brute force (culling.py:1-9,
test_acceptance.py criterion 2), and K1 applies the same p-vertex and
nearest-point tests in fp64 with one rounding per operation.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum
from typing import Callable, Iterable

import numpy as np

from .core import CameraIntrinsics, Pose, quat_to_matrix
from .grid import ChunkAabb, ChunkCoord, decode_ids, encode_id

__all__ = ["FrustumTest", "Frustum", "CullConfig", "ChunkExtent", "extract_frustum",
           "aabb_in_frustum", "visible_chunks", "VisibilityCache", "cull_ids"]


class FrustumTest(Enum):
    OUTSIDE = 0
    INTERSECTS = 1
    INSIDE = 2


@dataclass(frozen=True)
class Frustum:
    """Six inward planes [nx, ny, nz, d]; inside is n.x + d >= 0."""

    planes: np.ndarray

    def contains_point(self, p) -> bool:
        p = np.asarray(p, dtype=np.float64)
        return bool(np.all(self.planes[:, :3] @ p + self.planes[:, 3] >= 0.0))


@dataclass(frozen=True)
class CullConfig:
    max_distance_m: float = 200.0
    max_subdivision_depth: int = 8
    cache_capacity: int = 64
    pose_quantum_m: float = 0.01
    pose_quantum_rad: float = 0.001

    def __post_init__(self):
        if min(self.max_distance_m, self.max_subdivision_depth, self.cache_capacity,
               self.pose_quantum_m, self.pose_quantum_rad) <= 0:
            raise ValueError("all culling parameters must be positive")


@dataclass(frozen=True)
class ChunkExtent:
    min_coord: ChunkCoord
    max_coord: ChunkCoord

    def __post_init__(self):
        if any(a > b for a, b in zip(self.min_coord, self.max_coord)):
            raise ValueError("extent min must be <= max component-wise")


def extract_frustum(pose: Pose, intr: CameraIntrinsics) -> Frustum:
    """World-frame inward planes: near, far and the four pixel-bound sides."""
    w, h = float(intr.width), float(intr.height)
    normals = (
        (np.array([0.0, 0.0, 1.0]), -intr.near),
        (np.array([0.0, 0.0, -1.0]), intr.far),
        (np.array([intr.fx, 0.0, intr.cx]), 0.0),
        (np.array([-intr.fx, 0.0, w - intr.cx]), 0.0),
        (np.array([0.0, intr.fy, intr.cy]), 0.0),
        (np.array([0.0, -intr.fy, h - intr.cy]), 0.0),
    )
    r = quat_to_matrix(pose.rotation)
    t = pose.translation
    planes = []
    for n, d in normals:
        unit = n / np.linalg.norm(n)
        nw = r @ unit
        planes.append([*nw, d - float(nw @ t)])
    return Frustum(planes=np.array(planes))


def aabb_in_frustum(box: ChunkAabb, f: Frustum) -> FrustumTest:
    """p-vertex / n-vertex classification (host form of the K1 test)."""
    inside = True
    for nx, ny, nz, d in f.planes:
        hi = (box.max[0] if nx >= 0 else box.min[0], box.max[1] if ny >= 0 else box.min[1],
              box.max[2] if nz >= 0 else box.min[2])
        if nx * hi[0] + ny * hi[1] + nz * hi[2] + d < 0.0:
            return FrustumTest.OUTSIDE
        lo = (box.min[0] if nx >= 0 else box.max[0], box.min[1] if ny >= 0 else box.max[1],
              box.min[2] if nz >= 0 else box.max[2])
        if nx * lo[0] + ny * lo[1] + nz * lo[2] + d < 0.0:
            inside = False
    return FrustumTest.INSIDE if inside else FrustumTest.INTERSECTS


def cull_ids(ids: np.ndarray, pose: Pose, intr: CameraIntrinsics, max_distance: float,
             s: float, frustum: Frustum | None = None) -> np.ndarray:
    """K1 over a table of chunk ids; returns the visible subset (sorted)."""
    import ctypes

    import torch

    from . import _lib
    ids = np.asarray(ids, dtype=np.uint64)
    if ids.size == 0:
        return ids
    coords = torch.as_tensor(decode_ids(ids).astype(np.int32), device="cuda")
    return cull_table(ids, coords, pose, intr, max_distance, s, frustum)


def cull_table(ids: np.ndarray, coords, pose: Pose, intr: CameraIntrinsics, max_distance: float,
               s: float, frustum: Frustum | None = None) -> np.ndarray:
    """K1 over a chunk table already on the device (`coords` = the ids'
    int32 chunk coordinates, e.g. ChunkStore.chunk_table's, kept per chunk-set
    generation); returns the visible subset of `ids` (sorted)."""
    import ctypes

    import torch

    from . import _lib
    if ids.size == 0:
        return ids
    lib = _lib.load()
    fr = frustum or extract_frustum(pose, intr)
    out = torch.empty(ids.size, dtype=torch.uint8, device=coords.device)
    planes = np.ascontiguousarray(fr.planes, dtype=np.float64)
    cam = np.ascontiguousarray(pose.translation, dtype=np.float64)
    dp = ctypes.POINTER(ctypes.c_double)
    rc = lib.sm_cull_chunks(_lib.ptr(coords), int(ids.size), planes.ctypes.data_as(dp),
                            cam.ctypes.data_as(dp), float(max_distance), float(s), _lib.ptr(out),
                            _lib.stream_handle())
    _lib.check(rc, "cull_chunks")
    mask = out.cpu().numpy().astype(bool)
    return np.sort(ids[mask])


def _candidates(extent: ChunkExtent, existing: Callable[[int], bool],
                candidates: Iterable[int] | None) -> np.ndarray:
    lo = np.array(tuple(extent.min_coord))
    hi = np.array(tuple(extent.max_coord))
    if candidates is None:
        owner = getattr(existing, "__self__", None)
        if isinstance(owner, (set, frozenset, dict)) and getattr(existing, "__name__", "") == "__contains__":
            candidates = owner
    if candidates is not None:
        ids = np.fromiter((int(c) for c in candidates), dtype=np.uint64)
        if ids.size == 0:
            return ids
        c = decode_ids(ids)
        keep = np.all((c >= lo) & (c <= hi), axis=1)
        return ids[keep]
    span = hi - lo + 1
    if int(np.prod(span)) > (1 << 24):
        raise ValueError("extent too large to enumerate; pass candidates=")
    grids = np.meshgrid(*(np.arange(a, b + 1) for a, b in zip(lo, hi)), indexing="ij")
    coords = np.stack([g.reshape(-1) for g in grids], axis=1)
    ids = np.array([encode_id(ChunkCoord(int(x), int(y), int(z))) for x, y, z in coords],
                   dtype=np.uint64)
    return ids[np.array([bool(existing(int(i))) for i in ids], dtype=bool)]


def visible_chunks(pose: Pose, intr: CameraIntrinsics, extent: ChunkExtent,
                   existing: Callable[[int], bool], cfg: CullConfig, s: float,
                   candidates: Iterable[int] | None = None) -> set[int]:
    """Ids of existing chunks visible from the pose (culling.py:134-182)."""
    ids = _candidates(extent, existing, candidates)
    return {int(i) for i in cull_ids(ids, pose, intr, cfg.max_distance_m, s)}


def _rotation_angle(qa: np.ndarray, qb: np.ndarray) -> float:
    return 2.0 * math.acos(min(1.0, abs(float(np.dot(qa, qb)))))


@dataclass
class _CacheEntry:
    translation: np.ndarray
    rotation: np.ndarray
    intr: CameraIntrinsics
    chunk_size: float
    generation: int
    result: frozenset
    t3: tuple = ()   # translation as Python floats (the query's prefilter)
    r4: tuple = ()   # rotation as Python floats


@dataclass
class VisibilityCache:
    """Pose-quantised LRU over visible_chunks results (culling.py:200-246)."""

    cfg: CullConfig = field(default_factory=CullConfig)
    _entries: list = field(default_factory=list)
    version: int = 0   # bumped by every query (hits reorder the LRU)

    def _match(self, e: _CacheEntry, pose: Pose, intr, generation: int, s: float) -> bool:
        return (e.generation == generation and e.chunk_size == s and e.intr == intr
                and float(np.linalg.norm(e.translation - pose.translation)) < self.cfg.pose_quantum_m
                and _rotation_angle(e.rotation, pose.rotation) < self.cfg.pose_quantum_rad)

    def _match_fast(self, e: _CacheEntry, d: float, qa: tuple, pose: Pose, intr, generation: int,
                    s: float) -> bool:
        """_match's verdict from plain floats when both quantities are clear of
        their thresholds (NumPy's norm / dot differ from these by a few ulp,
        which moves the angle by < 1e-7 rad: far inside the margins), else
        _match itself."""
        if e.generation != generation or e.chunk_size != s or not (e.intr is intr or e.intr == intr):
            return False
        if e.r4 and d < self.cfg.pose_quantum_m * (1 - 1e-9):
            r = e.r4
            dot = abs(((r[0] * qa[0] + r[1] * qa[1]) + r[2] * qa[2]) + r[3] * qa[3])
            ang = 2.0 * math.acos(min(1.0, dot))
            if ang < self.cfg.pose_quantum_rad - 1e-6:
                return True
            if ang > self.cfg.pose_quantum_rad + 1e-6:
                return False
        return self._match(e, pose, intr, generation, s)

    def peek(self, pose: Pose, intr: CameraIntrinsics, generation: int, s: float) -> frozenset | None:
        """The result a query would return from the cache now (None on a
        miss), without touching the LRU order."""
        px, py, pz = (float(v) for v in pose.translation)
        qa = tuple(float(v) for v in pose.rotation)
        lim = self.cfg.pose_quantum_m * (1 + 1e-9) + 1e-300
        for i in range(len(self._entries) - 1, -1, -1):
            e = self._entries[i]
            ex, ey, ez = e.t3
            dx, dy, dz = ex - px, ey - py, ez - pz
            d = math.sqrt((dx * dx + dy * dy) + dz * dz)
            if d < lim and self._match_fast(e, d, qa, pose, intr, generation, s):
                return e.result
        return None

    def query(self, pose: Pose, intr: CameraIntrinsics, extent: ChunkExtent,
              existing: Callable[[int], bool], generation: int, s: float,
              candidates: Iterable[int] | None = None,
              compute: Callable[[], set[int] | None] | None = None) -> tuple[set[int], bool]:
        """compute: on a miss, a caller-held visible set of this very pose and
        chunk set (e.g. computed for a speculative read), else None."""
        # Most recent matching entry, as the reference scan (culling.py:213-229).
        # A vectorised distance prefilter (with a relative margin) limits the
        # exact per-entry test to plausible entries; the verdict is the exact one.
        self.version += 1
        if self._entries:   # newest first; plain-float prefilter (with margin), exact match after
            px, py, pz = (float(v) for v in pose.translation)
            qa = tuple(float(v) for v in pose.rotation)
            lim = self.cfg.pose_quantum_m * (1 + 1e-9) + 1e-300
            for i in range(len(self._entries) - 1, -1, -1):
                e = self._entries[i]
                ex, ey, ez = e.t3
                dx, dy, dz = ex - px, ey - py, ez - pz
                d = math.sqrt((dx * dx + dy * dy) + dz * dz)
                if d >= lim:
                    continue
                if self._match_fast(e, d, qa, pose, intr, generation, s):
                    self._entries.append(self._entries.pop(i))
                    return set(e.result), True
        result = compute() if compute is not None else None
        if result is None:
            if callable(candidates):   # built only on a miss
                candidates = candidates()
            result = visible_chunks(pose, intr, extent, existing, self.cfg, s, candidates)
        self._entries.append(_CacheEntry(pose.translation.copy(), pose.rotation.copy(), intr, s,
                                         generation, frozenset(result),
                                         tuple(float(v) for v in pose.translation),
                                         tuple(float(v) for v in pose.rotation)))
        if len(self._entries) > self.cfg.cache_capacity:
            del self._entries[: len(self._entries) - self.cfg.cache_capacity]
        return set(result), False
