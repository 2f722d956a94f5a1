"""ctypes front-end of the CPU checker (oracle/render_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg, never by the product
package.  Every function mirrors a reference function (cited) on NumPy fp64
arrays:

* ``render_arrays``  -> splatmap renderloss.py:170-218 (+ _composite 106-152)
* ``render_backward`` -> (absent in the reference) reverse-order backward of
  the same forward; pinned by finite differences of the reference forward
  (tests/golden/render_fd.npz).
* ``total_loss``     -> renderloss.py:226-274, optional dL/d(rgb, depth)
* ``adam``           -> torch.optim.Adam formula (the reference has no Adam)
* ``bin_tiles``      -> the device's K2/K3 arithmetic (oracle/bin_oracle.c):
  depth order (renderloss.py:202), 3-sigma boxes (renderloss.py:122-135),
  tile-sorted (tile, rank) instance keys and per-tile ranges, bit-exact.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build() -> Path:
    """Compile the checker in place (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(_LIB_PATH))
        _lib.or_render_fwd.restype = ctypes.c_int
        _lib.or_render_fwd.argtypes = (
            [ctypes.c_int64] + [_dp] * 7 + [ctypes.c_double] * 5 + [ctypes.c_int] * 2
            + [_dp] * 3 + [_i64p, ctypes.c_int])
        _lib.or_render_bwd.restype = ctypes.c_int
        _lib.or_render_bwd.argtypes = (
            [ctypes.c_int64] + [_dp] * 7 + [ctypes.c_double] * 5 + [ctypes.c_int] * 2
            + [_dp] * 3 + [_dp] * 5 + [ctypes.c_int])
        _lib.or_total_loss.restype = ctypes.c_double
        _lib.or_total_loss.argtypes = [_dp] * 4 + [ctypes.c_int] * 2 + [ctypes.c_double] * 2 + [_dp] * 2
        _lib.or_train_step.restype = ctypes.c_double
        _lib.or_train_step.argtypes = (
            [ctypes.c_int64] + [_dp] * 7 + [ctypes.c_double] * 5 + [ctypes.c_int] * 2 + [_dp] * 2
            + [ctypes.c_double] * 2 + [_dp] + [ctypes.c_double] * 4 + [_dp] * 2 + [_i64p, ctypes.c_int])
        _lib.ob_bin_tiles.restype = ctypes.c_int64
        _lib.ob_bin_tiles.argtypes = (
            [ctypes.c_int64, ctypes.POINTER(ctypes.c_float), _dp, _dp] + [ctypes.c_double] * 5
            + [ctypes.c_int] * 4 + [_i64p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int64,
                                     ctypes.POINTER(ctypes.c_uint32)])
        _lib.or_adam.restype = None
        _lib.or_adam.argtypes = ([ctypes.c_int64] + [_dp] * 4 + [ctypes.c_double] * 4
                                 + [ctypes.c_int64])
    return _lib


def _c(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


def default_threads() -> int:
    return int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1))


def quat_to_matrix(q) -> np.ndarray:
    """core.py:88-97 rotation matrix of a (w, x, y, z) quaternion."""
    w, x, y, z = (float(v) for v in q)
    return np.array(
        [
            [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
            [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
            [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
        ]
    )


def _scene_args(positions, rotations, scales, opacities, sh0):
    pos = _c(positions, (-1, 3))
    n = pos.shape[0]
    return n, pos, _c(rotations, (n, 4)), _c(scales, (n, 3)), _c(opacities, (n,)), _c(sh0, (n, 3))


def render_arrays(positions, rotations, scales, opacities, sh0, pose_rotation, pose_translation,
                  fx, fy, cx, cy, near, width, height, threads=None, return_pairs=False):
    """fp64 restatement of renderloss.render_arrays; returns (rgb, depth, alpha)."""
    n, pos, rot, sc, op, sh = _scene_args(positions, rotations, scales, opacities, sh0)
    r_wc = _c(quat_to_matrix(pose_rotation))
    t = _c(pose_translation, (3,))
    rgb = np.zeros((height, width, 3))
    depth = np.zeros((height, width))
    alpha = np.zeros((height, width))
    pairs = ctypes.c_int64(0)
    rc = lib().or_render_fwd(n, _p(pos), _p(rot), _p(sc), _p(op), _p(sh), _p(r_wc), _p(t),
                             fx, fy, cx, cy, near, width, height, _p(rgb), _p(depth), _p(alpha),
                             ctypes.byref(pairs), threads or default_threads())
    if rc:
        raise MemoryError("oracle render failed")
    if return_pairs:
        return rgb, depth, alpha, int(pairs.value)
    return rgb, depth, alpha


def render_backward(positions, rotations, scales, opacities, sh0, pose_rotation, pose_translation,
                    fx, fy, cx, cy, near, width, height, d_rgb=None, d_depth=None, d_alpha=None,
                    threads=None):
    """Analytic gradient of <d_rgb,rgb> + <d_depth,depth> + <d_alpha,alpha>.

    Returns dict of fp64 arrays: positions (n,3), rotations (n,4), scales (n,3),
    opacities (n,), sh0 (n,3).
    """
    n, pos, rot, sc, op, sh = _scene_args(positions, rotations, scales, opacities, sh0)
    r_wc = _c(quat_to_matrix(pose_rotation))
    t = _c(pose_translation, (3,))
    dr = None if d_rgb is None else _c(d_rgb, (height, width, 3))
    dd = None if d_depth is None else _c(d_depth, (height, width))
    da = None if d_alpha is None else _c(d_alpha, (height, width))
    out = {
        "positions": np.zeros((n, 3)), "rotations": np.zeros((n, 4)), "scales": np.zeros((n, 3)),
        "opacities": np.zeros(n), "sh0": np.zeros((n, 3)),
    }
    rc = lib().or_render_bwd(n, _p(pos), _p(rot), _p(sc), _p(op), _p(sh), _p(r_wc), _p(t),
                             fx, fy, cx, cy, near, width, height, _p(dr), _p(dd), _p(da),
                             _p(out["positions"]), _p(out["rotations"]), _p(out["scales"]),
                             _p(out["opacities"]), _p(out["sh0"]), threads or default_threads())
    if rc:
        raise MemoryError("oracle backward failed")
    return out


def total_loss(rgb, depth, gt_rgb, gt_depth, lambda_s=0.2, lambda_depth=0.5, grad=False):
    """renderloss.total_loss on arrays; with grad=True also (d_rgb, d_depth)."""
    rgb = _c(rgb)
    h, w = rgb.shape[:2]
    depth = _c(depth, (h, w))
    gt_rgb = _c(gt_rgb, (h, w, 3))
    gt_depth = _c(gt_depth, (h, w))
    if grad:
        d_rgb = np.zeros((h, w, 3))
        d_depth = np.zeros((h, w))
        val = lib().or_total_loss(_p(rgb), _p(depth), _p(gt_rgb), _p(gt_depth), h, w,
                                  lambda_s, lambda_depth, _p(d_rgb), _p(d_depth))
        return float(val), d_rgb, d_depth
    return float(lib().or_total_loss(_p(rgb), _p(depth), _p(gt_rgb), _p(gt_depth), h, w,
                                     lambda_s, lambda_depth, None, None))


class TrainState:
    """fp64 copy of a scene + per-Gaussian Adam state for or_train_step."""

    def __init__(self, positions, rotations, scales, opacities, sh0):
        n, self.pos, self.rot, self.scale, self.opac, self.sh0 = _scene_args(
            positions, rotations, scales, opacities, sh0)
        self.pos, self.rot, self.scale = self.pos.copy(), self.rot.copy(), self.scale.copy()
        self.opac, self.sh0 = self.opac.copy(), self.sh0.copy()
        self.n = n
        self.m = np.zeros((n, 14))
        self.v = np.zeros((n, 14))
        self.steps = np.zeros(n, dtype=np.int64)

    FIELDS = ("pos", "rot", "scale", "opac", "sh0", "m", "v", "steps")

    def step(self, pose_rotation, pose_translation, intr, gt_rgb, gt_depth, lambda_s, lambda_depth,
             lr14, beta1, beta2, eps, min_scale, threads=None, subset=None) -> float:
        """One CPU mapping iteration (fwd, loss+grad, bwd, Adam); returns the loss.

        subset: optional index array of the active set (sim.py:236-253 order);
        only those Gaussians are rendered and updated.
        """
        r_wc = _c(quat_to_matrix(pose_rotation))
        t = _c(pose_translation, (3,))
        h, w = intr.height, intr.width
        gt = _c(gt_rgb, (h, w, 3))
        gd = _c(gt_depth, (h, w))
        lr = _c(lr14, (14,))
        if subset is None:
            a = {f: getattr(self, f) for f in self.FIELDS}
            n = self.n
        else:
            a = {f: np.ascontiguousarray(getattr(self, f)[subset]) for f in self.FIELDS}
            n = len(subset)
        loss = float(lib().or_train_step(
            n, _p(a["pos"]), _p(a["rot"]), _p(a["scale"]), _p(a["opac"]), _p(a["sh0"]), _p(r_wc),
            _p(t), intr.fx, intr.fy, intr.cx, intr.cy, intr.near, w, h, _p(gt), _p(gd), lambda_s,
            lambda_depth, _p(lr), beta1, beta2, eps, min_scale, _p(a["m"]), _p(a["v"]),
            a["steps"].ctypes.data_as(_i64p), threads or default_threads()))
        if subset is not None:
            for f in self.FIELDS:
                getattr(self, f)[subset] = a[f]
        return loss


def frustum_planes(pose_rotation, pose_translation, intr) -> np.ndarray:
    """culling.py:80-101 extract_frustum (same NumPy expression sequence)."""
    w, h = float(intr.width), float(intr.height)
    cams = [(np.array([0.0, 0.0, 1.0]), -intr.near), (np.array([0.0, 0.0, -1.0]), intr.far),
            (np.array([intr.fx, 0.0, intr.cx]), 0.0), (np.array([-intr.fx, 0.0, w - intr.cx]), 0.0),
            (np.array([0.0, intr.fy, intr.cy]), 0.0), (np.array([0.0, -intr.fy, h - intr.cy]), 0.0)]
    r = quat_to_matrix(pose_rotation)
    t = np.asarray(pose_translation, dtype=np.float64)
    rows = []
    for n, d in cams:
        nw = r @ (n / np.linalg.norm(n))
        rows.append([*nw, d - float(nw @ t)])
    return np.array(rows)


def visible_chunk_mask(coords, pose_rotation, pose_translation, intr, max_distance, s) -> np.ndarray:
    """Brute-force chunk visibility (culling.py:104-131; the reference's own
    test oracle, test_acceptance.py:74-95): p-vertex outside test + nearest
    AABB point distance, vectorised over an (M, 3) integer coord table."""
    coords = np.asarray(coords, dtype=np.float64)
    planes = frustum_planes(pose_rotation, pose_translation, intr)
    cam = np.asarray(pose_translation, dtype=np.float64)
    mins, maxs = coords * s - s / 2.0, coords * s + s / 2.0
    outside = np.zeros(len(coords), dtype=bool)
    for nx, ny, nz, d in planes:
        px = np.where(nx >= 0, maxs[:, 0], mins[:, 0])
        py = np.where(ny >= 0, maxs[:, 1], mins[:, 1])
        pz = np.where(nz >= 0, maxs[:, 2], mins[:, 2])
        outside |= (nx * px + ny * py + nz * pz + d) < 0.0
    nearest = np.clip(cam, mins, maxs)
    dist = np.sqrt(((cam - nearest) ** 2).sum(axis=1))
    return ~outside & (dist <= max_distance)


def chunk_ids(positions, s) -> np.ndarray:
    """grid.py:110-121 encode_positions."""
    c = np.floor((np.asarray(positions, dtype=np.float64) + s / 2.0) / s)
    u = (c + float(1 << 20)).astype(np.uint64)
    return (u[:, 0] << np.uint64(42)) | (u[:, 1] << np.uint64(21)) | u[:, 2]


def active_set(positions, pose_rotation, pose_translation, intr, max_distance, s) -> np.ndarray:
    """Indices of the Gaussians in visible chunks, in sorted-chunk-id order
    (stable within a chunk) -- the SoA concatenation of sim.py:236-253."""
    ids = chunk_ids(positions, s)
    uniq, inv = np.unique(ids, return_inverse=True)
    m = np.uint64((1 << 21) - 1)
    coords = np.stack([(uniq >> np.uint64(42)) & m, (uniq >> np.uint64(21)) & m, uniq & m], 1)
    coords = coords.astype(np.int64) - (1 << 20)
    vis = visible_chunk_mask(coords, pose_rotation, pose_translation, intr, max_distance, s)
    keep = vis[inv]
    order = np.argsort(ids, kind="stable")
    return order[keep[order]]


def adam(param, m, v, grad, lr, beta1, beta2, eps, step):
    """In-place torch.optim.Adam step on fp64 flat arrays (step = post-increment count)."""
    for a in (param, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    g = _c(grad)
    lib().or_adam(param.size, _p(param), _p(m), _p(v), _p(g), lr, beta1, beta2, eps, int(step))


def bin_tiles(params, pose_rotation, pose_translation, fx, fy, cx, cy, near, width, height,
              ellipse_cull=True, rank_bits=None):
    """K2/K3 restatement on float32 param records (n, 16).

    Returns (order, keys, ranges): order[rank] = index (np.argsort(z,
    kind="stable") over the kept set, culled after); keys = sorted uint64
    (tile << rank_bits) | rank; ranges = uint32 (tiles, 2) [start, end).
    """
    p = np.ascontiguousarray(np.asarray(params, dtype=np.float32).reshape(-1, 16))
    n = p.shape[0]
    if rank_bits is None:
        rank_bits = max(1, int(np.ceil(np.log2(max(n, 2)))))
    r_wc = _c(quat_to_matrix(pose_rotation))
    t = _c(pose_translation, (3,))
    tiles = ((width + 15) // 16) * ((height + 15) // 16)
    order = np.zeros(max(n, 1), dtype=np.int64)
    ranges = np.zeros((tiles, 2), dtype=np.uint32)
    cap = max(16 * n, 1024)
    while True:
        keys = np.zeros(cap, dtype=np.uint64)
        cnt = lib().ob_bin_tiles(n, p.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), _p(r_wc), _p(t),
                                 fx, fy, cx, cy, near, int(width), int(height), int(bool(ellipse_cull)),
                                 int(rank_bits), order.ctypes.data_as(_i64p),
                                 keys.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), cap,
                                 ranges.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
        if cnt < 0:
            raise MemoryError("oracle binning failed")
        if cnt <= cap:
            return order[:n], keys[:cnt], ranges
        cap = int(cnt)
