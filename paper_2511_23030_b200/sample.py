"""Edge-driven sampling and depth lifting on the B200 (drop-in for splatmap sample.py).

Same public names and semantics as the reference module (sample.py:1-146):
``SampleConfig``, ``log_kernel``, ``log_norm``, ``sampling_probability``,
``sample_pixels``, ``lift_to_gaussians``.  The per-pixel work -- the |LoG|
scores of the luma image, their max-normalisation and the clamped
difference, and the unprojection of sampled pixels -- runs in
libsplatmap_cuda.so (csrc/ingest.cu, fp64 like the reference).  The draw
itself stays on the host: ``sample_pixels`` is NumPy's
``Generator.choice(replace=False, p=...)`` exactly as the reference calls it
(sample.py:87-101), which has no bit-reproducible device form.

``DeviceSampler`` keeps a keyframe ingest on the device end to end
(MappingEngine.ingest_keyframe): the keyframe's 8-bit ground truth and the
current render never leave HBM; only the probability map crosses to the host
for the draw and the drawn pixels come back.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import CameraIntrinsics, Gaussian, Keyframe, quat_to_matrix, unchecked_gaussian
from .errors import DeviceFailure, DimensionMismatch

__all__ = ["SampleConfig", "log_kernel", "log_norm", "sampling_probability", "sample_pixels",
           "lift_to_gaussians", "DeviceSampler"]

RGB_U8, RGB_F32, RGB_F64 = 0, 1, 2


@dataclass(frozen=True)
class SampleConfig:
    log_sigma: float = 1.0
    kernel_radius: int = 2
    samples_per_keyframe: int = 2000
    init_scale_factor: float = 1.0
    init_opacity: float = 0.1

    def __post_init__(self):
        if min(self.log_sigma, self.kernel_radius, self.samples_per_keyframe, self.init_scale_factor) <= 0:
            raise ValueError("sampling parameters must be positive")
        if not (0.0 < self.init_opacity <= 1.0):
            raise ValueError("init_opacity must be in (0,1]")


def log_kernel(sigma: float, radius: int) -> np.ndarray:
    """(2r+1)^2 Laplacian-of-Gaussian taps, shifted to zero sum (sample.py:49-60)."""
    ax = np.arange(-radius, radius + 1, dtype=np.float64)
    xx, yy = np.meshgrid(ax, ax)
    r2 = xx * xx + yy * yy
    s2 = sigma * sigma
    k = (r2 - 2.0 * s2) * np.exp(-r2 / (2.0 * s2))
    return k - k.mean()


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise DeviceFailure("no CUDA device: the sampling kernels have no CPU fallback")
    return torch


def _kind(t) -> int:
    torch = _torch()
    return {torch.uint8: RGB_U8, torch.float32: RGB_F32, torch.float64: RGB_F64}[t.dtype]


class DeviceSampler:
    """Workspace of the device ingest kernels for one image size."""

    def __init__(self, width: int, height: int, device=None):
        torch = _torch()
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        self.lib = _lib.load()
        self.w, self.h = int(width), int(height)
        n = self.w * self.h
        self.scores = torch.empty((2, n), dtype=torch.float64, device=self.device)
        self.peaks = torch.zeros(2, dtype=torch.int64, device=self.device)
        self.ps = torch.empty(n, dtype=torch.float64, device=self.device)
        self._taps = {}

    def _taps_for(self, sigma: float, radius: int):
        key = (float(sigma), int(radius))
        t = self._taps.get(key)
        if t is None:
            k = np.ascontiguousarray(log_kernel(sigma, radius).reshape(-1), dtype=np.float64)
            t = self._taps[key] = k
        return t

    def scores_of(self, rgb, slot: int, sigma: float, radius: int) -> None:
        """|LoG| scores of a device (H, W, 3) image into scores[slot] + peaks[slot]."""
        if tuple(rgb.shape) != (self.h, self.w, 3):
            raise DimensionMismatch(f"expected {self.h}x{self.w}x3 image, got {tuple(rgb.shape)}")
        taps = self._taps_for(sigma, radius)
        rc = self.lib.sm_log_scores(_lib.ptr(rgb), _kind(rgb), self.w, self.h,
                                    taps.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(radius),
                                    _lib.ptr(self.scores[slot]), _lib.ptr(self.peaks[slot:slot + 1]),
                                    _lib.stream_handle())
        _lib.check(rc, "log_scores")

    def probability(self, with_rendered: bool = True):
        """ps = max(log_norm(input) - log_norm(rendered), 0) (or log_norm(input))."""
        n = self.w * self.h
        b = self.scores[1] if with_rendered else None
        pb = self.peaks[1:2] if with_rendered else None
        rc = self.lib.sm_sampling_probability(_lib.ptr(self.scores[0]), _lib.ptr(self.peaks[0:1]), _lib.ptr(b),
                                              _lib.ptr(pb), n, _lib.ptr(self.ps), _lib.stream_handle())
        _lib.check(rc, "sampling_probability")
        return self.ps.view(self.h, self.w)

    def lift(self, pixels: np.ndarray, depth, rgb, pose_rotation, pose_translation, intr: CameraIntrinsics,
             cfg: SampleConfig):
        """Device lift of (k, 2) (row, col) pixels; returns (records (m, 16) f32
        numpy, kept pixel indices) for the pixels with depth > 0, in order."""
        torch = self.torch
        px = np.asarray(pixels, dtype=np.int64).reshape(-1, 2)
        k = px.shape[0]
        if k == 0:
            return np.zeros((0, 16), np.float32), np.zeros(0, np.int64)
        rows, cols = px[:, 0], px[:, 1]
        ok = (rows >= 0) & (rows < intr.height) & (cols >= 0) & (cols < intr.width)
        if not ok.all():
            bad = int(np.flatnonzero(~ok)[0])
            raise ValueError(f"pixel ({rows[bad]},{cols[bad]}) out of bounds")
        pix = torch.as_tensor(px.astype(np.int32), device=self.device)
        rec = torch.empty((k, 16), dtype=torch.float32, device=self.device)
        valid = torch.empty(k, dtype=torch.int32, device=self.device)
        r = np.ascontiguousarray(quat_to_matrix(pose_rotation), dtype=np.float64).reshape(-1)
        t = np.ascontiguousarray(pose_translation, dtype=np.float64).reshape(3)
        dp = ctypes.POINTER(ctypes.c_double)
        rc = self.lib.sm_lift_pixels(_lib.ptr(pix), k, _lib.ptr(depth), _lib.ptr(rgb), _kind(rgb), self.w, self.h,
                                     r.ctypes.data_as(dp), t.ctypes.data_as(dp), float(intr.fx), float(intr.fy),
                                     float(intr.cx), float(intr.cy), float(cfg.init_scale_factor),
                                     float(np.float32(cfg.init_opacity)), _lib.ptr(rec), _lib.ptr(valid),
                                     _lib.stream_handle())
        _lib.check(rc, "lift_pixels")
        keep = np.flatnonzero(valid.cpu().numpy() != 0)
        return rec.cpu().numpy()[keep], keep


_samplers: dict = {}


def _sampler(w: int, h: int) -> DeviceSampler:
    torch = _torch()
    key = (w, h, torch.cuda.current_device())
    s = _samplers.get(key)
    if s is None:
        s = _samplers[key] = DeviceSampler(w, h, torch.device("cuda", key[2]))
    return s


def _image(rgb):
    img = np.asarray(rgb, dtype=np.float64)
    if img.ndim != 3 or img.shape[2] != 3:
        raise DimensionMismatch(f"expected HxWx3 image, got {img.shape}")
    return img


def log_norm(rgb: np.ndarray, sigma: float = 1.0, radius: int = 2) -> np.ndarray:
    """|LoG| of the luma image, max-normalised to [0,1] unless all-zero (sample.py:63-75)."""
    img = _image(rgb)
    h, w = img.shape[:2]
    s = _sampler(w, h)
    s.scores_of(s.torch.as_tensor(np.ascontiguousarray(img), device=s.device), 0, sigma, radius)
    return s.probability(with_rendered=False).cpu().numpy().copy()


def sampling_probability(p_input: np.ndarray, p_rendered: np.ndarray) -> np.ndarray:
    """Per-pixel max(p_input - p_rendered, 0) (sample.py:78-84) on the device."""
    a = np.asarray(p_input, dtype=np.float64)
    b = np.asarray(p_rendered, dtype=np.float64)
    if a.shape != b.shape:
        raise DimensionMismatch(f"score maps {a.shape} vs {b.shape}")
    if a.ndim != 2:
        raise DimensionMismatch(f"expected 2-D score maps, got {a.shape}")
    h, w = a.shape
    s = _sampler(w, h)
    torch = s.torch
    s.scores[0].copy_(torch.as_tensor(a.reshape(-1)))
    s.scores[1].copy_(torch.as_tensor(b.reshape(-1)))
    s.peaks.zero_()   # peak 0: the maps are taken as they are (already normalised)
    return s.probability().cpu().numpy().copy()


def sample_pixels(ps: np.ndarray, n: int, rng_seed: int) -> list[tuple[int, int]]:
    """Draw up to n distinct pixels with probability proportional to ps
    (sample.py:87-101, the same NumPy draw: host policy)."""
    if n < 0:
        raise ValueError("n must be >= 0")
    ps = np.asarray(ps, dtype=np.float64)
    flat = ps.reshape(-1)
    total = flat.sum()
    positive = int(np.count_nonzero(flat > 0))
    k = min(n, positive)
    if k == 0 or total <= 0.0:
        return []
    rng = np.random.default_rng(rng_seed)
    chosen = rng.choice(flat.size, size=k, replace=False, p=flat / total)
    w = ps.shape[1]
    return [(int(i) // w, int(i) % w) for i in chosen]


def lift_to_gaussians(pixels: list[tuple[int, int]], kf: Keyframe, cfg: SampleConfig) -> list[Gaussian]:
    """Unproject sampled pixels with valid depth into world-space Gaussians
    (sample.py:104-146) with the device lift kernel."""
    intr = kf.intrinsics
    if not pixels:
        return []
    s = _sampler(intr.width, intr.height)
    torch = s.torch
    rec, _ = s.lift(pixels, torch.as_tensor(kf.depth, device=s.device),
                    torch.as_tensor(kf.rgb_u8(), device=s.device), kf.pose.rotation, kf.pose.translation,
                    intr, cfg)
    out = []
    for r in rec.astype(np.float64):
        sh = np.zeros(48)
        sh[[0, 16, 32]] = r[11:14]
        out.append(unchecked_gaussian(r[0:3].copy(), r[3:7].copy(), r[7:10].copy(), float(r[10]), sh))
    return out
