"""Splat renderer and loss stack on the B200 (drop-in for splatmap renderloss.py).

Same public names and semantics as the reference module (renderloss.py:22-274):
``RenderedFrame``, ``SceneArrays``, ``scene_arrays``, ``render_arrays``,
``render``, ``LossWeights``, ``ssim``, ``image_loss``, ``depth_loss``,
``total_loss``.  The work runs in libsplatmap_cuda.so (K2-K5 and the fused
loss kernel); the NumPy-in/NumPy-out signatures exist for parity and
compatibility, while the mapping step keeps everything device-resident
(``RenderEngine``).  There is no CPU fallback: without the CUDA library or a
device these raise ``DeviceFailure``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import SH_C0, CameraIntrinsics, Gaussian, Keyframe, Pose, quat_to_matrix
from .errors import DeviceFailure, DimensionMismatch

__all__ = ["RenderedFrame", "SceneArrays", "LossWeights", "render", "render_arrays",
           "scene_arrays", "ssim", "image_loss", "depth_loss", "total_loss", "RenderEngine",
           "LossEngine", "pack_params", "camera_for"]


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise DeviceFailure("no CUDA device: the splat renderer has no CPU fallback")
    return torch


@dataclass
class RenderedFrame:
    rgb: np.ndarray    # (H, W, 3) in [0, 1]
    depth: np.ndarray  # (H, W); 0 where nothing rendered
    alpha: np.ndarray  # (H, W) in [0, 1]


@dataclass
class SceneArrays:
    """Column layout of a splat list (renderloss.py:36-59)."""

    positions: np.ndarray  # (N, 3)
    rotations: np.ndarray  # (N, 4) (w, x, y, z)
    scales: np.ndarray     # (N, 3)
    opacities: np.ndarray  # (N,)
    sh0: np.ndarray        # (N, 3)

    def __len__(self) -> int:
        return int(self.positions.shape[0])

    @staticmethod
    def concatenate(blocks: list["SceneArrays"]) -> "SceneArrays":
        if not blocks:
            return _empty_arrays()
        return SceneArrays(*(np.concatenate([getattr(b, f) for b in blocks]) for f in
                             ("positions", "rotations", "scales", "opacities", "sh0")))


def _empty_arrays() -> SceneArrays:
    return SceneArrays(np.empty((0, 3)), np.empty((0, 4)), np.empty((0, 3)), np.empty(0),
                       np.empty((0, 3)))


def scene_arrays(gaussians: list[Gaussian]) -> SceneArrays:
    if not gaussians:
        return _empty_arrays()
    return SceneArrays(
        positions=np.array([g.position for g in gaussians], dtype=np.float64),
        rotations=np.array([g.rotation for g in gaussians], dtype=np.float64),
        scales=np.array([g.scale for g in gaussians], dtype=np.float64),
        opacities=np.array([g.opacity for g in gaussians], dtype=np.float64),
        sh0=np.array([g.sh[[0, 16, 32]] for g in gaussians], dtype=np.float64),
    )


def pack_params(scene: SceneArrays) -> np.ndarray:
    """SceneArrays -> (N, 16) float32 param records (include/splatmap_cuda.h)."""
    n = len(scene)
    rec = np.zeros((n, _lib.PARAM_STRIDE), dtype=np.float32)
    if n:
        rec[:, 0:3] = scene.positions
        rec[:, 3:7] = scene.rotations
        rec[:, 7:10] = scene.scales
        rec[:, 10] = scene.opacities
        rec[:, 11:14] = scene.sh0
    return rec


def camera_for(pose: Pose, intr: CameraIntrinsics) -> _lib.Camera:
    """sm_camera of a view: the reference's own quat_to_matrix (core.py:88)."""
    return _lib.make_camera(quat_to_matrix(pose.rotation), pose.translation, intr)


class RenderEngine:
    """One render workspace on one device (K2-K5 through the C ABI).

    Capacities grow geometrically; an instance-buffer overflow (flagged on the
    device) is detected with ``check()`` and the render is redone.
    """

    def __init__(self, device=None):
        torch = _torch()
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        self.lib = _lib.load()
        self.dims = _lib.RenderDims(0, 0, 0, 0)
        self.ws = None
        self._ctr = torch.zeros(16, dtype=torch.int32, pin_memory=True)

    def ensure(self, n: int, width: int, height: int, instances: int | None = None) -> None:
        d = self.dims
        grow_g = n > d.max_gaussians
        want_i = instances if instances is not None else 0
        if not grow_g and width == d.width and height == d.height and want_i <= d.max_instances:
            return
        g = max(int(n * 1.25) + 1024, d.max_gaussians if not grow_g else 0, 4096)
        i = max(want_i, d.max_instances, 8 * g, 1 << 20)
        self.dims = _lib.RenderDims(g, i, int(width), int(height))
        size = self.lib.sm_render_workspace_size(ctypes.byref(self.dims))
        self.ws = None
        self.ws = self.torch.empty(int(size), dtype=self.torch.uint8, device=self.device)

    @property
    def ws_bytes(self) -> int:
        return int(self.ws.numel())

    def forward(self, params, slots, n: int, cam: _lib.Camera, rgb, depth, alpha, stream=None,
                tile_order=None):
        """tile_order: optional per-view int32 device tensor (``new_tile_order``)
        carrying the view's longest-first tile schedule from render to render."""
        self.ensure(n, cam.width, cam.height)
        if tile_order is None:
            rc = self.lib.sm_render_forward(_lib.ptr(params), _lib.ptr(slots), int(n), ctypes.byref(cam),
                                            ctypes.byref(self.dims), _lib.ptr(self.ws), self.ws_bytes,
                                            _lib.ptr(rgb), _lib.ptr(depth), _lib.ptr(alpha),
                                            _lib.stream_handle(stream))
        else:
            if tile_order.numel() != self.n_tiles(cam.width, cam.height):
                raise ValueError("tile_order does not match the camera's tile count")
            rc = self.lib.sm_render_forward_ordered(_lib.ptr(params), _lib.ptr(slots), int(n),
                                                    ctypes.byref(cam), ctypes.byref(self.dims),
                                                    _lib.ptr(self.ws), self.ws_bytes, _lib.ptr(tile_order),
                                                    _lib.ptr(rgb), _lib.ptr(depth), _lib.ptr(alpha),
                                                    _lib.stream_handle(stream))
        _lib.check(rc, "render_forward")

    @staticmethod
    def n_tiles(width: int, height: int) -> int:
        return ((width + 15) // 16) * ((height + 15) // 16)

    def new_tile_order(self, width: int, height: int):
        """Identity schedule for a view's first render (device int32)."""
        return self.torch.arange(self.n_tiles(width, height), dtype=self.torch.int32, device=self.device)

    def backward(self, params, slots, n: int, cam: _lib.Camera, d_rgb, d_depth, d_alpha, grads,
                 stream=None):
        rc = self.lib.sm_render_backward(_lib.ptr(params), _lib.ptr(slots), int(n), ctypes.byref(cam),
                                         ctypes.byref(self.dims), _lib.ptr(self.ws), self.ws_bytes,
                                         _lib.ptr(d_rgb), _lib.ptr(d_depth), _lib.ptr(d_alpha),
                                         _lib.ptr(grads), _lib.stream_handle(stream))
        _lib.check(rc, "render_backward")

    def backward_adam(self, params, slots, n: int, cam: _lib.Camera, d_rgb, d_depth, d_alpha, adam_m, adam_v,
                      cfg: _lib.AdamConfig, skip_flag=None, stream=None):
        """Backward with the Adam step fused in (sm_render_backward_adam):
        params / adam_m / adam_v of the active slots are updated in place."""
        rc = self.lib.sm_render_backward_adam(_lib.ptr(params), _lib.ptr(slots), int(n), ctypes.byref(cam),
                                              ctypes.byref(self.dims), _lib.ptr(self.ws), self.ws_bytes,
                                              _lib.ptr(d_rgb), _lib.ptr(d_depth), _lib.ptr(d_alpha),
                                              _lib.ptr(adam_m), _lib.ptr(adam_v), ctypes.byref(cfg),
                                              _lib.ptr(skip_flag), _lib.stream_handle(stream))
        _lib.check(rc, "render_backward_adam")

    def counters_async(self, stream=None):
        """Queue a D2H copy of the workspace counters into pinned memory."""
        src = self.ws[:64].view(self.torch.int32)
        self._ctr.copy_(src, non_blocking=True)
        return self._ctr

    def counters(self) -> dict:
        self.counters_async()
        self.torch.cuda.current_stream().synchronize()
        c = self._ctr.numpy().view(np.uint32)
        return {"n_instances": int(c[0]), "overflow": int(c[1]), "max_instances": self.dims.max_instances}

    def overflow_flag(self):
        """Device uint32 that is non-zero when the last forward overflowed."""
        return self.ws[4:8].view(self.torch.int32)

    def grow_instances(self, needed: int) -> None:
        self.ensure(self.dims.max_gaussians, self.dims.width, self.dims.height,
                    instances=int(needed * 1.3) + 1024)


_engines: dict = {}


def default_engine(device=None) -> RenderEngine:
    torch = _torch()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    eng = _engines.get(str(dev))
    if eng is None:
        eng = _engines[str(dev)] = RenderEngine(dev)
    return eng


def render_device(params, slots, n: int, pose: Pose, intr: CameraIntrinsics, engine=None):
    """Render device-resident param records; returns (rgb, depth, alpha) CUDA tensors."""
    eng = engine or default_engine()
    torch = eng.torch
    h, w = intr.height, intr.width
    rgb = torch.empty((h, w, 3), dtype=torch.float32, device=eng.device)
    depth = torch.empty((h, w), dtype=torch.float32, device=eng.device)
    alpha = torch.empty((h, w), dtype=torch.float32, device=eng.device)
    cam = camera_for(pose, intr)
    for _ in range(8):
        eng.forward(params, slots, n, cam, rgb, depth, alpha)
        c = eng.counters()
        if not c["overflow"]:
            return rgb, depth, alpha
        eng.grow_instances(c["n_instances"])
    raise DeviceFailure("tile-instance buffer kept overflowing")


def render_arrays(scene: SceneArrays, pose: Pose, intr: CameraIntrinsics) -> RenderedFrame:
    """Render RGB, alpha-weighted mean depth and alpha (renderloss.py:170-218)."""
    eng = default_engine()
    torch = eng.torch
    params = torch.from_numpy(pack_params(scene)).to(eng.device)
    rgb, depth, alpha = render_device(params, None, len(scene), pose, intr, eng)
    return RenderedFrame(rgb=rgb.double().cpu().numpy(), depth=depth.double().cpu().numpy(),
                         alpha=alpha.double().cpu().numpy())


def render(gaussians: list[Gaussian], pose: Pose, intr: CameraIntrinsics) -> RenderedFrame:
    return render_arrays(scene_arrays(gaussians), pose, intr)


# ---------------------------------------------------------------------- loss


@dataclass(frozen=True)
class LossWeights:
    lambda_s: float = 0.2
    lambda_depth: float = 0.5

    def __post_init__(self):
        if not 0.0 <= self.lambda_s <= 1.0:
            raise ValueError("lambda_s must be in [0,1]")
        if self.lambda_depth < 0.0:
            raise ValueError("lambda_depth must be >= 0")


class LossEngine:
    """Workspace + outputs of the fused loss kernel on one device."""

    def __init__(self, device=None):
        torch = _torch()
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        self.lib = _lib.load()
        self.wh = (0, 0)
        self.ws = None
        self.out = torch.zeros(4, dtype=torch.float32, device=self.device)

    def ensure(self, width: int, height: int) -> None:
        if (width, height) != self.wh:
            size = self.lib.sm_loss_workspace_size(int(width), int(height))
            self.ws = self.torch.empty(int(size), dtype=self.torch.uint8, device=self.device)
            self.wh = (width, height)

    def run(self, rgb, depth, gt_u8, gt_f32, gt_depth, channels: int, w: LossWeights,
            d_rgb=None, d_depth=None, out=None, stream=None):
        h, wd = int(rgb.shape[0]), int(rgb.shape[1])
        self.ensure(wd, h)
        out = self.out if out is None else out
        rc = self.lib.sm_loss_forward_backward(
            _lib.ptr(rgb), _lib.ptr(depth), _lib.ptr(gt_u8), _lib.ptr(gt_f32), _lib.ptr(gt_depth),
            wd, h, int(channels), float(w.lambda_s), float(w.lambda_depth), _lib.ptr(self.ws),
            int(self.ws.numel()), _lib.ptr(out), _lib.ptr(d_rgb), _lib.ptr(d_depth),
            _lib.stream_handle(stream))
        _lib.check(rc, "loss")
        return out


_loss_engines: dict = {}


def default_loss_engine() -> LossEngine:
    torch = _torch()
    key = torch.cuda.current_device()
    if key not in _loss_engines:
        _loss_engines[key] = LossEngine(torch.device("cuda", key))
    return _loss_engines[key]


def _dev(a, torch, device):
    return torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float32)), device=device)


def _image_terms(a, b, lambda_s: float):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise DimensionMismatch(f"inputs {a.shape} vs {b.shape}")
    if a.ndim not in (2, 3) or min(a.shape[:2]) < 11:
        raise ValueError("ssim needs 2-D or (H, W, C) images of at least 11x11")
    eng = default_loss_engine()
    torch = eng.torch
    c = 1 if a.ndim == 2 else a.shape[2]
    out = eng.run(_dev(a, torch, eng.device), None, None, _dev(b, torch, eng.device), None, c,
                  LossWeights(lambda_s, 0.0))
    return out.cpu().numpy().astype(np.float64)


def ssim(a: np.ndarray, b: np.ndarray) -> float:
    """Mean SSIM, 11x11 Gaussian window sigma 1.5 (renderloss.py:226-248)."""
    return float(_image_terms(a, b, 1.0)[2])


def image_loss(rendered: np.ndarray, gt: np.ndarray, w: LossWeights) -> float:
    """(1 - lambda_s) * L1 + lambda_s * (1 - SSIM) (renderloss.py:251-259)."""
    t = _image_terms(rendered, gt, w.lambda_s)
    return float((1.0 - w.lambda_s) * t[1] + w.lambda_s * (1.0 - t[2]))


def depth_loss(d_rendered: np.ndarray, d_gt: np.ndarray) -> float:
    """Mean |D - Dgt| over pixels with Dgt > 0 (renderloss.py:262-269)."""
    torch = _torch()
    a = torch.as_tensor(np.asarray(d_rendered, dtype=np.float64), device="cuda")
    b = torch.as_tensor(np.asarray(d_gt, dtype=np.float64), device="cuda")
    if a.shape != b.shape:
        raise DimensionMismatch(f"depth_loss inputs {tuple(a.shape)} vs {tuple(b.shape)}")
    valid = b > 0.0
    if not bool(valid.any()):
        return 0.0
    return float((a[valid] - b[valid]).abs().mean())


def total_loss(frame: RenderedFrame, kf: Keyframe, w: LossWeights) -> float:
    """image_loss + lambda_depth * depth_loss against the keyframe (renderloss.py:272-274)."""
    eng = default_loss_engine()
    torch = eng.torch
    rgb = np.asarray(frame.rgb)
    if rgb.shape != kf.rgb.shape or np.asarray(frame.depth).shape != kf.depth.shape:
        raise DimensionMismatch("rendered frame and keyframe differ in shape")
    gt = torch.as_tensor(kf.rgb_u8(), device=eng.device)
    out = eng.run(_dev(rgb, torch, eng.device), _dev(frame.depth, torch, eng.device), gt, None,
                  _dev(kf.depth, torch, eng.device), 3, w)
    return float(out[0].item())
