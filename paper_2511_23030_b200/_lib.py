"""ctypes binding of libsplatmap_cuda.so (include/splatmap_cuda.h).

The product path has no CPU fallback: if the shared library is missing or a
CUDA device is absent, every call raises ``DeviceFailure``.  ``load()`` builds
the library in-tree (nvcc, sm_100a) when it is missing and nvcc is present.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_int32, c_int64, c_uint32, c_void_p
from pathlib import Path

import numpy as np

from .errors import CorruptChunk, DeviceFailure, DimensionMismatch, OutOfRange

LIB_PATH = Path(__file__).resolve().parent / "libsplatmap_cuda.so"
if os.environ.get("SM_LIB_VARIANT"):   # A/B experiments: libsplatmap_cuda.<variant>.so next to it
    LIB_PATH = LIB_PATH.with_name(f"libsplatmap_cuda.{os.environ['SM_LIB_VARIANT']}.so")
ABI_VERSION = 1
PARAM_STRIDE = 16
TILE = 16


class Camera(ctypes.Structure):
    _fields_ = [("r_wc", c_double * 9), ("t", c_double * 3), ("fx", c_double), ("fy", c_double),
                ("cx", c_double), ("cy", c_double), ("near_plane", c_double),
                ("far_plane", c_double), ("width", c_int32), ("height", c_int32)]


class RenderDims(ctypes.Structure):
    _fields_ = [("max_gaussians", c_int64), ("max_instances", c_int64), ("width", c_int32),
                ("height", c_int32)]


class RenderCounters(ctypes.Structure):
    _fields_ = [("n_instances", c_uint32), ("overflow", c_uint32), ("n_visible", c_uint32),
                ("n_fallback", c_uint32), ("reserved", c_uint32 * 12)]


class AdamConfig(ctypes.Structure):
    _fields_ = [("lr", c_float * 14), ("beta1", c_float), ("beta2", c_float), ("eps", c_float),
                ("min_scale", c_float)]


SM_OK, SM_ERR_INVALID, SM_ERR_CUDA, SM_ERR_WORKSPACE, SM_ERR_RANGE, SM_ERR_CORRUPT, SM_ERR_DIMENSION = range(7)

_lib = None


def _sig(fn, restype, *argtypes):
    fn.restype = restype
    fn.argtypes = list(argtypes)


def load():
    """Load (building if needed) the CUDA library; raises DeviceFailure otherwise."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        try:
            from .build import build
            build()
        except Exception as exc:  # pragma: no cover - depends on toolchain
            raise DeviceFailure(f"libsplatmap_cuda.so missing and build failed: {exc}") from exc
    try:
        lib = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:
        raise DeviceFailure(f"cannot load {LIB_PATH}: {exc}") from exc
    vp, i64, i32 = c_void_p, c_int64, c_int32
    _sig(lib.sm_abi_version, c_int)
    _sig(lib.sm_last_error, ctypes.c_char_p)
    _sig(lib.sm_device_sm_count, c_int)
    _sig(lib.sm_render_workspace_size, i64, POINTER(RenderDims))
    _sig(lib.sm_render_forward, c_int, vp, vp, i64, POINTER(Camera), POINTER(RenderDims), vp, i64,
         vp, vp, vp, vp)
    _sig(lib.sm_render_forward_ordered, c_int, vp, vp, i64, POINTER(Camera), POINTER(RenderDims), vp,
         i64, vp, vp, vp, vp, vp)
    _sig(lib.sm_render_backward, c_int, vp, vp, i64, POINTER(Camera), POINTER(RenderDims), vp, i64,
         vp, vp, vp, vp, vp)
    _sig(lib.sm_render_backward_adam, c_int, vp, vp, i64, POINTER(Camera), POINTER(RenderDims), vp, i64,
         vp, vp, vp, vp, vp, POINTER(AdamConfig), vp, vp)
    _sig(lib.sm_set_ellipse_cull, None, c_int)
    _sig(lib.sm_render_ws_offset, i64, POINTER(RenderDims), c_int)
    _sig(lib.sm_render_key_layout, c_int, POINTER(RenderDims), POINTER(i32), POINTER(i32))
    _sig(lib.sm_loss_workspace_size, i64, i32, i32)
    _sig(lib.sm_loss_forward_backward, c_int, vp, vp, vp, vp, vp, i32, i32, i32, c_float, c_float,
         vp, i64, vp, vp, vp, vp)
    _sig(lib.sm_adam_step, c_int, vp, vp, vp, vp, vp, i64, POINTER(AdamConfig), vp, vp)
    _sig(lib.sm_pack_grads, c_int, vp, vp, i64, vp, vp)
    _sig(lib.sm_transform_rows, c_int, vp, i64, POINTER(c_double), POINTER(c_double), POINTER(c_double), vp)
    _sig(lib.sm_reset_rows, c_int, vp, vp, vp, i64, c_float, vp)
    _sig(lib.sm_keyframe_pack, c_int, vp, vp, vp, i32, i32, vp, vp)
    _dp = POINTER(c_double)
    _sig(lib.sm_log_scores, c_int, vp, i32, i32, i32, _dp, i32, vp, vp, vp)
    _sig(lib.sm_sampling_probability, c_int, vp, vp, vp, vp, i64, vp, vp)
    _sig(lib.sm_lift_pixels, c_int, vp, i64, vp, vp, i32, i32, i32, _dp, _dp, c_double, c_double, c_double,
         c_double, c_double, c_float, vp, vp, vp)
    _sig(lib.sm_adam_step_packed, c_int, vp, vp, vp, vp, vp, i64, POINTER(AdamConfig), vp, vp)
    _sig(lib.sm_cull_chunks, c_int, vp, i64, POINTER(c_double), POINTER(c_double), c_double,
         c_double, vp, vp)
    _sig(lib.sm_encode_positions, c_int, vp, i64, c_double, vp, vp, vp)
    _sig(lib.sm_expand_segments, c_int, vp, vp, vp, i64, i64, vp, vp)
    _sig(lib.sm_chunk_unpack, c_int, vp, i64, i64, vp, vp, vp, vp, vp, vp)
    _sig(lib.sm_chunk_pack, c_int, vp, vp, vp, vp, i64, i64, vp, vp)
    _sig(lib.sm_profile_enable, None, c_int)
    _sig(lib.sm_launch_count, ctypes.c_longlong)
    _sig(lib.sm_profile_stage_count, c_int)
    _sig(lib.sm_profile_stage_name, ctypes.c_char_p, c_int)
    _sig(lib.sm_profile_collect, c_int, POINTER(c_double), POINTER(ctypes.c_longlong))
    _sig(lib.sm_profile_capture_begin, c_int)
    _sig(lib.sm_profile_capture_end, None)
    _sig(lib.sm_profile_graph_replayed, None, c_int)
    _sig(lib.sm_profile_graph_free, None, c_int)
    _sig(lib.sm_profile_graph_timing_errors, ctypes.c_longlong)
    if lib.sm_abi_version() != ABI_VERSION:
        raise DeviceFailure(f"ABI mismatch: library {lib.sm_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    """Map an SM_ERR_* status to the reference's error vocabulary."""
    if rc == SM_OK:
        return
    msg = (load().sm_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == SM_ERR_DIMENSION:
        raise DimensionMismatch(text)
    if rc == SM_ERR_RANGE:
        raise OutOfRange(text)
    if rc == SM_ERR_CORRUPT:
        raise CorruptChunk(text)
    if rc in (SM_ERR_INVALID, SM_ERR_WORKSPACE):
        raise ValueError(text)
    raise DeviceFailure(text)


def profile_collect() -> dict:
    """{stage: (ms, calls)} since the last collect (blocks on recorded events)."""
    lib = load()
    n = lib.sm_profile_stage_count()
    ms = (c_double * n)()
    calls = (ctypes.c_longlong * n)()
    lib.sm_profile_collect(ms, calls)
    return {lib.sm_profile_stage_name(i).decode(): (ms[i], calls[i]) for i in range(n)}


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    if t is None:
        return None
    return int(t.data_ptr())


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def make_camera(r_wc: np.ndarray, t: np.ndarray, intr) -> Camera:
    cam = Camera()
    r = np.ascontiguousarray(r_wc, dtype=np.float64).reshape(9)
    for k in range(9):
        cam.r_wc[k] = float(r[k])
    for k in range(3):
        cam.t[k] = float(t[k])
    cam.fx, cam.fy, cam.cx, cam.cy = float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy)
    cam.near_plane, cam.far_plane = float(intr.near), float(intr.far)
    cam.width, cam.height = int(intr.width), int(intr.height)
    return cam
