"""The C-ABI library loads and exports every entry point include/splatmap_cuda.h
declares (no device needed: nothing here launches a kernel)."""
import ctypes
import re

import numpy as np
import pytest

from tests.conftest import ROOT

HEADER = ROOT / "include" / "splatmap_cuda.h"


def _declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sm_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ("sm_render_forward", "sm_render_backward", "sm_loss_forward_backward",
                 "sm_adam_step", "sm_cull_chunks", "sm_encode_positions", "sm_chunk_unpack",
                 "sm_chunk_pack", "sm_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2511_23030_b200 import _lib
    lib = _lib.load()
    raw = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in _declared() if not hasattr(raw, n)]
    assert not missing, missing
    assert lib.sm_abi_version() == _lib.ABI_VERSION


def test_workspace_sizing_is_host_only():
    from paper_2511_23030_b200 import _lib
    lib = _lib.load()
    d = _lib.RenderDims(1_000_000, 8_000_000, 640, 480)
    size = lib.sm_render_workspace_size(ctypes.byref(d))
    assert 300e6 < size < 2e9
    assert lib.sm_loss_workspace_size(640, 480) > 12 * 640 * 480 * 4


def test_invalid_arguments_map_to_errors():
    import pytest

    from paper_2511_23030_b200 import _lib
    lib = _lib.load()
    rc = lib.sm_render_forward(None, None, 10, None, None, None, 0, None, None, None, None)
    assert rc == _lib.SM_ERR_INVALID
    assert b"null" in lib.sm_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc, "x")


def test_oracle_library_builds_and_loads():
    from oracle import oracle
    assert oracle.lib().or_render_fwd is not None


def test_no_cpu_fallback_without_a_device():
    """Without a CUDA device the product path raises DeviceFailure: nothing
    silently falls back to a CPU (or oracle) implementation."""
    import torch

    from paper_2511_23030_b200 import renderloss as rl
    from paper_2511_23030_b200.core import CameraIntrinsics, Pose
    from paper_2511_23030_b200.errors import DeviceFailure
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    sa = rl.SceneArrays(np.array([[0.0, 0.0, 2.0]]), np.array([[1.0, 0, 0, 0]]), np.full((1, 3), 0.1),
                        np.array([0.5]), np.zeros((1, 3)))
    with pytest.raises(DeviceFailure):
        rl.render_arrays(sa, Pose(), CameraIntrinsics(fx=40.0, fy=40.0, cx=16, cy=16, width=32, height=32,
                                                      near=0.1))
