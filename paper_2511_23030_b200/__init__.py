"""B200-native (sm_100a) mapping hot path of DiskChunGS (arXiv 2511.23030).

Drop-in for the reference ``splatmap`` package's rendering, mapping-step and
chunk-manager API (splatmap/__init__.py:10-40).  The data plane is
libsplatmap_cuda.so (include/splatmap_cuda.h): hand-written CUDA for
projection, depth order + tile binning (radix sort), compositing forward /
backward, the fused loss, fused Adam, chunk culling and the chunk codec.
Host policy (keyframe selection, residency, metrics) is Python, decision-for-
decision identical to the reference.  No CPU fallback: without the library
or a CUDA device, render / loss / store calls raise DeviceFailure.
"""

from .core import (CameraIntrinsics, Gaussian, Keyframe, Pose, RigidTransform, pose_compose,
                   pose_inverse, transform_gaussian)
from .culling import ChunkExtent, CullConfig, Frustum, VisibilityCache, extract_frustum, visible_chunks
from .errors import DeviceFailure, SplatmapError
from .grid import ChunkCoord, assign_gaussians, chunk_aabb, chunk_coord, decode_id, encode_id
from .renderloss import (LossWeights, RenderedFrame, SceneArrays, depth_loss, image_loss, render,
                         render_arrays, scene_arrays, ssim, total_loss)
from .select import KeyframeIndex, SelectConfig, candidate_set, overlap, record_loss, select_keyframe
from .store import ChunkStore, StoreConfig

__version__ = "0.1.0"


def __getattr__(name):   # heavy modules on first use
    if name in ("MappingEngine", "FrameMetrics", "AdamSettings", "METRICS_HEADER"):
        from . import mapping
        return getattr(mapping, name)
    raise AttributeError(name)
