"""On-disk .dcg / .dkf formats (splatmap diskformat.py:1-250), little-endian.

Chunk file: "DCG1" | version u32 | id u64 | count u64 | reserved u64, then
per Gaussian a 240-byte record <3f4f3ff48fI> (position, rotation wxyz, scale,
opacity, 48 SH, opt_state length) followed by the opt_state bytes.
Keyframe file: <4sIQ7d6dIIdI> header (140 B), RGB u8, depth f32.

The host functions here are the reference-compatible codec on Gaussian
objects.  The store's bulk path parses and builds whole chunk files as NumPy
record arrays and runs the field shuffle on the GPU (K8/K9,
sm_chunk_unpack / sm_chunk_pack); ``parse_chunk_records`` /
``build_chunk_file`` are that path's host halves.  Adam state rides in
opt_state as a 120-byte tail "ADM1" | step u32 | m[14] f32 | v[14] f32;
b"" means fresh state (loopclose.py:241 contract).
"""

from __future__ import annotations

import struct

import numpy as np

from .core import CameraIntrinsics, Gaussian, Keyframe, Pose, unchecked_gaussian, validate_gaussian_arrays
from .errors import CorruptChunk

__all__ = ["CHUNK_MAGIC", "KEYFRAME_MAGIC", "FORMAT_VERSION", "RECORD_DTYPE", "ADAM_TAIL",
           "storage_canonical", "storage_canonical_batch", "pack_chunk", "unpack_chunk",
           "read_chunk_header", "pack_keyframe", "unpack_keyframe", "parse_chunk_records",
           "build_chunk_file"]

CHUNK_MAGIC = b"DCG1"
KEYFRAME_MAGIC = b"DKF1"
FORMAT_VERSION = 1
ADAM_TAIL = 120
ADAM_MAGIC = b"ADM1"

_HDR = struct.Struct("<4sIQQQ")
_REC = struct.Struct("<3f4f3ff48fI")
_KF = struct.Struct("<4sIQ7d6dIIdI")

RECORD_DTYPE = np.dtype([("position", "<f4", (3,)), ("rotation", "<f4", (4,)),
                         ("scale", "<f4", (3,)), ("opacity", "<f4"), ("sh", "<f4", (48,)),
                         ("opt_len", "<u4")])
assert RECORD_DTYPE.itemsize == 240
_ADAM_DTYPE = np.dtype(RECORD_DTYPE.descr + [("tail", "V120")])
assert _ADAM_DTYPE.itemsize == 360


def _f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def storage_canonical(g: Gaussian) -> Gaussian:
    """Quantise through float32 (a fixed point of pack/unpack)."""
    return Gaussian(position=_f32(g.position), rotation=_f32(g.rotation), scale=_f32(g.scale),
                    opacity=float(np.float32(g.opacity)), sh=_f32(g.sh), opt_state=g.opt_state)


def storage_canonical_batch(gs: list[Gaussian]) -> list[Gaussian]:
    if not gs:
        return []
    pos = _f32([g.position for g in gs])
    rot = _f32([g.rotation for g in gs])
    sc = _f32([g.scale for g in gs])
    op = np.array([g.opacity for g in gs], dtype=np.float32).astype(np.float64)
    sh = _f32([g.sh for g in gs])
    validate_gaussian_arrays(pos, rot, sc, op, sh)
    return [unchecked_gaussian(pos[i], rot[i], sc[i], float(op[i]), sh[i], gs[i].opt_state)
            for i in range(len(gs))]


def pack_chunk(encoded_id: int, gaussians: list[Gaussian]) -> bytes:
    head = _HDR.pack(CHUNK_MAGIC, FORMAT_VERSION, encoded_id, len(gaussians), 0)
    if gaussians and not any(g.opt_state for g in gaussians):
        rec = np.zeros(len(gaussians), dtype=RECORD_DTYPE)
        rec["position"] = [g.position for g in gaussians]
        rec["rotation"] = [g.rotation for g in gaussians]
        rec["scale"] = [g.scale for g in gaussians]
        rec["opacity"] = [g.opacity for g in gaussians]
        rec["sh"] = [g.sh for g in gaussians]
        return head + rec.tobytes()
    out = [head]
    for g in gaussians:
        out.append(_REC.pack(*np.asarray(g.position, np.float32), *np.asarray(g.rotation, np.float32),
                             *np.asarray(g.scale, np.float32), np.float32(g.opacity),
                             *np.asarray(g.sh, np.float32), len(g.opt_state)))
        out.append(g.opt_state)
    return b"".join(out)


def _header(data: bytes, magic: bytes, size: int, kind: str) -> None:
    if len(data) < size:
        raise CorruptChunk(f"{kind} file truncated before header end")
    if bytes(data[:4]) != magic:
        raise CorruptChunk(f"bad {kind} magic {data[:4]!r}")


def read_chunk_header(data: bytes) -> tuple[int, int]:
    _header(data, CHUNK_MAGIC, _HDR.size, "chunk")
    _, version, cid, count, _ = _HDR.unpack_from(data, 0)
    if version != FORMAT_VERSION:
        raise CorruptChunk(f"unsupported chunk format version {version}")
    return cid, count


def parse_chunk_records(data: bytes) -> tuple[int, int, np.ndarray | None, int]:
    """(id, count, uniform-stride record view or None, stride).

    Returns a zero-copy view when every record has the same opt_state length
    of 0 or ADAM_TAIL (the device codec's two layouts); otherwise None and
    the caller takes the per-record host path.
    """
    cid, count = read_chunk_header(data)
    payload = len(data) - _HDR.size
    for stride, dt in ((240, RECORD_DTYPE), (360, _ADAM_DTYPE)):
        if payload == count * stride:
            if count == 0:
                return cid, 0, np.zeros(0, dtype=dt), stride
            arr = np.frombuffer(data, dtype=dt, count=count, offset=_HDR.size)
            if (arr["opt_len"] == stride - 240).all():
                return cid, count, arr, stride
    return cid, count, None, 0


def unpack_chunk(data: bytes) -> tuple[int, list[Gaussian]]:
    cid, count = read_chunk_header(data)
    body = memoryview(data)[_HDR.size:]
    try:
        if len(body) == count * 240:
            arr = np.frombuffer(body, dtype=RECORD_DTYPE)
            if count == 0 or not arr["opt_len"].any():
                pos, rot = arr["position"].astype(np.float64), arr["rotation"].astype(np.float64)
                sc, op = arr["scale"].astype(np.float64), arr["opacity"].astype(np.float64)
                sh = arr["sh"].astype(np.float64)
                validate_gaussian_arrays(pos, rot, sc, op, sh)
                return cid, [unchecked_gaussian(pos[i], rot[i], sc[i], float(op[i]), sh[i])
                             for i in range(count)]
        out, off = [], 0
        for _ in range(count):
            if off + _REC.size > len(body):
                raise CorruptChunk("chunk record truncated")
            f = _REC.unpack_from(body, off)
            off += _REC.size
            n = f[-1]
            if off + n > len(body):
                raise CorruptChunk("chunk opt_state truncated")
            opt = bytes(body[off:off + n])
            off += n
            out.append(Gaussian(position=np.array(f[0:3], np.float64), rotation=np.array(f[3:7], np.float64),
                                scale=np.array(f[7:10], np.float64), opacity=float(f[10]),
                                sh=np.array(f[11:59], np.float64), opt_state=opt))
        if off != len(body):
            raise CorruptChunk("chunk file has trailing bytes")
        return cid, out
    except ValueError as exc:
        raise CorruptChunk(f"chunk record fails invariants: {exc}") from exc


def build_chunk_file(encoded_id: int, records: np.ndarray, count: int | None = None) -> bytes:
    """Header + packed records (240- or 360-byte stride): a structured record
    array, or raw bytes from K9 with an explicit record `count`."""
    n = len(records) if count is None else int(count)
    return _HDR.pack(CHUNK_MAGIC, FORMAT_VERSION, encoded_id, n, 0) + records.tobytes()


def keyframe_header(kf: Keyframe) -> bytes:
    """The 140-byte .dkf header (<4sIQ7d6dIIdI, diskformat.py:53,198-212)."""
    i = kf.intrinsics
    return _KF.pack(KEYFRAME_MAGIC, FORMAT_VERSION, kf.id, *kf.pose.translation, *kf.pose.rotation,
                    i.fx, i.fy, i.cx, i.cy, i.near, i.far, i.width, i.height, kf.last_loss,
                    kf.usage_remaining)


def pack_keyframe(kf: Keyframe) -> bytes:
    return keyframe_header(kf) + kf.rgb_u8().tobytes() + kf.depth.astype("<f4").tobytes()


def keyframe_file_size(kf: Keyframe) -> int:
    return _KF.size + kf.intrinsics.width * kf.intrinsics.height * 7


def unpack_keyframe(data: bytes) -> Keyframe:
    _header(data, KEYFRAME_MAGIC, _KF.size, "keyframe")
    f = _KF.unpack_from(data, 0)
    if f[1] != FORMAT_VERSION:
        raise CorruptChunk(f"unsupported keyframe format version {f[1]}")
    tx, ty, tz, qw, qx, qy, qz = f[3:10]
    fx, fy, cx, cy, near, far = f[10:16]
    w, h = f[16], f[17]
    if len(data) != _KF.size + h * w * 7:
        raise CorruptChunk("keyframe payload truncated or oversized")
    rgb = np.frombuffer(data, np.uint8, h * w * 3, _KF.size).reshape(h, w, 3)
    depth = np.frombuffer(data, "<f4", h * w, _KF.size + h * w * 3).reshape(h, w)
    try:
        return Keyframe(id=f[2], pose=Pose(np.array([qw, qx, qy, qz]), np.array([tx, ty, tz])),
                        intrinsics=CameraIntrinsics(fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h,
                                                    near=near, far=far),
                        rgb=rgb.astype(np.float32) / np.float32(255.0), depth=depth.astype(np.float32),
                        last_loss=f[18], usage_remaining=f[19])
    except ValueError as exc:
        raise CorruptChunk(f"keyframe fields fail invariants: {exc}") from exc
