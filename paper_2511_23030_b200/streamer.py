"""Chunk streamer: .dcg bytes <-> pinned host <-> HBM slab, codec on the GPU.

Load:  file bytes -> pinned staging -> cudaMemcpyAsync on the copy stream ->
       K8 sm_chunk_unpack (AoS records -> slab SoA + Adam moments) on the
       copy stream; the compute stream waits on an event, not the host.
Evict: K9 sm_chunk_pack (slab SoA -> AoS records) -> D2H into pinned staging
       -> file write (diskformat.build_chunk_file).

Replaces the reference's unpack_chunk / pack_chunk object codecs
(diskformat.py:86-186, 82-138 MB/s on the survey host) on the chunk paging
path (store.py:241-272).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import CorruptChunk


class ChunkStreamer:
    def __init__(self, slab):
        import torch
        self.torch = torch
        self.slab = slab
        self.lib = _lib.load()
        self.copy_stream = torch.cuda.Stream(device=slab.device)
        self._dev = torch.empty(0, dtype=torch.uint8, device=slab.device)
        self._pin = torch.empty(0, dtype=torch.uint8, pin_memory=True)
        self._err = torch.empty(1, dtype=torch.int64, device=slab.device)
        self.bytes_h2d = 0
        self.bytes_d2h = 0

    def _staging(self, nbytes: int):
        torch = self.torch
        if self._dev.numel() < nbytes:
            self._dev = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, device=self.slab.device)
        if self._pin.numel() < nbytes:
            self._pin = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, pin_memory=True)
        return self._dev, self._pin

    def unpack_into(self, records: np.ndarray, stride: int, offset: int) -> None:
        n = int(records.shape[0])
        if n == 0:
            return
        nbytes = n * stride
        dev, pin = self._staging(nbytes)
        torch = self.torch
        pin[:nbytes].numpy()[:] = np.frombuffer(records.tobytes() if not records.flags.c_contiguous
                                                else records.view(np.uint8).reshape(-1), np.uint8)
        cur = torch.cuda.current_stream(self.slab.device)
        self.copy_stream.wait_stream(cur)   # slab rows may still be in use by queued work
        with torch.cuda.stream(self.copy_stream):
            dev[:nbytes].copy_(pin[:nbytes], non_blocking=True)
            s = self.slab
            rows = slice(offset, offset + n)
            rc = self.lib.sm_chunk_unpack(_lib.ptr(dev), n, int(stride), _lib.ptr(s.params[rows]),
                                          _lib.ptr(s.sh_rest[rows]), _lib.ptr(s.adam_m[rows]),
                                          _lib.ptr(s.adam_v[rows]), _lib.ptr(self._err),
                                          _lib.stream_handle(self.copy_stream))
            _lib.check(rc, "chunk_unpack")
        s.grads[offset:offset + n].zero_()
        cur.wait_stream(self.copy_stream)
        self.bytes_h2d += nbytes
        err = int(self._err.item())   # synchronises: the policy needs the verdict
        if err >= 0:
            raise CorruptChunk(f"chunk record {err} fails invariants")

    def pack_from(self, offset: int, n: int, stride: int) -> np.ndarray:
        if n == 0:
            return np.zeros(0, dtype=np.uint8)
        nbytes = n * stride
        dev, pin = self._staging(nbytes)
        s = self.slab
        rows = slice(offset, offset + n)
        rc = self.lib.sm_chunk_pack(_lib.ptr(s.params[rows]), _lib.ptr(s.sh_rest[rows]),
                                    _lib.ptr(s.adam_m[rows]), _lib.ptr(s.adam_v[rows]), n, int(stride),
                                    _lib.ptr(dev), _lib.stream_handle())
        _lib.check(rc, "chunk_pack")
        pin[:nbytes].copy_(dev[:nbytes], non_blocking=True)
        self.torch.cuda.current_stream(s.device).synchronize()
        self.bytes_d2h += nbytes
        return pin[:nbytes].numpy().copy()
