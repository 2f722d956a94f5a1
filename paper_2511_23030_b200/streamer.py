"""Chunk streamer: .dcg bytes <-> pinned host <-> HBM slab, codec on the GPU.

Replaces the reference's synchronous unpack_chunk / pack_chunk object codecs
(diskformat.py:86-186, 82-138 MB/s on the survey host) on the paging path
(store.py:241-272, 493-515) without changing any policy decision or the
io_ns cost model (the store charges bytes exactly as the reference does).

Load:   the file is read straight into a pinned buffer (readinto; reader
        threads do it ahead of use for prefetched chunks); the copy stream
        moves it into a device staging slot and validates the records there
        (the host waits for that verdict only -- CorruptChunk is raised inside
        ensure_resident like the reference); the K8 unpack into the chunk's
        slab rows is queued on the compute stream behind the work already
        there, so a load never waits for the render in flight.
        A chunk whose eviction write is still pending is unpacked straight
        from the device buffer it was packed into (no host round trip).
Evict:  K9 sm_chunk_pack on the compute stream into a device buffer (so the
        slab rows can be reused immediately, stream-ordered); a writer
        thread then takes a pinned buffer, copies the records down on its
        own stream (after the pack's event) and writes the file: eviction
        write-back overlaps with rendering (write-behind), and the backlog
        of unwritten chunks waits in HBM, not in pinned memory.  Under a
        hard HBM cap (small device share) the copy down is issued at
        eviction instead and the device buffer returns to the pool once it
        completed; the backlog then waits in pinned memory, and a reload of
        a chunk still queued is served from that pinned copy.
Prefetch: speculative reads on reader threads into a FIFO tier of pinned
        buffers that never blocks real I/O (loads and write-behinds take
        back the oldest unclaimed read when the pool is empty).
flush():  drains the writer queue (the store's durability point).
"""

from __future__ import annotations

import queue
import threading
import time
from collections import OrderedDict
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

from . import _lib
from .errors import CorruptChunk, IoFailure


class _PendingWrite:
    __slots__ = ("path", "header", "pin", "nbytes", "event", "done", "dev", "stride", "make", "cache",
                 "inline", "borrowers", "settled")

    def __init__(self, path, header, pin, nbytes, event, dev, stride, make=None, cache=True):
        self.path, self.header, self.pin, self.nbytes = path, header, pin, nbytes
        self.event, self.dev, self.stride = event, dev, stride
        self.make = make   # host-built file (keyframes): bytes produced on the writer thread
        self.cache = cache   # keep the device bytes in the victim cache once written (chunks)
        self.inline = False   # pin holds the whole file (header + records), D2H issued at eviction
        self.borrowers = 0   # reloads reading `pin` right now (it returns to the pool after them)
        self.settled = False
        self.done = threading.Event()


class PinnedFile:
    """A chunk file's bytes in pinned host memory (`view()` = the file)."""
    __slots__ = ("pin", "size")

    def __init__(self, pin, size: int):
        self.pin, self.size = pin, size

    def view(self) -> np.ndarray:
        return self.pin[:self.size].numpy()


class BorrowedPinned(PinnedFile):
    """A pending write-behind's pinned file bytes lent to a reload (capped
    stores, whose device copy already went back to the pool)."""
    __slots__ = ("pw",)

    def __init__(self, pw):
        super().__init__(pw.pin, len(pw.header) + pw.nbytes)
        self.pw = pw


class DeviceRecords:
    """A chunk whose write-behind is pending: header + packed records on device."""
    __slots__ = ("header", "dev", "nbytes", "stride")

    def __init__(self, header: bytes, dev, nbytes: int, stride: int):
        self.header, self.dev, self.nbytes, self.stride = header, dev, nbytes, stride


class ChunkStreamer:
    def __init__(self, slab, write_behind: bool = True, reader_threads: int = 4,
                 writer_threads: int = 4, victim_bytes: int = 4 << 30, device_pool_bytes: int | None = None,
                 pinned_pool_bytes: int | None = None):
        """device_pool_bytes: a hard bound on the streamer's HBM (pack buffers
        + victim cache + the load staging ring) for an HBM-capped store; the
        pool is then never grown on demand -- a pack waits for a write-behind
        to land instead.  None: the default 6 GB pool, grown if it runs dry."""
        import torch
        self.torch = torch
        self.slab = slab
        self.device_pool_bytes = device_pool_bytes
        if pinned_pool_bytes is not None:   # host staging: pending write-behinds + prefetched reads
            self.PINNED_SLOTS = max(16, int(pinned_pool_bytes) // self.PINNED_SLOT_BYTES)
        if device_pool_bytes is not None:
            # headroom for the 4 load staging slots + the synchronous staging
            # buffer (<= 1.25 x the largest chunk each) and oversized packs
            self.DEVICE_SLOTS = max(2, int(device_pool_bytes) // self.PINNED_SLOT_BYTES - 8)
            victim_bytes = min(victim_bytes, (self.DEVICE_SLOTS // 2) * self.PINNED_SLOT_BYTES)
        self.lib = _lib.load()
        self.copy_stream = torch.cuda.Stream(device=slab.device)   # H2D + validation of loads
        self.device_bytes = 0   # every device buffer this streamer allocated (pool, staging)
        self._dev = torch.empty(0, dtype=torch.uint8, device=slab.device)
        self._pin = torch.empty(0, dtype=torch.uint8, pin_memory=True)
        self._err = torch.empty(1, dtype=torch.int64, device=slab.device)
        self._err_unpack = torch.empty(1, dtype=torch.int64, device=slab.device)
        self._err_host = torch.empty(1, dtype=torch.int64, pin_memory=True)
        self._slots = [{"buf": None, "event": None} for _ in range(4)]   # device staging ring
        self._slot_i = 0
        self.bytes_h2d = 0
        self.bytes_d2h = 0
        self.write_behind = write_behind
        self._pending: dict[Path, _PendingWrite] = {}
        self._lock = threading.Lock()
        self._freed = threading.Condition(self._lock)   # a pooled buffer came back
        self._queue: queue.Queue = queue.Queue()
        self._writer_error: BaseException | None = None
        self._failed: list[_PendingWrite] = []   # write-behinds that raised (kept pending)
        self._free_pins: list = []
        self._arena_ready = False
        # device victim cache: packed records of chunks whose write-behind
        # landed, kept in HBM so a reload is one K8 (the OS page cache, one
        # level up); never changes a policy decision or a charged byte
        self._victims: "OrderedDict[Path, DeviceRecords]" = OrderedDict()
        self._victim_bytes = 0
        self.victim_limit = victim_bytes
        self._free_devs: list = []
        self._writers = [threading.Thread(target=self._write_loop, daemon=True) for _ in range(writer_threads)]
        for t in self._writers:
            t.start()
        self._pool = ThreadPoolExecutor(max_workers=reader_threads)
        self._prefetched: dict[Path, object] = {}
        self.stats = {"prefetch_hits": 0, "pending_hits": 0, "victim_hits": 0, "async_writes": 0,
                      "superseded_writes": 0, "pool_wait_s": 0.0, "alloc_pinned": 0,
                      "alloc_device": 0, "alloc_s": 0.0, "read_s": 0.0, "stage_wait_s": 0.0,
                      "validate_wait_s": 0.0, "read_file_s": 0.0, "unpack_s": 0.0, "write_async_s": 0.0,
                      "disk_bytes_read": 0, "write_s": 0.0, "write_d2h_s": 0.0, "writer_pin_wait_s": 0.0, "prefetch_issued": 0, "prefetch_dropped": 0, "pending_pinned_hits": 0}
        self._largest = {True: 2 * self.PINNED_SLOT_BYTES, False: 2 * self.PINNED_SLOT_BYTES}   # per pool kind
        self._wlocal = threading.local()
        self._rename_locks = [threading.Lock() for _ in range(64)]
        self._early: list = []   # capped stores: write-behinds whose device copy is still held
        self._d2h = torch.cuda.Stream(device=slab.device)   # capped stores: eviction D2H   # per writer thread: its D2H stream

    # ---------------------------------------------------------------- staging
    def _staging(self, nbytes: int):
        torch = self.torch
        if self._dev.numel() < nbytes:
            self.device_bytes -= self._dev.numel()
            self._dev = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, device=self.slab.device)
            self.device_bytes += self._dev.numel()
        if self._pin.numel() < nbytes:
            self._pin = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, pin_memory=True)
        return self._dev, self._pin

    _QUANTUM = 8 << 20   # pooled buffers are whole multiples: any freed one fits the next chunk
    # Pre-allocated pools, sized for a write-behind queue that outruns the disk
    # (C4: ~0.9 GB/s of write-back) plus the HBM victim cache; page-locking or
    # cudaMalloc on demand costs 10-40 ms per buffer on the paging path.
    PINNED_SLOTS = 96    # 3 GB pinned host
    DEVICE_SLOTS = 192   # 6 GB HBM: pending pack buffers + the victim cache
    PINNED_SLOT_BYTES = 32 << 20

    def _ensure_arena(self) -> None:
        """Page-lock the pinned staging pool once, on the first paging operation."""
        if self._arena_ready:
            return
        self._arena_ready = True
        torch = self.torch
        t0 = time.perf_counter()
        # every 16th slot is twice the size: dense chunks (C4: the largest
        # file is ~1.3 slots) never wait for, or allocate, a buffer
        def size(i):
            return self.PINNED_SLOT_BYTES * (2 if i % 16 == 15 else 1)
        bufs = [torch.empty(size(i), dtype=torch.uint8, pin_memory=True) for i in range(self.PINNED_SLOTS)]
        devs = [torch.empty(size(i), dtype=torch.uint8, device=self.slab.device)
                for i in range(self.DEVICE_SLOTS if self.write_behind else 0)]
        self.device_bytes += sum(d.numel() for d in devs)
        with self._lock:
            self._free_pins.extend(bufs)
            self._free_devs.extend(devs)
            self.stats["arena_s"] = time.perf_counter() - t0

    def warm(self) -> None:
        """Allocate the staging pools now (else on the first paging operation)."""
        self._ensure_arena()

    def _pinned_free(self) -> int:
        with self._lock:
            return len(self._free_pins)

    def _take(self, pool: list, nbytes: int, pinned: bool, wait_stat: str = "pool_wait_s", steal: bool = True):
        """A pooled buffer of >= nbytes.  When the pool is empty: a device
        buffer is taken back from the oldest victim-cache entry, a pinned one
        from the oldest unclaimed prefetch (unless the caller is a prefetch
        read itself), else it is waited for briefly while write-behinds are
        in flight (each landed file frees one) -- under a hard HBM cap for as
        long as it takes; only then is a buffer allocated."""
        torch = self.torch
        self._ensure_arena()

        def fit():
            best = None
            for i, t in enumerate(pool):   # smallest buffer that fits
                if t.numel() >= nbytes and (best is None or t.numel() < pool[best].numel()):
                    best = i
            return best

        with self._lock:
            # without a hard cap, wait for a landing write about as long as
            # allocating would take (page-locking 32 MB: ~10-40 ms; a pooled
            # cudaMalloc: well under that), then grow the pool
            deadline = time.perf_counter() + (0.03 if pinned else 0.005)
            while True:
                best = fit()
                if best is None and pinned and steal:
                    # speculative reads never block real I/O: take back the
                    # buffer of the oldest finished, still unclaimed prefetch
                    for path, fut in list(self._prefetched.items()):   # oldest first
                        if not fut.done() or fut.exception() is not None:
                            continue
                        del self._prefetched[path]
                        pool.append(fut.result().pin)
                        self.stats["prefetch_dropped"] += 1
                        best = fit()
                        if best is not None:
                            break
                if best is None and not pinned and self._early:
                    self._reclaim_early()
                    best = fit()
                if best is None and not pinned:
                    for path in list(self._victims):   # oldest first
                        old = self._victims.pop(path)
                        self._victim_bytes -= old.dev.numel()
                        pool.append(old.dev)
                        best = fit()
                        if best is not None:
                            break
                if best is not None:
                    return pool.pop(best)
                left = deadline - time.perf_counter()
                hard = not pinned and self.device_pool_bytes is not None
                if not self._pending or (left <= 0 and not hard):
                    break
                if nbytes > self._largest[pinned] and not hard:
                    break   # no buffer in circulation fits: waiting cannot help
                t0 = time.perf_counter()
                # a write landing returns its buffers (a completed eviction
                # D2H does not notify: poll for those)
                self._freed.wait(timeout=left if not hard else (0.0005 if self._early else 1.0))
                self.stats[wait_stat] += time.perf_counter() - t0
        size = -(-(nbytes + 4096) // self._QUANTUM) * self._QUANTUM
        if not pinned and self.device_pool_bytes is not None:
            with self._lock:   # trade free (too small) pool buffers for one that fits the cap
                while self.device_bytes + size > self.device_pool_bytes and pool:
                    self.device_bytes -= pool.pop().numel()
            if self.device_bytes + size > self.device_pool_bytes:
                from .errors import HbmCapExceeded
                raise HbmCapExceeded(f"the streamer's device pool ({self.device_pool_bytes} B of the HBM cap) "
                                     f"cannot hold another {size} B buffer")
        t0 = time.perf_counter()
        with self._lock:
            self._largest[pinned] = max(self._largest[pinned], size)
        if pinned:
            buf = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        else:
            buf = torch.empty(size, dtype=torch.uint8, device=self.slab.device)
            self.device_bytes += size
        with self._lock:
            self.stats["alloc_pinned" if pinned else "alloc_device"] += 1
            self.stats["alloc_s"] += time.perf_counter() - t0
        return buf

    # ------------------------------------------------------------------- load
    def _read_pinned(self, path: Path, steal: bool = True) -> PinnedFile:
        size = path.stat().st_size
        pin = self._take(self._free_pins, max(size, 1), pinned=True, steal=steal)
        t0 = time.perf_counter()
        with open(path, "rb", buffering=0) as f:
            got = f.readinto(memoryview(pin.numpy())[:size])
        with self._lock:
            self.stats["read_s"] += time.perf_counter() - t0
            self.stats["disk_bytes_read"] += got
        if got != size:
            raise OSError(f"short read of {path}: {got} of {size} bytes")
        return PinnedFile(pin, size)

    def release(self, src) -> None:
        """Return a PinnedFile's buffer to the pool (after its H2D completed)."""
        if isinstance(src, BorrowedPinned):
            with self._lock:
                pw = src.pw
                pw.borrowers -= 1
                if pw.borrowers == 0 and pw.settled and pw.pin is not None:
                    self._free_pins.append(pw.pin)
                    pw.pin = None
                    self._freed.notify_all()
        elif isinstance(src, PinnedFile):
            with self._lock:
                self._free_pins.append(src.pin)
                self._freed.notify_all()

    def read_file(self, path: Path):
        self.check()   # a failed write-behind surfaces at the next paging operation
        t0 = time.perf_counter()
        try:
            return self._read_file(path)
        finally:
            self.stats["read_file_s"] += time.perf_counter() - t0

    def _read_file(self, path: Path):
        """PinnedFile of `path` from the prefetch tier or the disk, or a
        DeviceRecords if its eviction write is still pending."""
        path = Path(path)
        with self._lock:   # one critical section: a write cannot settle in between
            pw = self._pending.get(path)
            pending = None
            if pw is not None:
                if pw.dev is not None:
                    pending = DeviceRecords(pw.header, pw.dev, pw.nbytes, pw.stride)
                elif pw.pin is not None:   # capped store: the device copy is back in the
                    pw.borrowers += 1      # pool, the pinned one (D2H done) serves the reload
                    pending = BorrowedPinned(pw)
            vic = self._victims.get(path)
            if vic is not None:
                self._victims.move_to_end(path)
            fut = self._prefetched.pop(path, None)
        if fut is not None and (pw is not None or vic is not None):   # served from HBM: the read was moot
            fut.add_done_callback(lambda f: f.exception() is None and self.release(f.result()))
            fut = None
        if pending is not None:
            self.stats["pending_hits"] += 1
            if isinstance(pending, BorrowedPinned):
                self.stats["pending_pinned_hits"] += 1
            return pending
        if pw is not None:   # a host-built file still being written: let it land
            pw.done.wait()
            self.check()
        if vic is not None:
            self.stats["victim_hits"] += 1
            return vic
        if fut is not None:
            try:
                src = fut.result()
                self.stats["prefetch_hits"] += 1
                return src
            except OSError:
                pass
        return self._read_pinned(path)

    def prefetch(self, paths) -> None:
        """Speculatively read chunk files into pinned memory (reader threads);
        never takes the last pinned buffers a load or eviction needs.  The
        prefetch tier is FIFO: when it is full, the oldest finished,
        unclaimed reads make room for the newer speculation."""
        self._ensure_arena()
        reserve = max(8, self.PINNED_SLOTS // 4)   # loads and write-behinds come first
        paths = [Path(p) for p in paths]
        asked = set(paths)
        with self._lock:
            spare = len(self._free_pins) - reserve
            for p in paths:
                if p in self._prefetched or p in self._pending or p in self._victims:
                    continue
                if spare <= 0:
                    old = next((q for q, f in self._prefetched.items()
                                if q not in asked and f.done() and f.exception() is None), None)
                    if old is None:
                        break
                    self._free_pins.append(self._prefetched.pop(old).result().pin)
                    self.stats["prefetch_dropped"] += 1
                    spare += 1
                self._prefetched[p] = self._pool.submit(self._read_pinned, p, False)
                self.stats["prefetch_issued"] += 1
                spare -= 1

    def drop_prefetch(self, path: Path) -> None:
        with self._lock:
            fut = self._prefetched.pop(Path(path), None)
        if fut is not None:
            fut.add_done_callback(lambda f: f.exception() is None and self.release(f.result()))

    def _stage_slot(self, nbytes: int):
        """A device staging buffer whose previous unpack has completed."""
        torch = self.torch
        slot = self._slots[self._slot_i]
        self._slot_i = (self._slot_i + 1) % len(self._slots)
        if slot["event"] is not None:
            t0 = time.perf_counter()
            slot["event"].synchronize()
            self.stats["stage_wait_s"] += time.perf_counter() - t0
        if slot["buf"] is None or slot["buf"].numel() < nbytes:
            if slot["buf"] is not None:
                self.device_bytes -= slot["buf"].numel()
            slot["buf"] = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, device=self.slab.device)
            self.device_bytes += slot["buf"].numel()
        return slot

    def unpack_into(self, src, records: np.ndarray | None, n: int, stride: int, offset: int) -> None:
        t0 = time.perf_counter()
        try:
            self._unpack_into(src, records, n, stride, offset)
        finally:
            self.stats["unpack_s"] += time.perf_counter() - t0

    def _unpack_into(self, src, records: np.ndarray | None, n: int, stride: int, offset: int) -> None:
        """Chunk records -> slab rows [offset, offset + n) (K8)."""
        if n == 0:
            self.release(src)
            return
        torch = self.torch
        nbytes = n * stride
        s = self.slab
        rows = slice(offset, offset + n)
        cur = torch.cuda.current_stream(self.slab.device)
        if isinstance(src, DeviceRecords):   # our own packed bytes, still on the device
            dev = src.dev
        else:
            slot = self._stage_slot(nbytes)
            dev = slot["buf"]
            if isinstance(src, PinnedFile):
                host = src.pin[records.ctypes.data - src.pin.data_ptr():][:nbytes]
            else:   # plain bytes (API callers): through the pinned staging buffer
                _, host = self._staging(nbytes)
                host[:nbytes].numpy()[:] = records.view(np.uint8).reshape(-1)[:nbytes]
                host = host[:nbytes]
            with torch.cuda.stream(self.copy_stream):
                dev[:nbytes].copy_(host, non_blocking=True)
                rc = self.lib.sm_chunk_unpack(_lib.ptr(dev), n, int(stride), None, None, None, None,
                                              _lib.ptr(self._err), _lib.stream_handle(self.copy_stream))
                _lib.check(rc, "chunk_validate")
                self._err_host.copy_(self._err, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.copy_stream)
            t0 = time.perf_counter()
            ev.synchronize()   # H2D + validation only; the render keeps running
            self.stats["validate_wait_s"] += time.perf_counter() - t0
            self.release(src)
            err = int(self._err_host[0])
            if err >= 0:
                raise CorruptChunk(f"chunk record {err} fails invariants")
            cur.wait_event(ev)
        rc = self.lib.sm_chunk_unpack(_lib.ptr(dev), n, int(stride), _lib.ptr(s.params[rows]),
                                      _lib.ptr(s.sh_rest[rows]), _lib.ptr(s.adam_m[rows]),
                                      _lib.ptr(s.adam_v[rows]), _lib.ptr(self._err_unpack),
                                      _lib.stream_handle(cur))
        _lib.check(rc, "chunk_unpack")
        s.grads[offset:offset + n].zero_()
        if not isinstance(src, DeviceRecords):
            slot["event"] = torch.cuda.Event()
            slot["event"].record(cur)
        self.bytes_h2d += nbytes

    # ------------------------------------------------------------------ evict
    def _pack_to_device(self, offset: int, n: int, stride: int, dev):
        s = self.slab
        rows = slice(offset, offset + n)
        rc = self.lib.sm_chunk_pack(_lib.ptr(s.params[rows]), _lib.ptr(s.sh_rest[rows]),
                                    _lib.ptr(s.adam_m[rows]), _lib.ptr(s.adam_v[rows]), n, int(stride),
                                    _lib.ptr(dev), _lib.stream_handle())
        _lib.check(rc, "chunk_pack")

    def pack_from(self, offset: int, n: int, stride: int) -> np.ndarray:
        """Synchronous pack (flush, API materialisation)."""
        if n == 0:
            return np.zeros(0, dtype=np.uint8)
        nbytes = n * stride
        dev, pin = self._staging(nbytes)
        self._pack_to_device(offset, n, stride, dev)
        pin[:nbytes].copy_(dev[:nbytes], non_blocking=True)
        self.torch.cuda.current_stream(self.slab.device).synchronize()
        self.bytes_d2h += nbytes
        return pin[:nbytes].numpy().copy()

    def write_async(self, path: Path, header: bytes, offset: int, n: int, stride: int) -> None:
        self.check()
        t0 = time.perf_counter()
        try:
            self._write_async(path, header, offset, n, stride)
        finally:
            self.stats["write_async_s"] += time.perf_counter() - t0

    def _write_async(self, path: Path, header: bytes, offset: int, n: int, stride: int) -> None:
        """Write-behind eviction of slab rows [offset, offset+n) to `path`.

        The compute stream packs the rows into a pooled device buffer; the
        rest is a writer thread's: it takes a pinned buffer only when it
        starts the write (D2H on its own stream, then the file), so the
        write-behind backlog waits in HBM -- where a reload is served from --
        and pinned memory is held by in-flight I/O only."""
        torch = self.torch
        nbytes = n * stride
        dev = self._take(self._free_devs, max(nbytes, 1), pinned=False)
        if n:
            self._pack_to_device(offset, n, stride, dev)
        ev = torch.cuda.Event()
        cur = torch.cuda.current_stream(self.slab.device)
        if self.device_pool_bytes is None:
            ev.record(cur)
            pw = _PendingWrite(Path(path), header, None, nbytes, ev, dev, stride)
        else:
            # hard HBM cap: the device share is small, so the backlog waits in
            # pinned memory -- copy down now; the device buffer returns to the
            # pool as soon as that copy completed (_reclaim_early)
            h = len(header)
            pin = self._take(self._free_pins, h + max(nbytes, 1), pinned=True)
            pin[:h].numpy()[:] = np.frombuffer(header, dtype=np.uint8)
            self._d2h.wait_stream(cur)
            with torch.cuda.stream(self._d2h):
                if n:
                    pin[h:h + nbytes].copy_(dev[:nbytes], non_blocking=True)
                ev.record(self._d2h)
            pw = _PendingWrite(Path(path), header, pin, nbytes, ev, dev, stride, cache=False)
            pw.inline = True
            self._early.append(pw)
        with self._lock:
            self._release_superseded(self._pending.get(pw.path))
            self._pending[pw.path] = pw
            self._drop_victim(pw.path)
            fut = self._prefetched.pop(pw.path, None)
        if fut is not None:
            fut.add_done_callback(lambda f: f.exception() is None and self.release(f.result()))
        self.bytes_d2h += nbytes
        self.stats["async_writes"] += 1
        self._queue.put(pw)

    def _reclaim_early(self) -> None:   # caller holds the lock
        """Capped stores: device buffers of write-behinds whose D2H completed
        go back to the pool (reloads of those chunks read the pinned copy)."""
        if not self._early:
            return
        keep = []
        for pw in self._early:
            if pw.event.query():
                if pw.dev is not None:
                    self._free_devs.append(pw.dev)
                    pw.dev = None
            else:
                keep.append(pw)
        self._early = keep

    def write_file_async(self, path: Path, nbytes: int, fill) -> None:
        """Write-behind of a file assembled by a kernel: fill(pin) writes its
        nbytes into a pooled pinned buffer (device-addressable host memory)
        on the current stream, e.g. sm_keyframe_pack; a writer thread writes
        the file once that kernel completed.  Uses no device buffer."""
        self.check()
        torch = self.torch
        pin = self._take(self._free_pins, max(nbytes, 1), pinned=True)
        fill(pin)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.slab.device))
        pw = _PendingWrite(Path(path), b"", pin, nbytes, ev, None, 0, cache=False)
        with self._lock:
            self._release_superseded(self._pending.get(pw.path))
            self._pending[pw.path] = pw
            self._drop_victim(pw.path)
        self.bytes_d2h += nbytes
        self.stats["async_writes"] += 1
        self._queue.put(pw)

    def write_bytes_async(self, path: Path, make) -> None:
        """Write-behind of a host-built file: `make()` runs on a writer thread
        and returns the file's bytes (same newest-write-wins and wait_path
        rules as the chunk write-behind)."""
        pw = _PendingWrite(Path(path), b"", None, 0, None, None, 0, make)
        with self._lock:
            self._release_superseded(self._pending.get(pw.path))
            self._pending[pw.path] = pw
            self._drop_victim(pw.path)
            fut = self._prefetched.pop(pw.path, None)
        if fut is not None:
            fut.add_done_callback(lambda f: f.exception() is None and self.release(f.result()))
        self.stats["async_writes"] += 1
        self._queue.put(pw)

    def _write_loop(self) -> None:
        while True:
            pw = self._queue.get()
            if pw is None:
                return
            failed = False
            try:
                self._write_one(pw)
            except BaseException as exc:   # surfaced at the next paging call / drain()
                self._writer_error = exc
                failed = True
            if pw.event is not None:
                # a superseded write skipped its wait: the pack (or fill)
                # kernel may still be writing `dev` / `pin`, so neither goes
                # back to a pool before it completes
                pw.event.synchronize()
            self._settle(pw, failed)
            pw.done.set()
            self._queue.task_done()

    def _write_one(self, pw: _PendingWrite) -> None:
        with self._lock:   # superseded by a newer write of the path: skip the disk work
            stale = self._pending.get(pw.path) is not pw
        if stale:
            self.stats["superseded_writes"] += 1
            return
        if pw.dev is not None and pw.pin is None:   # chunk: D2H of the packed records now
            t0 = time.perf_counter()
            pin = self._take(self._free_pins, max(pw.nbytes, 1), pinned=True, wait_stat="writer_pin_wait_s")
            t1 = time.perf_counter()
            torch = self.torch
            stream = getattr(self._wlocal, "stream", None)
            if stream is None:
                stream = self._wlocal.stream = torch.cuda.Stream(device=self.slab.device)
            with torch.cuda.stream(stream):
                stream.wait_event(pw.event)   # the pack kernel
                if pw.nbytes:
                    pin[:pw.nbytes].copy_(pw.dev[:pw.nbytes], non_blocking=True)
                done = torch.cuda.Event()
                done.record(stream)
            pw.pin = pin
            done.synchronize()
            with self._lock:
                self.stats["write_d2h_s"] += time.perf_counter() - t1
        elif pw.event is not None:
            pw.event.synchronize()   # the kernel that filled the pinned buffer
        t0 = time.perf_counter()
        tmp = pw.path.with_name(f"{pw.path.name}.{threading.get_ident()}.tmp")
        with open(tmp, "wb") as f:   # straight from pinned memory, no bytes copy
            if pw.make is not None:
                f.write(pw.make())
            elif pw.inline:
                f.write(memoryview(pw.pin.numpy())[:len(pw.header) + pw.nbytes])
            else:
                f.write(pw.header)
                f.write(memoryview(pw.pin.numpy())[:pw.nbytes])
        # several writers: only the newest write of a path lands.  The rename
        # (milliseconds on some filesystems) holds only the path's stripe
        # lock, never the streamer lock the paging path needs: a newer write
        # of the same path renames after this one, under the same stripe
        with self._rename_locks[hash(pw.path) % len(self._rename_locks)]:
            with self._lock:
                current = self._pending.get(pw.path) is pw
            if current:
                tmp.replace(pw.path)
        with self._lock:
            self.stats["write_s"] += time.perf_counter() - t0
        if not current:
            tmp.unlink(missing_ok=True)

    def _settle(self, pw: _PendingWrite, failed: bool) -> None:
        """Return a finished write's buffers (or keep them, see below)."""
        with self._lock:
            current = self._pending.get(pw.path) is pw
            if failed and current:
                # keep the entry and its packed device bytes: a reload is still
                # served from them (no silent stale read of the old file) and
                # the next drain() re-queues the write
                self._failed.append(pw)
                self._freed.notify_all()
                return
            landed = current and not failed
            if current:
                del self._pending[pw.path]
            pw.settled = True
            if pw.pin is not None and pw.borrowers == 0:   # (else the last borrower returns it)
                self._free_pins.append(pw.pin)
                pw.pin = None
            self._freed.notify_all()   # (waiters run once this block releases the lock)
            dev, pw.dev = pw.dev, None
            if dev is None:
                pass
            elif landed and pw.cache and self.victim_limit > 0:   # keep the packed bytes in HBM
                self._drop_victim(pw.path)
                self._victims[pw.path] = DeviceRecords(pw.header, dev, pw.nbytes, pw.stride)
                self._victim_bytes += dev.numel()
                while self._victim_bytes > self.victim_limit and self._victims:
                    _, old = self._victims.popitem(last=False)
                    self._victim_bytes -= old.dev.numel()
                    self._free_devs.append(old.dev)
            else:
                self._free_devs.append(dev)

    def _drop_victim(self, path: Path) -> None:   # caller holds the lock
        old = self._victims.pop(path, None)
        if old is not None:
            self._victim_bytes -= old.dev.numel()
            self._free_devs.append(old.dev)

    def forget(self, path: Path) -> None:
        """The store is about to rewrite or delete `path`: let a pending write
        land first and drop every cached copy of the old bytes."""
        path = Path(path)
        self.wait_path(path)
        with self._lock:
            self._drop_victim(path)
            fut = self._prefetched.pop(path, None)
        if fut is not None:
            fut.add_done_callback(lambda f: f.exception() is None and self.release(f.result()))

    def check(self) -> None:
        if self._writer_error is not None:
            exc, self._writer_error = self._writer_error, None
            raise IoFailure(f"write-behind failed: {exc}") from exc

    def _retry_failed(self) -> None:
        """Re-queue the write-behinds that failed and are still the newest
        write of their path (their packed bytes were kept)."""
        with self._lock:
            retry = [pw for pw in self._failed if self._pending.get(pw.path) is pw]
            self._failed = []
        for pw in retry:
            pw.done = threading.Event()
            self._queue.put(pw)

    def _release_superseded(self, old) -> None:   # caller holds the lock
        """A new write replaces a failed one of the same path: its buffers
        return to the pools (its D2H completed before it was attempted)."""
        if old is not None and old in self._failed:
            self._failed.remove(old)
            old.settled = True
            if old.pin is not None and old.borrowers == 0:
                self._free_pins.append(old.pin)
                old.pin = None
            if old.dev is not None:
                self._free_devs.append(old.dev)
                old.dev = None

    def drain(self) -> None:
        """Block until every pending write reached the disk (flush point).
        A write that failed before is retried once per drain."""
        self._retry_failed()
        self._queue.join()
        self.check()

    def wait_path(self, path: Path) -> None:
        with self._lock:
            pw = self._pending.get(Path(path))
        if pw is not None:
            pw.done.wait()
        self.check()
