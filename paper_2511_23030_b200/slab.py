"""HBM slab holding the active tier's Gaussians as device SoA.

Every resident chunk owns one contiguous segment [offset, offset+capacity) of
the slab; its ``count`` first rows are live.  Columns (all float32, CUDA):

  params  [cap, 16]  param records (include/splatmap_cuda.h): 14 trainable
                     scalars + 2 pad; read by K2/K6, written by K7/K8
  adam_m  [cap, 16]  Adam first moment; column 14 = per-Gaussian step count
  adam_v  [cap, 16]  Adam second moment
  grads   [cap, 16]  gradient accumulator (K6 +=, K7 reads then zeroes)
  sh_rest [cap, 45]  the 45 higher-order SH coefficients (never trained;
                     carried for bit-exact .dcg round trips)

Segments come from a first-fit free list with coalescing; the slab grows
geometrically (one device copy) when no extent fits.  Sized for HBM: 1.5 M
Gaussians (the paper's budget) take ~0.6 GB.
"""

from __future__ import annotations

import bisect

COLS16 = ("params", "adam_m", "adam_v", "grads")


class GaussianSlab:
    """max_rows (an HBM cap): the slab is allocated at that size once and never
    grows -- so the cap holds at every instant -- and an allocation that finds
    no free extent first asks ``compact_hook`` (the store's defragmentation)
    to pack the live segments to the front, then raises HbmCapExceeded."""

    def __init__(self, capacity: int, device=None, growth: float = 1.5, max_rows: int | None = None):
        import torch
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        self.growth = growth
        self.max_rows = max_rows
        self.compact_hook = None
        self.compactions = 0
        self.capacity = 0
        self.params = self.adam_m = self.adam_v = self.grads = self.sh_rest = None
        self._free: list[tuple[int, int]] = []   # sorted (offset, size)
        self._resize(int(max_rows) if max_rows else max(int(capacity), 1024))

    # ---------------------------------------------------------- storage
    def _resize(self, new_cap: int) -> None:
        torch = self.torch
        old = self.capacity
        cols = {}
        for name in COLS16:
            t = torch.zeros((new_cap, 16), dtype=torch.float32, device=self.device)
            if old:
                t[:old].copy_(getattr(self, name))
            cols[name] = t
        sh = torch.zeros((new_cap, 45), dtype=torch.float32, device=self.device)
        if old:
            sh[:old].copy_(self.sh_rest)
        for name, t in cols.items():
            setattr(self, name, t)
        self.sh_rest = sh
        self.capacity = new_cap
        self._release(old, new_cap - old)

    @staticmethod
    def bytes_per_gaussian() -> int:
        return 4 * (16 * len(COLS16) + 45)

    def hbm_bytes(self) -> int:
        return self.capacity * self.bytes_per_gaussian()

    # -------------------------------------------------------- allocator
    def _release(self, off: int, size: int) -> None:
        if size <= 0:
            return
        i = bisect.bisect_left(self._free, (off, 0))
        self._free.insert(i, (off, size))
        # coalesce with neighbours
        if i + 1 < len(self._free) and off + size == self._free[i + 1][0]:
            self._free[i] = (off, size + self._free[i + 1][1])
            del self._free[i + 1]
        if i > 0 and self._free[i - 1][0] + self._free[i - 1][1] == self._free[i][0]:
            self._free[i - 1] = (self._free[i - 1][0], self._free[i - 1][1] + self._free[i][1])
            del self._free[i]

    def _first_fit(self, size: int) -> int | None:
        for i, (off, sz) in enumerate(self._free):
            if sz >= size:
                if sz == size:
                    del self._free[i]
                else:
                    self._free[i] = (off + size, sz - size)
                return off
        return None

    def alloc(self, size: int) -> int:
        size = max(int(size), 1)
        off = self._first_fit(size)
        if off is not None:
            return off
        if self.max_rows:   # capped: defragment, never grow
            if self.compact_hook is not None and self.capacity - self.used() >= size:
                self.compact_hook()
                self.compactions += 1
                off = self._first_fit(size)
                if off is not None:
                    return off
            from .errors import HbmCapExceeded
            raise HbmCapExceeded(f"{size} rows do not fit the HBM cap of {self.max_rows} rows "
                                 f"({self.used()} in use)")
        # grow: keep the tail extent contiguous with the new space
        tail_free = self._free[-1][1] if self._free and sum(self._free[-1]) == self.capacity else 0
        need = self.capacity + size - tail_free
        self._resize(max(need, int(self.capacity * self.growth)))
        return self.alloc(size)

    def free(self, off: int, size: int) -> None:
        if size > 0:
            self.grads[off:off + size].zero_()
            self._release(off, size)

    def used(self) -> int:
        return self.capacity - sum(s for _, s in self._free)

    def high_water(self) -> int:
        """One past the highest allocated row (bound for slab-wide passes)."""
        if self._free and sum(self._free[-1]) == self.capacity:
            return self._free[-1][0]
        return self.capacity

    def pack(self, segments: list[tuple[int, int, int]]) -> list[int]:
        """Move the live segments [(offset, capacity, rows in use)] (any order)
        to the front of the slab in offset order; returns their new offsets
        (same order as given) and leaves one free extent at the tail.  Unused
        rows (a segment's spare capacity, the tail) get zero gradients, the
        invariant `free` keeps."""
        order = sorted(range(len(segments)), key=lambda k: segments[k][0])
        new = [0] * len(segments)
        pos = 0
        for k in order:
            off, cap, used = segments[k]
            if off != pos and used:   # pos <= off: overlapping moves are safe (move clones)
                self.move(off, pos, used)
            if off != pos and cap > used:
                self.grads[pos + used:pos + cap].zero_()
            new[k] = pos
            pos += cap
        if pos < self.capacity:
            self.grads[pos:self.capacity].zero_()
        self._free = [(pos, self.capacity - pos)] if pos < self.capacity else []
        return new

    def move(self, src: int, dst: int, n: int) -> None:
        """Copy n rows of every column from src to dst (device to device)."""
        if n <= 0 or src == dst:
            return
        for name in COLS16 + ("sh_rest",):
            t = getattr(self, name)
            t[dst:dst + n].copy_(t[src:src + n].clone() if abs(src - dst) < n else t[src:src + n])
