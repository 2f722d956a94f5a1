"""The mapping step on the B200: drop-in for splatmap sim._Replay.optimization_step.

One step (sim.py:319-370) keeps the reference's host policy -- candidate
set, loss-weighted keyframe draw with derived seeds, keyframe tier access,
visibility (VisibilityCache + K1), overlap, ensure_resident, loss record,
metrics row with the deterministic cost model -- and replaces the
render + loss + projected-residual nudge (sim.py:280-317) with the device
pipeline: K2-K4 forward, fused loss forward/backward, K5-K6 backward and K7
fused Adam over the active set, with a single 32-byte device->host read
(loss + overflow flag) per step.

Data-parallel mode (``optimization_step_dp``): K keyframes per step, rank r
renders keyframes r, r+G, ...; the union active set's gradient records are
packed and summed with one NCCL all-reduce, then every rank applies the
identical Adam update to its replica of the active tier.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import CameraIntrinsics, Keyframe, Pose
from .culling import ChunkExtent, CullConfig, VisibilityCache, cull_table
from .errors import DeviceFailure, EmptyCandidates
from .renderloss import LossEngine, LossWeights, RenderEngine, camera_for
from .select import (KeyframeIndex, SelectConfig, candidate_set, draw_uniform, overlap, record_loss,
                     select_keyframe)
from .store import ChunkStore

__all__ = ["METRICS_HEADER", "FrameMetrics", "AdamSettings", "MappingEngine", "derive_seed"]

METRICS_HEADER = ("frame,step,active_gaussians,active_chunks,active_keyframes,"
                  "loads,evictions,io_ns,step_ns,selected_kf,overlap,loss")

# Deterministic step-cost model (sim.py:53-57)
NS_PER_RENDERED_GAUSSIAN = 150
NS_PER_PIXEL = 40
NS_PER_INSERTED_GAUSSIAN = 300
NS_STEP_BASE = 20_000


def derive_seed(master: int, purpose: int, counter: int) -> int:
    """sim.py:158 _derive_seed."""
    return int(np.random.SeedSequence([master, purpose, counter]).generate_state(1)[0])


def dp_select(index: KeyframeIndex, latest_kf: int, seed: int, step_counter: int,
              k: int) -> list[int]:
    """The K keyframes of one data-parallel mapping step, identical on every
    rank: K loss-weighted draws (select.py policy) from the same candidate
    set with derived seeds (seed, 2, step * K + j).  Keyframe j is rendered
    by rank j mod G (C3: K = 8 over G = 1, 2, 4, 8).  K = 1 is exactly the
    single-GPU step's draw (sim.py:331)."""
    try:
        candidates = candidate_set(index.position_of(latest_kf), index)
    except EmptyCandidates:
        candidates = [latest_kf]
    return [select_keyframe(candidates, index, derive_seed(seed, 2, step_counter * k + j))
            for j in range(k)]


def owned_keyframes(k: int, world: int, rank: int) -> list[int]:
    """Positions j of the step's K keyframes that rank `rank` renders."""
    return list(range(rank, k, world))


def allreduce_step(packed, lossbuf, group=None) -> None:
    """The DP exchange: sum the packed gradient records of the union active
    set and the [loss_0 .. loss_{K-1}, overflow] vector over the ranks (NCCL
    on GPUs, gloo in the CPU tests)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    dist.all_reduce(packed, group=group)
    dist.all_reduce(lossbuf, group=group)


@dataclass
class FrameMetrics:
    frame: int
    step: int
    active_gaussians: int
    active_chunks: int
    active_keyframes: int
    loads: int
    evictions: int
    io_ns: int
    step_ns: int
    selected_kf: int
    overlap: float | None
    loss: float

    def csv_row(self) -> str:
        ov = "" if self.overlap is None else f"{self.overlap:.9g}"
        return (f"{self.frame},{self.step},{self.active_gaussians},{self.active_chunks},"
                f"{self.active_keyframes},{self.loads},{self.evictions},{self.io_ns},"
                f"{self.step_ns},{self.selected_kf},{ov},{self.loss:.9g}")


@dataclass
class AdamSettings:
    """Per-scalar learning rates on the stored (activated) parameters."""

    lr_position: float = 1e-4
    lr_rotation: float = 1e-3
    lr_scale: float = 5e-5
    lr_opacity: float = 1e-2
    lr_sh0: float = 2.5e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15
    min_scale: float = 1e-5

    def to_c(self) -> _lib.AdamConfig:
        c = _lib.AdamConfig()
        lrs = [self.lr_position] * 3 + [self.lr_rotation] * 4 + [self.lr_scale] * 3 + \
              [self.lr_opacity] + [self.lr_sh0] * 3
        for k, v in enumerate(lrs):
            c.lr[k] = v
        c.beta1, c.beta2, c.eps, c.min_scale = self.beta1, self.beta2, self.eps, self.min_scale
        return c


class _ActiveSet:
    """Slot lists of visible-chunk sets (sorted ids -> slab rows), LRU-cached by
    segment layout so revisited keyframes reuse their list (and CUDA graph)."""

    CAPACITY = 64
    rebuilds = 0   # slot buffers refilled in place after paging

    def __init__(self, device):
        import torch
        self.torch = torch
        self.device = device
        self.key = None
        self.n = 0
        self._cache: dict = {}

    def build(self, segments: list[tuple[int, int]]):
        key = tuple(segments)
        hit = self._cache.pop(key, None)
        if hit is not None:
            self._cache[key] = hit
            self.key, self.n = key, hit[1]
            return hit
        total = sum(c for _, c in segments)
        slots = self.torch.empty(max(total, 1), dtype=self.torch.int32, device=self.device)
        return self._fill(slots, key, segments)

    def rebuild(self, slots, segments: list[tuple[int, int]]):
        """The same chunks (same row count) at new slab rows: re-expand into
        the existing buffer, stream-ordered behind the passes that read it,
        so the CUDA graphs captured over this buffer stay valid."""
        for k in [k for k, v in self._cache.items() if v[0] is slots]:
            del self._cache[k]
        self.rebuilds += 1
        return self._fill(slots, tuple(segments), segments)

    def _fill(self, slots, key, segments):
        counts = np.array([c for _, c in segments], dtype=np.int64)
        offs = np.array([o for o, _ in segments], dtype=np.int64)
        total = int(counts.sum())
        if total:
            prefix = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
            meta = self.torch.as_tensor(np.stack([offs, counts, prefix]), device=self.device)
            rc = _lib.load().sm_expand_segments(_lib.ptr(meta[0]), _lib.ptr(meta[1]), _lib.ptr(meta[2]),
                                                len(segments), total, _lib.ptr(slots),
                                                _lib.stream_handle())
            _lib.check(rc, "expand_segments")
        self._cache.pop(key, None)
        self._cache[key] = (slots, total)
        while len(self._cache) > self.CAPACITY:
            self._cache.pop(next(iter(self._cache)))
        self.key, self.n = key, total
        return slots, total


@dataclass
class _DeviceKeyframe:
    rgb_u8: object
    depth: object
    pending: object = None   # side stream still uploading (e2e mode)


class MappingEngine:
    """Owns the device pipeline of the mapping step for one store / camera.

    Mirrors splatmap sim._Replay's state (sim.py:199-225): the store, the
    visibility cache, the keyframe index, the latest keyframe and the step
    counter driving the derived seeds.
    """

    def __init__(self, store: ChunkStore, intr: CameraIntrinsics, seed: int = 7,
                 cull: CullConfig | None = None, select: SelectConfig | None = None,
                 weights: LossWeights | None = None, adam: AdamSettings | None = None,
                 comm=None, sample=None):
        import torch
        self.torch = torch
        self.store = store
        self.intr = intr
        self.seed = seed
        self.cull_cfg = cull or CullConfig()
        self.cache = VisibilityCache(cfg=self.cull_cfg)
        self.index = KeyframeIndex(config=select or SelectConfig())
        self.weights = weights or LossWeights()
        self.adam = adam or AdamSettings()
        if sample is None:
            from .sample import SampleConfig
            sample = SampleConfig()
        self.sample_cfg = sample
        self._adam_c = self.adam.to_c()
        self.comm = comm
        self.latest_kf: int | None = None
        self.step_counter = 0
        self.rows: list[FrameMetrics] = []
        dev = store.slab.device
        self.device = dev
        self.render = RenderEngine(dev)
        self.loss = LossEngine(dev)
        self.active = _ActiveSet(dev)
        h, w = intr.height, intr.width
        self.rgb = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
        self.depth = torch.empty((h, w), dtype=torch.float32, device=dev)
        self.alpha = torch.empty((h, w), dtype=torch.float32, device=dev)
        self.d_rgb = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
        self.d_depth = torch.empty((h, w), dtype=torch.float32, device=dev)
        # HBM keyframe tier: ground-truth RGB (u8) + depth (f32) of the store's
        # resident keyframes (store.py:427-489 LRU), dropped when the store
        # evicts the keyframe (its .dkf write-back is the store's)
        self._kf_dev: dict[int, _DeviceKeyframe] = {}
        store.keyframe_evict_hooks.append(self._drop_device_keyframe)
        store.keyframe_device_packer = self._pack_device_keyframe
        self._readback = torch.zeros(12, dtype=torch.float32, pin_memory=True)
        self._flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.cam = None
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.upload_keyframes_each_step = False   # e2e mode: GT from pinned host every step
        self.upload_side_stream = True   # the e2e upload overlaps the forward on its own stream
        self._pinned_kf: dict[int, tuple] = {}
        self._uniforms: dict[int, float] = {}
        self._eager_seen: dict = {}
        self._layout_cache: dict = {}   # visible ids -> (store.layout_version, (slots, n))
        self._tile_orders: dict[int, object] = {}   # keyframe id -> its longest-first tile schedule

    # -------------------------------------------------------------- inputs
    def add_keyframe(self, kf: Keyframe, index_usage: int | None = None) -> None:
        """store.keyframe_add + index.add (sim.py:264-268), without ingestion;
        the new keyframe's on-disk chunks start streaming in right away."""
        self.store.keyframe_add(kf)
        self.index.add(kf.id, kf.position,
                       usage_remaining=self.index.config.initial_usage if index_usage is None else index_usage)
        self.latest_kf = kf.id
        self._prefetch_view(kf.pose)

    def render_current(self, pose: Pose):
        """sim._Replay._render_current (sim.py:255-262) on the device: the
        visible chunks made resident and rendered into self.rgb / depth /
        alpha (overflow retried); returns the active-set size."""
        visible, _ = self._visible_for_pose(pose)
        ids = sorted(visible)
        if ids:
            self.store.ensure_resident(ids)
        slots, n = self.active.build(self.store.segments(ids))
        cam = camera_for(pose, self.intr)
        for _ in range(8):
            self.render.forward(self.store.slab.params, slots, n, cam, self.rgb, self.depth, self.alpha)
            c = self.render.counters()
            if not c["overflow"]:
                return n
            self.render.grow_instances(c["n_instances"])
            self.drop_graphs()
        raise DeviceFailure("tile-instance buffer kept overflowing")

    def ingest_keyframe(self, index: int, pose: Pose, rgb: np.ndarray, depth: np.ndarray) -> int:
        """sim._Replay.ingest_keyframe (sim.py:264-278) with the per-pixel work
        on the device: keyframe tier + index, the current view rendered in
        HBM, |LoG| scores of the keyframe's 8-bit ground truth and of the
        render (csrc/ingest.cu), the probability map down to the host for the
        reference's own draw (Generator.choice, seed (seed, 1, index)), the
        drawn pixels lifted on the device, inserted through the store's
        policy.  Returns the number of Gaussians inserted."""
        from .sample import DeviceSampler, sample_pixels
        cfg = self.sample_cfg
        kf = Keyframe(id=index, pose=pose, intrinsics=self.intr, rgb=rgb, depth=depth,
                      usage_remaining=self.index.config.initial_usage)
        self.add_keyframe(kf)
        self.render_current(pose)
        dk = self._device_keyframe(kf)
        if getattr(dk, "pending", None) is not None:
            self.torch.cuda.current_stream(self.device).wait_stream(dk.pending)
            dk.pending = None
        smp = getattr(self, "_sampler", None)
        if smp is None:
            smp = self._sampler = DeviceSampler(self.intr.width, self.intr.height, self.device)
        smp.scores_of(dk.rgb_u8, 0, cfg.log_sigma, cfg.kernel_radius)
        smp.scores_of(self.rgb, 1, cfg.log_sigma, cfg.kernel_radius)
        ps = smp.probability().cpu().numpy()
        self.d2h_bytes += ps.nbytes
        pixels = sample_pixels(ps, cfg.samples_per_keyframe, derive_seed(self.seed, 1, index))
        rec, _ = smp.lift(pixels, dk.depth, dk.rgb_u8, pose.rotation, pose.translation, self.intr, cfg)
        if not len(rec):
            return 0
        sh = np.zeros((len(rec), 48), np.float64)
        sh[:, [0, 16, 32]] = rec[:, 11:14]
        return self.store.insert_arrays(rec[:, 0:3], rec[:, 3:7], rec[:, 7:10], rec[:, 10], sh)

    def _pack_device_keyframe(self, kid: int, kf: Keyframe, path) -> bool:
        """The store evicts a dirty keyframe whose ground truth is in HBM:
        assemble its .dkf on the device (sm_keyframe_pack, byte-identical to
        diskformat.pack_keyframe) and hand it to the write-behind."""
        d = self._kf_dev.get(kid)
        if d is None:
            return False
        from .diskformat import keyframe_file_size, keyframe_header
        head = np.frombuffer(keyframe_header(kf), dtype=np.uint8).copy()
        w, h = kf.intrinsics.width, kf.intrinsics.height
        lib = _lib.load()

        def fill(pin):   # the kernel writes the file image straight into pinned host memory (UVA)
            _lib.check(lib.sm_keyframe_pack(head.ctypes.data_as(_lib.ctypes.c_void_p), _lib.ptr(d.rgb_u8),
                                            _lib.ptr(d.depth), w, h, _lib.ptr(pin), _lib.stream_handle()),
                       "keyframe_pack")
        self.store.streamer.write_file_async(path, keyframe_file_size(kf), fill)
        return True

    def _drop_device_keyframe(self, kid: int) -> None:
        self._kf_dev.pop(kid, None)
        self._tile_orders.pop(kid, None)
        # captured graphs of this keyframe read the dropped buffers
        graphs = getattr(self, "_graphs", {})
        stale = [k for k in graphs if k[0] == kid]
        if stale:
            lib = _lib.load()
            for k in stale:
                lib.sm_profile_graph_free(graphs.pop(k)[1])

    view_tile_order = True   # keep each keyframe's longest-first tile schedule

    def _tile_order(self, kf: Keyframe):
        if not self.view_tile_order:
            return None
        o = self._tile_orders.get(kf.id)
        if o is None:
            o = self._tile_orders[kf.id] = self.render.new_tile_order(kf.intrinsics.width, kf.intrinsics.height)
        return o

    def device_keyframe_ids(self) -> set[int]:
        return {k for k in self._kf_dev if k >= 0}

    def _device_keyframe(self, kf: Keyframe) -> _DeviceKeyframe:
        torch = self.torch
        if self.upload_keyframes_each_step:
            pin = self._pinned_kf.get(kf.id)
            if pin is None:
                pin = (torch.from_numpy(kf.rgb_u8()).pin_memory(), torch.from_numpy(kf.depth).pin_memory())
                self._pinned_kf[kf.id] = pin
            d = self._kf_dev.get(-1)
            if d is None:
                d = self._kf_dev[-1] = _DeviceKeyframe(torch.empty_like(pin[0], device=self.device),
                                                       torch.empty_like(pin[1], device=self.device))
            # H2D on a side stream, overlapped with the forward render (which
            # does not read the ground truth); the loss waits for it
            cur = torch.cuda.current_stream(self.device)
            if not self.upload_side_stream:   # (A/B: the copy in line with the forward)
                d.rgb_u8.copy_(pin[0], non_blocking=True)
                d.depth.copy_(pin[1], non_blocking=True)
                return d
            if not hasattr(self, "_up_stream"):
                self._up_stream = torch.cuda.Stream(device=self.device)
            self._up_stream.wait_stream(cur)   # the previous step's loss is done with d
            with torch.cuda.stream(self._up_stream):
                d.rgb_u8.copy_(pin[0], non_blocking=True)
                d.depth.copy_(pin[1], non_blocking=True)
            d.pending = self._up_stream
            return d
        d = self._kf_dev.get(kf.id)
        if d is None:
            d = _DeviceKeyframe(torch.as_tensor(kf.rgb_u8(), device=self.device),
                                torch.as_tensor(kf.depth, device=self.device))
            self._kf_dev[kf.id] = d
        return d

    def _visible_for_pose(self, pose: Pose) -> tuple[set[int], bool]:
        ext = self.store.coord_extent()
        if ext is None:
            return set(), False
        memo = self._view_memo
        key = (pose.translation.tobytes(), pose.rotation.tobytes(), self.store.generation)
        return self.cache.query(pose, self.intr, ChunkExtent(*ext), self.store.has_chunk,
                                self.store.generation, self.store.chunk_size,
                                compute=lambda: set(memo[1]) if memo is not None and memo[0] == key
                                else self._cull_view(pose))

    def _cull_view(self, pose: Pose) -> set[int]:
        """visible_chunks over the store's cached device chunk table (the
        brute-force candidates of culling.py:134-182, without rebuilding and
        uploading them for every cull)."""
        ids, coords = self.store.chunk_table()
        return {int(i) for i in cull_table(ids, coords, pose, self.intr, self.cull_cfg.max_distance_m,
                                           self.store.chunk_size)}

    _view_memo = None   # (pose bytes, chunk-set generation) -> the visible set _prefetch_view culled

    # ------------------------------------------------------------ device
    # single-keyframe steps: Adam fused into the backward (sm_render_backward_adam).  Measured
    # slower at C2 (0.900 vs 0.880 ms/step: the fused projection backward spills and its
    # one-thread-per-record Adam streams worse than K7's quarter threads), so off by default.
    fused_adam = False

    def _device_pass(self, kf: Keyframe, slots, n: int, backward: bool = True, adam: bool = False):
        """fwd -> loss(+grad) -> bwd for one keyframe; grads accumulate in the
        slab, or with adam=True the Adam step is applied by the backward
        itself (no gradient buffer) or by K7 right after it."""
        slab = self.store.slab
        cam = camera_for(kf.pose, kf.intrinsics)
        dk = self._device_keyframe(kf)
        self.render.forward(slab.params, slots, n, cam, self.rgb, self.depth, self.alpha,
                            tile_order=self._tile_order(kf))
        if getattr(dk, "pending", None) is not None:   # join the side-stream upload
            self.torch.cuda.current_stream(self.device).wait_stream(dk.pending)
            dk.pending = None
        self.loss.run(self.rgb, self.depth, dk.rgb_u8, None, dk.depth, 3, self.weights,
                      self.d_rgb if backward else None, self.d_depth if backward else None)
        if backward and n and adam and self.fused_adam:
            self.render.backward_adam(slab.params, slots, n, cam, self.d_rgb, self.d_depth, None, slab.adam_m,
                                      slab.adam_v, self._adam_c, self.render.overflow_flag())
        elif backward and n:
            self.render.backward(slab.params, slots, n, cam, self.d_rgb, self.d_depth, None, slab.grads)
            if adam:
                self._adam(slots, n)

    def _adam(self, slots, n: int) -> None:
        s = self.store.slab
        rc = _lib.load().sm_adam_step(_lib.ptr(s.params), _lib.ptr(s.adam_m), _lib.ptr(s.adam_v),
                                      _lib.ptr(s.grads), _lib.ptr(slots), int(n),
                                      self._adam_c, _lib.ptr(self.render.overflow_flag()),
                                      _lib.stream_handle())
        _lib.check(rc, "adam_step")

    def _queue_readback(self) -> None:
        """D2H copy of {loss[4], n_instances, overflow} into pinned memory (async)."""
        rb = self._readback
        rb[:4].copy_(self.loss.out, non_blocking=True)
        rb[4:11].copy_(self.render.ws[:28].view(self.torch.float32), non_blocking=True)

    def _finish_readback(self) -> tuple[float, bool]:
        self.torch.cuda.current_stream(self.device).synchronize()
        self.d2h_bytes += 44
        v = self._readback.numpy()
        ctr = v[4:11].view(np.uint32)   # sm_render_counters[0:7]
        self.counter_instances += int(ctr[0])
        self.counter_visited += int(ctr[6])   # instances the backward revisited
        return float(v[0]), bool(ctr[1])

    counter_speculative = 0   # steps whose graph was launched before their host policy

    def reset_counters(self) -> None:
        self.counter_speculative = 0
        self.counter_steps = 0
        self.counter_gaussians = 0
        self.counter_instances = 0
        self.counter_visited = 0

    counter_steps = counter_gaussians = counter_instances = counter_visited = 0
    counter_replays = counter_eager = 0
    use_graphs = True
    capture_after = 2   # eager visits of a (keyframe, active set) before its graph is captured

    _while_gpu = None

    def _run_while_gpu(self) -> None:
        """Host bookkeeping of the current step that does not need its loss
        (store flags, look-ahead prefetch), run once while the device pass is
        in flight."""
        f, self._while_gpu = self._while_gpu, None
        if f is not None:
            f()
            self._lookahead_prefetch()

    prefetch_lookahead = True   # read the next draw's candidate views' chunks ahead of use

    def _lookahead_prefetch(self) -> None:
        """Speculative reads for the next step: every keyframe
        the next draw can pick (the candidate set of the latest keyframe,
        select.py:115-121) may need chunks that are on disk; their files are
        read into pinned memory on the streamer's reader threads while the
        device works.  No policy effect: the visibility sets come from the
        cache without touching its LRU (or are computed without inserting)
        and the store's residency is unchanged until ensure_resident."""
        store = self.store
        if not self.prefetch_lookahead or not store.has_disk_chunks() or self.latest_kf is None:
            return
        ext = store.coord_extent()
        if ext is None:
            return
        key = (self.latest_kf, self.index.version, store.generation)
        memo = getattr(self, "_ahead", None)
        if memo is None or memo[0] != key or memo[2] >= 8:
            # the union of the candidates' views (only views the cache already
            # knows: no cull on the step's host path; a new keyframe's view is
            # computed once, in add_keyframe); rebuilt when the candidate set or
            # the chunk set changes, and every 8 steps for views cached since
            try:
                cands = candidate_set(self.index.position_of(self.latest_kf), self.index)
            except EmptyCandidates:
                cands = [self.latest_kf]
            want: set[int] = set()
            for c in cands:
                kf = store._keyframes.get(c)
                if kf is None:
                    continue
                vis = self.cache.peek(kf.pose, self.intr, store.generation, store.chunk_size)
                if vis is not None:
                    want.update(vis)
            memo = self._ahead = [key, sorted(want), 0]
        memo[2] += 1
        want = memo[1]
        if want and store.resident_count_of(want) < len(want):
            store.prefetch(want)

    def _prefetch_view(self, pose: Pose) -> None:
        """A new keyframe's on-disk chunks start streaming in (one cull, no
        visibility-cache insertion: no policy effect)."""
        store = self.store
        ext = store.coord_extent()
        if not self.prefetch_lookahead or ext is None or not store.has_disk_chunks():
            return
        vis = self._cull_view(pose)
        # the step that first draws this keyframe misses the visibility cache
        # with exactly this pose and chunk set: it takes this set, not a second cull
        self._view_memo = ((pose.translation.tobytes(), pose.rotation.tobytes(), store.generation),
                           frozenset(vis))
        store.prefetch(sorted(vis))

    def _precompute_next_draw(self) -> None:
        """The next single-GPU step's uniform draw depends only on its derived
        seed (not on this step's loss): compute it while the GPU works."""
        nxt = self.step_counter + 1
        if nxt not in self._uniforms:
            self._uniforms = {nxt: draw_uniform(derive_seed(self.seed, 2, nxt))}

    def _graph_key(self, kf: Keyframe, slots, n: int, dp: bool = False):
        """A captured graph bakes in the camera (sm_camera is copied by value
        into the kernel arguments), so the key carries the pose bytes and the
        intrinsics: a pose correction (store.update_keyframe_pose, the
        reference's loopclose.py:183) re-captures instead of replaying the old
        camera."""
        s = self.store.slab
        cam = (kf.pose.rotation.tobytes(), kf.pose.translation.tobytes(), kf.intrinsics)
        return (kf.id, cam, slots.data_ptr(), n, s.params.data_ptr(), s.grads.data_ptr(), s.adam_m.data_ptr(),
                self.render.ws.data_ptr(), self.upload_keyframes_each_step, dp, self.fused_adam)

    def drop_graphs(self) -> None:
        lib = _lib.load()
        for _, gid in getattr(self, "_graphs", {}).values():
            lib.sm_profile_graph_free(gid)
        self._graphs = {}

    def _capture(self, kf: Keyframe, slots, n: int, dp: bool = False):
        """Capture fwd -> loss -> bwd -> Adam -> readback as one CUDA graph
        (dp: fwd -> loss -> bwd only; the all-reduce and Adam follow eagerly)."""
        torch, lib = self.torch, _lib.load()
        if not hasattr(self, "_cap_stream"):
            self._cap_stream = torch.cuda.Stream(device=self.device)
            self._graphs = {}
        torch.cuda.current_stream(self.device).synchronize()
        g = torch.cuda.CUDAGraph()
        gid = lib.sm_profile_capture_begin()
        try:
            # thread-local capture: the streamer's reader / writer threads keep
            # synchronising events and page-locking buffers while a graph is
            # captured, which would invalidate a global-mode capture
            with torch.cuda.graph(g, stream=self._cap_stream, capture_error_mode="thread_local"):
                self._device_pass(kf, slots, n, adam=not dp)
                if not dp:
                    self._queue_readback()
        finally:
            lib.sm_profile_capture_end()
        key = self._graph_key(kf, slots, n, dp)
        # graphs of this keyframe under an older camera can never replay again
        for k in [k for k in self._graphs if k[0] == kf.id and k[1] != key[1]]:
            lib.sm_profile_graph_free(self._graphs.pop(k)[1])
        self._graphs[key] = (g, gid)

    def _dp_device_pass(self, kf: Keyframe, slots, n: int) -> None:
        """fwd -> loss -> bwd of this rank's keyframe: graph replay when captured,
        else eager (captured on the second visit, like train_view)."""
        if self.upload_keyframes_each_step:
            self.h2d_bytes += kf.intrinsics.width * kf.intrinsics.height * 7
        self.render.ensure(n, kf.intrinsics.width, kf.intrinsics.height)
        key = self._graph_key(kf, slots, n, True)
        entry = getattr(self, "_graphs", {}).get(key) if self.use_graphs else None
        if entry is not None:
            g, gid = entry
            g.replay()
            self.counter_replays += 1
            _lib.load().sm_profile_graph_replayed(gid)
            return
        self.counter_eager += 1
        self._device_pass(kf, slots, n)
        if self.use_graphs and n:
            seen = self._eager_seen.get(key, 0) + 1
            self._eager_seen[key] = seen
            if seen >= self.capture_after:
                self._capture(kf, slots, n, dp=True)
                self._eager_seen.pop(key, None)

    def _speculate(self) -> None:
        """While the device pass runs: for every keyframe the next draw can
        pick, what the next step's policy would hand the device if nothing
        had to be paged -- its visible set as the visibility cache would
        answer (peek: no LRU change), the active-set slots from the layout
        cache and the captured graph.  The next step validates the entry of
        the keyframe it draws (same latest keyframe, store generation, layout
        and cache state, every visible chunk resident) and launches that graph
        before running the policy, which then only has to agree with it; the
        host policy time leaves the gap between device passes."""
        self._spec = None
        store = self.store
        graphs = getattr(self, "_graphs", None)
        if not self.use_graphs or not graphs or self.latest_kf is None or store.coord_extent() is None:
            return
        try:
            cands = candidate_set(self.index.position_of(self.latest_kf), self.index)
        except EmptyCandidates:
            cands = [self.latest_kf]
        self._spec_cands = (self.latest_kf, self.index.version, cands)
        gen, lv = store.generation, store.layout_version
        out = {}
        for c in cands:
            kf = store._keyframes.get(c)   # resident keyframes only (no load, no LRU tick)
            if kf is None:
                continue
            res = self.cache.peek(kf.pose, self.intr, gen, store.chunk_size)
            if not res:
                continue
            ids_t = tuple(sorted(res))
            ent = self._layout_cache.get(ids_t)
            if ent is None or ent[0] != lv:
                continue
            slots, n = ent[1]
            key = self._graph_key(kf, slots, n)
            entry = graphs.get(key)
            if entry is not None:
                out[c] = (ids_t, slots, n, kf, entry, key)
        self._spec = (self.latest_kf, gen, lv, self.cache.version, out)

    _spec = None
    _spec_cands = None

    def _take_speculation(self, selected: int):
        sp, self._spec = self._spec, None
        if sp is None:
            return None
        latest, gen, lv, cv, out = sp
        st = self.store
        if (latest != self.latest_kf or gen != st.generation or lv != st.layout_version
                or cv != self.cache.version):
            return None
        e = out.get(selected)
        if e is None or st._keyframes.get(selected) is not e[3] or st.resident_count_of(e[0]) != len(e[0]):
            return None
        if self._graph_key(e[3], e[1], e[2]) != e[5] or self._graphs.get(e[5]) is not e[4]:
            return None   # mode / workspace changed, or the graph was dropped
        return e

    def train_view(self, kf: Keyframe, slots, n: int, launched: bool = False) -> float:
        """One device iteration with overflow recovery; returns the loss.

        The first visit of a (keyframe, active set) runs eagerly and then
        captures the whole device pass as a CUDA graph; later visits replay it
        (one launch instead of ~45), which the B200 front end needs here.
        """
        if self.upload_keyframes_each_step:   # GT RGB (u8) + depth (f32) cross PCIe every step
            self.h2d_bytes += kf.intrinsics.width * kf.intrinsics.height * 7
        self.render.ensure(n, kf.intrinsics.width, kf.intrinsics.height)
        self.last_n = n
        graphs = getattr(self, "_graphs", {})
        entry = graphs.get(self._graph_key(kf, slots, n)) if self.use_graphs else None
        if launched and entry is None:
            raise RuntimeError("speculatively launched graph not found")
        if entry is not None:
            g, gid = entry
            if not launched:   # (optimization_step launched it speculatively)
                g.replay()
            self.counter_replays += 1
            self._precompute_next_draw()   # host work overlapped with the GPU pass
            self._run_while_gpu()
            self._speculate()
            loss, overflow = self._finish_readback()
            _lib.load().sm_profile_graph_replayed(gid)
            if not overflow:
                self.counter_steps += 1
                self.counter_gaussians += n
                return loss
            self.store.slab.grads.zero_()
            self.render.grow_instances(self.render.counters()["n_instances"])
            self.drop_graphs()
        for _ in range(6):
            self.counter_eager += 1
            self._device_pass(kf, slots, n, adam=True)
            self._queue_readback()
            self._run_while_gpu()
            loss, overflow = self._finish_readback()
            if not overflow:
                self.counter_steps += 1
                self.counter_gaussians += n
                if self.use_graphs and n:
                    # capture on the second eager visit of a (keyframe, active
                    # set): one-off sets (a moving camera paging chunks in and
                    # out) never pay the capture
                    key = self._graph_key(kf, slots, n)
                    seen = self._eager_seen.get(key, 0) + 1
                    self._eager_seen[key] = seen
                    if seen >= self.capture_after:
                        self._capture(kf, slots, n)
                        self._eager_seen.pop(key, None)
                    elif len(self._eager_seen) > 4096:
                        self._eager_seen.clear()
                return loss
            self.store.slab.grads.zero_()
            self.render.grow_instances(self.render.counters()["n_instances"])
            self.drop_graphs()
        raise DeviceFailure("tile-instance buffer kept overflowing")

    def warm_graphs(self) -> None:
        """Run one device iteration per resident keyframe (capturing its graph)."""
        after, self.capture_after = self.capture_after, 1
        try:
            for kid in sorted(self.store.resident_keyframe_ids()):
                kf = self.store.keyframe_get(kid)
                ids = sorted(self._visible_for_pose(kf.pose)[0])
                if ids:
                    self.store.ensure_resident(ids)
                slots, n = self.active.build(self.store.segments(ids))
                self.train_view(kf, slots, n)
                if ids:
                    self.store.mark_trained(ids)
        finally:
            self.capture_after = after

    # --------------------------------------------------------------- step
    def optimization_step(self, frame_idx: int, step_idx: int, inserted: int = 0) -> FrameMetrics:
        store, stats = self.store, self.store.stats
        io0, loads0, ev0 = stats.io_nanos, stats.chunk_loads, stats.chunk_evictions
        if self.latest_kf is None:
            raise RuntimeError("no keyframe ingested yet")
        sc = self._spec_cands   # (prepared while the previous pass ran)
        if sc is not None and sc[0] == self.latest_kf and sc[1] == self.index.version:
            candidates = sc[2]
        else:
            try:
                candidates = candidate_set(self.index.position_of(self.latest_kf), self.index)
            except EmptyCandidates:
                candidates = [self.latest_kf]
        pre = self._uniforms.pop(self.step_counter, None)
        seed = derive_seed(self.seed, 2, self.step_counter) if pre is None else None   # else unused
        selected = select_keyframe(candidates, self.index, seed, uniform=pre)
        spec = self._take_speculation(selected)
        if spec is not None:   # launch first; the policy below then only confirms it
            spec[4][0].replay()
            self.counter_speculative += 1
        kf = store.keyframe_get(selected)
        visible, _ = self._visible_for_pose(kf.pose)
        # overlap(visible, resident) (select.py), counted without building the sets
        overlap_val = store.resident_count_of(visible) / len(visible) if visible else None
        ids = sorted(visible)
        if ids:
            store.ensure_resident(ids)
        ids_t = tuple(ids)
        ent = self._layout_cache.get(ids_t)
        if ent is not None and ent[0] == store.layout_version:   # same chunks at the same rows
            slots, n = ent[1]
        else:
            segs = store.segments(ids)
            if ent is not None and ent[1][1] == sum(c for _, c in segs):
                # a chunk of this view was paged out and back in elsewhere:
                # refill its slot buffer in place, its graphs keep replaying
                slots, n = self.active.rebuild(ent[1][0], segs)
            else:
                slots, n = self.active.build(segs)
            self._layout_cache.pop(ids_t, None)
            self._layout_cache[ids_t] = (store.layout_version, (slots, n))
            while len(self._layout_cache) > 64:
                self._layout_cache.pop(next(iter(self._layout_cache)))
        if spec is not None and (ids_t != spec[0] or slots.data_ptr() != spec[1].data_ptr() or n != spec[2]):
            raise RuntimeError("speculative launch diverged from the step's policy")

        def bookkeeping():   # needs no loss: runs while the GPU works (train_view)
            store.mark_keyframe_dirty(selected)
            if ids:
                store.mark_trained(ids)
        self._while_gpu = bookkeeping
        loss = self.train_view(kf, slots, n, launched=spec is not None)
        self._run_while_gpu()   # (if train_view did not)
        record_loss(selected, loss, self.index)
        kf.last_loss = loss
        kf.usage_remaining = self.index.usage_of(selected)
        self.step_counter += 1
        io = stats.io_nanos - io0
        step_ns = (io + NS_PER_RENDERED_GAUSSIAN * n + NS_PER_PIXEL * self.intr.width * self.intr.height
                   + NS_PER_INSERTED_GAUSSIAN * inserted + NS_STEP_BASE)
        row = FrameMetrics(frame_idx, step_idx, stats.active_gaussians, stats.active_chunks,
                           stats.active_keyframes, stats.chunk_loads - loads0,
                           stats.chunk_evictions - ev0, io, step_ns, selected, overlap_val, loss)
        self.rows.append(row)
        return row

    # ------------------------------------------------------ data parallel
    def _packed_buffer(self, n: int):
        buf = getattr(self, "_packed", None)
        if buf is None or buf.shape[0] < n:
            buf = self._packed = self.torch.empty((max(int(n * 1.25), 1024), 16), dtype=self.torch.float32,
                                                  device=self.device)
        return buf

    def optimization_step_dp(self, frame_idx: int, step_idx: int, world: int, rank: int,
                             group=None, inserted: int = 0, keyframes: int | None = None) -> list[FrameMetrics]:
        """One data-parallel mapping step over K keyframes.

        Every rank runs the same host policy (same derived seeds), so the K
        keyframe draws, their visible sets and the residency of the
        replicated active tier are identical everywhere.  Rank r renders and
        backpropagates keyframes r, r + G, ... into its slab gradients; the
        union active set's gradient records are packed (K6 output rows ->
        [n_union, 16]) and summed with one all-reduce, together with the
        per-keyframe losses and an overflow count; every rank then applies
        the same Adam update over the union from the summed buffer.  The
        host reads the losses while Adam runs (the next draw needs them).
        K = 1, G = 1 is bit-identical to ``optimization_step``.
        """
        torch = self.torch
        k = int(keyframes or world)
        store, stats = self.store, self.store.stats
        io0, loads0, ev0 = stats.io_nanos, stats.chunk_loads, stats.chunk_evictions
        selected = dp_select(self.index, self.latest_kf, self.seed, self.step_counter, k)
        kfs = [store.keyframe_get(s) for s in selected]
        vis = [self._visible_for_pose(kf.pose)[0] for kf in kfs]
        union = sorted(set().union(*vis))
        overlap_val = overlap(set(union), store.resident_chunk_ids()) if union else None
        if union:
            store.ensure_resident(union)
        if getattr(self, "_union_set", None) is None:
            self._union_set = _ActiveSet(self.device)
        if getattr(self, "_lossbuf", None) is None or self._lossbuf.numel() != k + 1:
            self._lossbuf = torch.zeros(k + 1, dtype=torch.float32, device=self.device)
            self._loss_host = torch.zeros(k + 1, dtype=torch.float32, pin_memory=True)
        mine = owned_keyframes(k, world, rank)
        slots_u, n_u = self._union_set.build(store.segments(union))
        packed = self._packed_buffer(n_u)
        lib, stream = _lib.load(), _lib.stream_handle()
        buf, host = self._lossbuf, self._loss_host
        n_mine = 0
        for _ in range(6):
            buf.zero_()
            n_mine = 0
            for j in mine:
                slots_j, n_j = self.active.build(store.segments(sorted(vis[j])))
                self._dp_device_pass(kfs[j], slots_j, n_j)
                buf[j:j + 1].copy_(self.loss.out[:1])
                buf[k:k + 1].add_(self.render.overflow_flag().float())
                n_mine += n_j
            _lib.check(lib.sm_pack_grads(_lib.ptr(store.slab.grads), _lib.ptr(slots_u), n_u,
                                         _lib.ptr(packed), stream), "pack_grads")
            allreduce_step(packed[:n_u], buf, group)
            host.copy_(buf, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            # Adam over the union from the summed records; skipped on the device
            # when any rank overflowed (the overflow sum's float bits are non-zero)
            _lib.check(lib.sm_adam_step_packed(_lib.ptr(store.slab.params), _lib.ptr(store.slab.adam_m),
                                               _lib.ptr(store.slab.adam_v), _lib.ptr(packed), _lib.ptr(slots_u),
                                               n_u, self._adam_c, _lib.ptr(buf[k:k + 1]), stream),
                       "adam_step_packed")
            ev.synchronize()
            self.d2h_bytes += 4 * (k + 1)
            if host[k] == 0:
                break
            self.render.grow_instances(self.render.counters()["n_instances"] * 2)
            self.drop_graphs()
        else:
            raise DeviceFailure("tile-instance buffer kept overflowing")
        self.counter_steps += 1
        self.counter_gaussians += n_mine
        losses = host.numpy().astype(np.float64)
        rows = []
        for j, (sel, kf) in enumerate(zip(selected, kfs)):
            loss = float(losses[j])
            record_loss(sel, loss, self.index)
            kf.last_loss = loss
            kf.usage_remaining = self.index.usage_of(sel)
            if sel in store.resident_keyframe_ids():
                store.mark_keyframe_dirty(sel)
            io = stats.io_nanos - io0
            step_ns = (io + NS_PER_RENDERED_GAUSSIAN * n_u + NS_PER_PIXEL * self.intr.width *
                       self.intr.height * k + NS_PER_INSERTED_GAUSSIAN * inserted + NS_STEP_BASE)
            rows.append(FrameMetrics(frame_idx, step_idx, stats.active_gaussians, stats.active_chunks,
                                     stats.active_keyframes, stats.chunk_loads - loads0,
                                     stats.chunk_evictions - ev0, io, step_ns, sel, overlap_val, loss))
        if union:
            store.mark_trained(union)
        self.step_counter += 1
        self.rows.extend(rows)
        return rows
