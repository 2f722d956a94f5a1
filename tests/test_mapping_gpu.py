"""The mapping step on the GPU: Adam vs its oracle, training progress, CUDA-graph
replay identical to eager execution, paging under a budget, determinism."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_adam_kernel_matches_oracle(cuda):
    import torch

    from oracle import oracle as O
    from paper_2511_23030_b200 import _lib
    from paper_2511_23030_b200.mapping import AdamSettings
    rng = np.random.default_rng(3)
    n = 1000
    p = np.zeros((n, 16), np.float32)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    p[:, 0:3] = rng.normal(size=(n, 3))
    p[:, 3:7] = q
    p[:, 7:10] = rng.uniform(0.01, 0.1, (n, 3))
    p[:, 10] = rng.uniform(0.1, 0.9, n)
    p[:, 11:14] = rng.normal(size=(n, 3))
    s = AdamSettings()
    lr = np.array([s.lr_position] * 3 + [s.lr_rotation] * 4 + [s.lr_scale] * 3 + [s.lr_opacity] + [s.lr_sh0] * 3)
    params = torch.as_tensor(p, device="cuda")
    m = torch.zeros_like(params)
    v = torch.zeros_like(params)
    ref_p = p[:, :14].astype(np.float64).copy()
    ref_m = np.zeros((n, 14))
    ref_v = np.zeros((n, 14))
    for step in range(1, 4):
        g = rng.normal(size=(n, 14)).astype(np.float32)
        grads = torch.zeros_like(params)
        grads[:, :14] = torch.as_tensor(g, device="cuda")
        _lib.check(_lib.load().sm_adam_step(_lib.ptr(params), _lib.ptr(m), _lib.ptr(v), _lib.ptr(grads),
                                            None, n, s.to_c(), None, _lib.stream_handle()))
        assert float(grads.abs().max()) == 0.0   # K7 zeroes the accumulator
        for k in range(14):   # per-scalar Adam in fp64 (torch.optim.Adam formula)
            col_p, col_m, col_v = ref_p[:, k].copy(), ref_m[:, k].copy(), ref_v[:, k].copy()
            O.adam(col_p, col_m, col_v, g[:, k].astype(np.float64), lr[k], s.beta1, s.beta2, s.eps, step)
            ref_p[:, k], ref_m[:, k], ref_v[:, k] = col_p, col_m, col_v
        # invariants the store requires (core.py:186-190)
        ref_p[:, 3:7] /= np.linalg.norm(ref_p[:, 3:7], axis=1, keepdims=True)
        ref_p[:, 7:10] = np.maximum(ref_p[:, 7:10], s.min_scale)
        ref_p[:, 10] = np.clip(ref_p[:, 10], 0, 1)
    got = params.cpu().numpy()[:, :14].astype(np.float64)
    assert np.abs(got - ref_p).max() <= 1e-6 * (1 + np.abs(ref_p)).max()
    assert np.all(m.cpu().numpy()[:, 14] == 3.0)


def _c1_engine(tmp_path, budget=12_000, n=20_000, use_graphs=True, keyframe_budget=400):
    from paper_2511_23030_b200.workloads import build_c1
    eng = build_c1(n=n, keyframes=10, budget=budget, store_dir=tmp_path, keyframe_budget=keyframe_budget)
    eng.use_graphs = use_graphs
    return eng


def test_training_reduces_loss(cuda, tmp_path):
    eng = _c1_engine(tmp_path, budget=100_000)
    kf = eng.store.keyframe_get(4)
    ids = sorted(eng._visible_for_pose(kf.pose)[0])
    eng.store.ensure_resident(ids)
    slots, n = eng.active.build(eng.store.segments(ids))
    losses = [eng.train_view(kf, slots, n) for _ in range(60)]
    assert all(np.isfinite(losses))
    assert np.mean(losses[-5:]) < 0.9 * np.mean(losses[:5]), (losses[:5], losses[-5:])


def test_graph_replay_equals_eager(cuda, tmp_path):
    """Graph replay (incl. speculative launches: the drawn keyframe's graph
    starts before its policy runs) = eager execution, bit for bit."""
    import torch
    a = _c1_engine(tmp_path / "a", budget=100_000, use_graphs=True)
    b = _c1_engine(tmp_path / "b", budget=100_000, use_graphs=False)
    for s in range(12):
        ra = a.optimization_step(0, s)
        rb = b.optimization_step(0, s)
        assert ra.selected_kf == rb.selected_kf and ra.loss == rb.loss
    sa, sb = a.store.slab, b.store.slab
    hw = sa.high_water()
    assert torch.equal(sa.params[:hw], sb.params[:hw])
    assert torch.equal(sa.adam_m[:hw], sb.adam_m[:hw])
    assert a.counter_speculative > 0   # steps launched before their host policy ran


def test_dp_step_world1_equals_single_step(cuda, tmp_path):
    """optimization_step_dp with one rank = optimization_step (same draws,
    same device pass, same Adam) -- the N>1 path minus the collectives."""
    import torch
    a = _c1_engine(tmp_path / "a", budget=100_000)
    b = _c1_engine(tmp_path / "b", budget=100_000)
    for s in range(6):
        ra = a.optimization_step(0, s)
        (rb,) = b.optimization_step_dp(0, s, world=1, rank=0)
        assert ra.selected_kf == rb.selected_kf and ra.loss == rb.loss
    hw = a.store.slab.high_water()
    assert torch.equal(a.store.slab.params[:hw], b.store.slab.params[:hw])


def test_paging_steps_are_deterministic(cuda, tmp_path):
    """Budget 12k < 20k splats: the steps load and evict chunks; two identical
    runs give byte-identical metrics (test_acceptance.py criterion 10)."""
    rows = []
    for name in ("x", "y"):
        eng = _c1_engine(tmp_path / name, budget=12_000)
        out = [eng.optimization_step(f, s).csv_row() for f in range(3) for s in range(5)]
        rows.append(out)
        st = eng.store.stats
        assert st.chunk_evictions > 0 and st.chunk_writes > 0
        assert st.budget_overshoot == max(0, st.active_gaussians - 12_000)
    assert rows[0] == rows[1]


def test_paging_keeps_graphs_and_training(cuda, tmp_path):
    """Paging never changes the training, and a view whose chunks come back at
    other slab rows keeps its CUDA graph (its slot buffer is refilled in
    place).  (1) Under a paging budget: same keyframe draws and bit-identical
    losses as the all-resident run and as an eager run.  (2) Graph-captured
    views, then every chunk evicted and reloaded in reverse order (new rows):
    the next steps replay the captured graphs after an in-place refill and
    still equal the eager run."""
    runs = {}
    for name, budget, graphs in (("resident", 100_000, True), ("paged", 12_000, True),
                                 ("paged_eager", 12_000, False)):
        eng = _c1_engine(tmp_path / name, budget=budget, use_graphs=graphs)
        runs[name] = [(r.selected_kf, r.loss) for r in (eng.optimization_step(f, s)
                                                        for f in range(4) for s in range(10))]
        if name == "paged":
            assert eng.store.stats.chunk_evictions > 0 and eng.counter_replays > 0
    assert runs["paged"] == runs["resident"] == runs["paged_eager"]
    a = _c1_engine(tmp_path / "ga", budget=100_000, use_graphs=True)
    b = _c1_engine(tmp_path / "gb", budget=100_000, use_graphs=False)
    for s in range(12):
        assert a.optimization_step(0, s).loss == b.optimization_step(0, s).loss
    for eng in (a, b):
        st = eng.store
        st.evict_lru(st.stats.active_gaussians, protected=set())
        st.ensure_resident(sorted(st.known_chunk_ids())[::-1])
    replays = a.counter_replays
    for s in range(12, 24):
        ra, rb = a.optimization_step(0, s), b.optimization_step(0, s)
        assert (ra.selected_kf, ra.loss) == (rb.selected_kf, rb.loss)
    assert a.active.rebuilds > 0 and a.counter_replays > replays


def test_cached_chunk_table_cull_equals_visible_chunks(cuda, tmp_path):
    """The engine culls over the store's cached device chunk table; across
    paging (chunks created, evicted, reloaded) it returns exactly
    visible_chunks' brute-force answer over the known chunks."""
    from paper_2511_23030_b200.culling import ChunkExtent, visible_chunks
    eng = _c1_engine(tmp_path, budget=12_000)
    st = eng.store
    for f in range(3):
        for s in range(4):
            eng.optimization_step(f, s)
        for kid in sorted(st.resident_keyframe_ids()):
            pose = st.keyframe_get(kid).pose
            want = visible_chunks(pose, eng.intr, ChunkExtent(*st.coord_extent()), st.has_chunk, eng.cull_cfg,
                                  st.chunk_size, candidates=st.known_chunk_ids())
            assert eng._cull_view(pose) == want


def test_render_through_store_matches_oracle(cuda, tmp_path):
    """The active set rendered from the slab equals the oracle render of the
    same splats gathered in sorted-chunk-id order (sim.py:236-253)."""
    import torch

    from oracle import oracle as O
    from paper_2511_23030_b200.renderloss import camera_for
    eng = _c1_engine(tmp_path, budget=100_000)
    kf = eng.store.keyframe_get(2)
    ids = sorted(eng._visible_for_pose(kf.pose)[0])
    eng.store.ensure_resident(ids)
    slots, n = eng.active.build(eng.store.segments(ids))
    eng.render.forward(eng.store.slab.params, slots, n, camera_for(kf.pose, kf.intrinsics),
                       eng.rgb, eng.depth, eng.alpha)
    torch.cuda.synchronize()
    p = eng.store.slab.params[slots[:n].long()].cpu().numpy().astype(np.float64)
    i = kf.intrinsics
    ref = O.render_arrays(p[:, 0:3], p[:, 3:7], p[:, 7:10], p[:, 10], p[:, 11:14], kf.pose.rotation,
                          kf.pose.translation, i.fx, i.fy, i.cx, i.cy, i.near, i.width, i.height)
    assert np.abs(eng.rgb.cpu().numpy() - ref[0]).max() <= 1e-4
    assert np.abs(eng.alpha.cpu().numpy() - ref[2]).max() <= 1e-4


def test_device_keyframe_tier_follows_store_lru(cuda, tmp_path):
    """The HBM keyframe tier holds ground truth only for the store's resident
    keyframes (store.py:427-489 LRU): keyframes the store evicts (and writes
    as .dkf) leave HBM, reloads come back from disk bit-exact, so training is
    identical to an unbounded keyframe tier."""
    import torch
    a = _c1_engine(tmp_path / "a", budget=100_000, keyframe_budget=3)
    b = _c1_engine(tmp_path / "b", budget=100_000)
    for s in range(16):
        ra = a.optimization_step(0, s)
        rb = b.optimization_step(0, s)
        assert ra.selected_kf == rb.selected_kf and ra.loss == rb.loss
        assert a.device_keyframe_ids() <= a.store.resident_keyframe_ids()
        assert len(a.store.resident_keyframe_ids()) <= 3
        # graphs captured for an evicted keyframe read its dropped buffers: gone too
        assert {k[0] for k in getattr(a, "_graphs", {})} <= a.store.resident_keyframe_ids()
    for kid in (0, 1, 2):   # evicted keyframes come back from their .dkf files
        losses = []
        for e in (a, b):
            kf = e.store.keyframe_get(kid)
            ids = sorted(e._visible_for_pose(kf.pose)[0])
            e.store.ensure_resident(ids)
            slots, n = e.active.build(e.store.segments(ids))
            losses.append(e.train_view(kf, slots, n))
        assert losses[0] == losses[1], kid
        assert a.device_keyframe_ids() <= a.store.resident_keyframe_ids()
    assert a.store.stats.keyframe_writes > 0 and a.store.stats.keyframe_loads > 0
    hw = a.store.slab.high_water()
    assert torch.equal(a.store.slab.params[:hw], b.store.slab.params[:hw])


def test_instance_overflow_recovers_identically(cuda, tmp_path):
    """A render workspace too small for the step's tile instances flags
    overflow (device counter, no partial image), the step skips Adam, grows
    the workspace and retries: results equal a run that never overflowed."""
    import torch
    a = _c1_engine(tmp_path / "a", budget=100_000)
    b = _c1_engine(tmp_path / "b", budget=100_000)
    assert a.optimization_step(0, 0).loss == b.optimization_step(0, 0).loss
    d = a.render.dims
    a.render.dims = type(d)(d.max_gaussians, 4096, d.width, d.height)   # far below the need
    a.render.ws = torch.empty(a.render.lib.sm_render_workspace_size(a.render.dims), dtype=torch.uint8,
                              device="cuda")
    a.drop_graphs()
    for s in range(1, 5):
        ra = a.optimization_step(0, s)
        rb = b.optimization_step(0, s)
        assert ra.selected_kf == rb.selected_kf and ra.loss == rb.loss
    assert a.render.dims.max_instances > 4096
    hw = a.store.slab.high_water()
    assert torch.equal(a.store.slab.params[:hw], b.store.slab.params[:hw])


def test_keyframes_arriving_mid_run_graphs_equal_eager(cuda, tmp_path):
    """Keyframes joining between steps (a moving camera): the speculative
    launch and the graph cache must notice the new latest keyframe and the
    changed candidate set -- graph replay stays bit-identical to eager runs."""
    import torch

    from paper_2511_23030_b200.core import Keyframe
    from paper_2511_23030_b200.synthetic import C1_INTR, perturbed
    from paper_2511_23030_b200.workloads import _gt_frames, c1_poses, c1_scene
    engines = [_c1_engine(tmp_path / "a", budget=100_000, use_graphs=True),
               _c1_engine(tmp_path / "b", budget=100_000, use_graphs=False)]
    poses = c1_poses(14)[10:]   # four more keyframes further along the trajectory
    frames = _gt_frames(perturbed(c1_scene(20_000), 49), poses, C1_INTR, torch.device("cuda"))
    step = 0
    for k, (pose, (rgb, depth)) in enumerate(zip(poses, frames)):
        for e in engines:
            e.add_keyframe(Keyframe(id=100 + k, pose=pose, intrinsics=C1_INTR, rgb=rgb, depth=depth))
        for _ in range(4):
            ra, rb = (e.optimization_step(k, step) for e in engines)
            assert ra.selected_kf == rb.selected_kf and ra.loss == rb.loss, step
            step += 1
    sa, sb = engines[0].store.slab, engines[1].store.slab
    hw = sa.high_water()
    assert torch.equal(sa.params[:hw], sb.params[:hw])


def test_pose_update_recaptures_graph(cuda, tmp_path):
    """store.update_keyframe_pose (the reference's loopclose.py:183 call) by
    less than the visibility cache's pose quantum keeps the visible set, the
    slots and the layout; the captured graph must not replay the old camera.
    Graph replay after the correction equals eager execution bit for bit."""
    import torch

    from paper_2511_23030_b200.core import Pose
    a = _c1_engine(tmp_path / "a", budget=100_000, use_graphs=True)
    b = _c1_engine(tmp_path / "b", budget=100_000, use_graphs=False)
    for s in range(10):   # every keyframe's graph captured
        assert a.optimization_step(0, s).loss == b.optimization_step(0, s).loss
    assert getattr(a, "_graphs", {})
    for e in (a, b):
        for kid in sorted(e.store.resident_keyframe_ids()):
            kf = e.store.keyframe_get(kid)
            e.store.update_keyframe_pose(kid, Pose(rotation=kf.pose.rotation,
                                                   translation=kf.pose.translation + np.array([2e-3, -1e-3, 0.0])))
    for s in range(10, 20):
        ra, rb = a.optimization_step(0, s), b.optimization_step(0, s)
        assert ra.selected_kf == rb.selected_kf and ra.loss == rb.loss, s
    hw = a.store.slab.high_water()
    assert torch.equal(a.store.slab.params[:hw], b.store.slab.params[:hw])
    # at most one camera per keyframe among the live graphs
    cams = {}
    for k in a._graphs:
        assert cams.setdefault(k[0], k[1]) == k[1]


def _oracle_state(eng):
    """fp64 oracle TrainState holding the slab rows [0, high water) exactly."""
    from oracle import oracle as O
    s = eng.store.slab
    hw = s.high_water()
    p = s.params[:hw].cpu().numpy().astype(np.float64)
    st = O.TrainState(p[:, 0:3], p[:, 3:7], p[:, 7:10], p[:, 10], p[:, 11:14])
    st.m = s.adam_m[:hw, :14].cpu().numpy().astype(np.float64).copy()
    st.v = s.adam_v[:hw, :14].cpu().numpy().astype(np.float64).copy()
    st.steps = s.adam_m[:hw, 14].cpu().numpy().astype(np.int64).copy()
    return st, p


STEP_GROUPS = {"positions": slice(0, 3), "rotations": slice(3, 7), "scales": slice(7, 10),
               "opacities": slice(10, 11), "sh0": slice(11, 14)}


def test_optimization_step_matches_oracle(cuda, tmp_path):
    """a15: MappingEngine.optimization_step (the drop-in for sim.py:319-370:
    policy + fwd -> loss -> bwd -> Adam, graph-replayed) against the oracle's
    fused CPU step (oracle/render_oracle.c or_train_step, fp64) on the same
    keyframe and active set (sorted-chunk-id order), step by step from the
    same state.  Tolerances (written here): loss 1e-4 (the images' tolerance; the
    depth term divides by alpha in fp32); Adam moments
    per parameter group ||dm|| <= 1e-3 ||m|| (the gradient tolerance, m is a
    gradient average) and ||dv|| <= 2e-3 ||v||; the parameter update of every
    Gaussian within 1e-6 (1 + |p|) + 1e-3 |update|, except elements whose
    first moment is not resolved in fp32 (|dm| > 1e-3 |m|: a gradient at the
    noise floor of the compositing sums, which Adam's eps = 1e-15 turns into
    a full-size signed step whose sign is noise in either precision): those
    moments must be < 1e-3 of their parameter's largest, at most 2 % of the
    active set, and their steps bounded by 2 lr."""
    from paper_2511_23030_b200.mapping import AdamSettings
    eng = _c1_engine(tmp_path, budget=100_000)
    a = AdamSettings()
    lr = np.array([a.lr_position] * 3 + [a.lr_rotation] * 4 + [a.lr_scale] * 3 + [a.lr_opacity] + [a.lr_sh0] * 3)
    worst = []
    for s in range(8):
        st, before = _oracle_state(eng)
        row = eng.optimization_step(0, s)
        kf = eng.store.keyframe_get(row.selected_kf)
        ids = sorted(eng._visible_for_pose(kf.pose)[0])
        sub = np.concatenate([np.arange(o, o + c) for o, c in eng.store.segments(ids)])
        loss = st.step(kf.pose.rotation, kf.pose.translation, kf.intrinsics, kf.rgb.astype(np.float64),
                       kf.depth.astype(np.float64), eng.weights.lambda_s, eng.weights.lambda_depth, lr,
                       a.beta1, a.beta2, a.eps, a.min_scale, subset=sub)
        assert abs(row.loss - loss) <= 1e-4 * max(1.0, abs(loss)), (s, row.loss, loss)
        slab = eng.store.slab
        hw = slab.high_water()
        got = slab.params[:hw].cpu().numpy().astype(np.float64)[sub][:, :14]
        gm = slab.adam_m[:hw].cpu().numpy().astype(np.float64)[sub]
        gv = slab.adam_v[:hw].cpu().numpy().astype(np.float64)[sub]
        want = np.concatenate([st.pos, st.rot, st.scale, st.opac[:, None], st.sh0], 1)[sub]
        assert np.array_equal(gm[:, 14], st.steps[sub].astype(np.float64)), s
        for name, sl in STEP_GROUPS.items():
            dm = np.linalg.norm(gm[:, sl] - st.m[sub][:, sl])
            dv = np.linalg.norm(gv[:, sl] - st.v[sub][:, sl])
            assert dm <= 1e-3 * np.linalg.norm(st.m[sub][:, sl]) + 1e-30, (s, name, "m", dm)
            assert dv <= 2e-3 * np.linalg.norm(st.v[sub][:, sl]) + 1e-30, (s, name, "v", dv)
        upd_g = got - before[sub][:, :14]
        upd_o = want - before[sub][:, :14]
        bad = np.abs(upd_g - upd_o) > 1e-6 * (1 + np.abs(want)) + 1e-3 * np.abs(upd_o)
        # an update may differ only where its first moment is not resolved in
        # fp32 (|dm| > 1e-3 |m|: a gradient at the noise floor of the
        # compositing sums; Adam normalises it to a full signed step), and
        # those moments are tiny against their parameter's scale
        m_o, m_g = st.m[sub], gm[:, :14]
        own = np.abs(m_g - m_o) > 1e-3 * np.abs(m_o)
        # the quaternion is renormalised after the step: one unresolved
        # component moves all four
        unresolved = own.copy()
        unresolved[:, 3:7] |= own[:, 3:7].any(axis=1, keepdims=True)
        colmax = np.abs(m_o).max(axis=0)
        worst.append((int(bad.any(1).sum()), int((bad & ~unresolved).sum()),
                      float((np.abs(m_o[bad]) / colmax[np.nonzero(bad)[1]]).max(initial=0))))
        assert not np.any(bad & ~unresolved), (s, np.argwhere(bad & ~unresolved)[:5])
        assert np.all(np.abs(m_o[bad & own]) <= 1e-3 * colmax[np.nonzero(bad & own)[1]]), s
        assert bad.any(1).mean() <= 0.02, (s, int(bad.any(1).sum()), len(sub))
        assert np.all(np.abs(upd_g[bad]) <= 2.0 * np.broadcast_to(lr, bad.shape)[bad] + 1e-7), s
    print("per step: rows outside the elementwise bound, unexplained elements, max |m|/colmax:", worst)


def test_fused_adam_backward_bit_identical(cuda, tmp_path):
    """sm_render_backward_adam (Adam applied by the backward's last stage, no
    gradient buffer) = sm_render_backward + sm_adam_step, bit for bit, over
    steps that include splats the view does not reach (zero-gradient steps)."""
    import torch
    a = _c1_engine(tmp_path / "a", budget=100_000)
    b = _c1_engine(tmp_path / "b", budget=100_000)
    a.fused_adam, b.fused_adam = True, False
    for s in range(8):
        ra, rb = a.optimization_step(0, s), b.optimization_step(0, s)
        assert ra.selected_kf == rb.selected_kf and ra.loss == rb.loss, s
    sa, sb = a.store.slab, b.store.slab
    hw = sa.high_water()
    for name in ("params", "adam_m", "adam_v"):
        assert torch.equal(getattr(sa, name)[:hw], getattr(sb, name)[:hw]), name
    assert float(sb.grads[:hw].abs().max()) == 0.0
