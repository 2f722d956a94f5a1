"""Ingest path: splatmap sample.py on the device against
fixtures recorded by running the reference (tests/golden/sample.npz):
log_norm (random, blocky-edge, black, constant and rendered images; two
kernel sizes), sampling_probability, the host draw fed by the device map,
lift_to_gaussians (rotated poses, invalid depth), and two whole
_Replay.ingest_keyframe calls (sim.py:264-278) replayed through
MappingEngine.ingest_keyframe.

Tolerances: scores and probabilities are fp64 on both sides but summed in a
different order (BLAS dot / ndimage vs row-by-row taps): 1e-12 absolute on
[0, 1] maps.  Lifted records are float32-canonical (storage_canonical,
diskformat.py:69-83): equal to the reference's after the same rounding.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_log_norm_matches_reference(cuda, golden):
    from paper_2511_23030_b200 import sample as S
    g = golden("sample.npz")
    for k in range(int(g["n_img"])):
        for sig, rad in ((1.0, 2), (1.5, 3)):
            got = S.log_norm(g[f"img{k}"], sig, rad)
            want = g[f"log{k}_{sig}_{rad}"]
            assert got.shape == want.shape
            assert np.abs(got - want).max() <= 1e-12, (k, sig, rad, np.abs(got - want).max())


def test_sampling_probability_and_draw_match_reference(cuda, golden):
    from paper_2511_23030_b200 import sample as S
    g = golden("sample.npz")
    ps = S.sampling_probability(g["log0_1.0_2"], g["log4_1.0_2"])
    assert np.array_equal(ps, g["ps"])   # max(a - b, 0): one rounding, identical
    for n, seed in ((50, 3), (500, 4), (5000, 5)):
        draw = np.array(S.sample_pixels(ps, n, seed), dtype=np.int64).reshape(-1, 2)
        assert np.array_equal(draw, g[f"draw_{n}_{seed}"]), (n, seed)
    # the map computed on the device from the images draws the same pixels
    a = S.log_norm(g["img0"])
    b = S.log_norm(g["img4"])
    draw = np.array(S.sample_pixels(S.sampling_probability(a, b), 500, 4), dtype=np.int64).reshape(-1, 2)
    assert np.array_equal(draw, g["draw_500_4"])


def test_lift_matches_reference(cuda, golden):
    from paper_2511_23030_b200 import sample as S
    from paper_2511_23030_b200.core import CameraIntrinsics, Keyframe, Pose
    g = golden("sample.npz")
    intr = CameraIntrinsics(fx=50.0, fy=50.0, cx=31.5, cy=23.5, width=64, height=48, near=0.2, far=100.0)
    for k in range(3):
        kf = Keyframe(id=k, pose=Pose(rotation=g[f"lift{k}_q"], translation=g[f"lift{k}_t"]), intrinsics=intr,
                      rgb=g[f"lift{k}_rgb"], depth=g[f"lift{k}_depth"])
        pix = [tuple(p) for p in g[f"lift{k}_pix"].tolist()]
        gs = S.lift_to_gaussians(pix, kf, S.SampleConfig(init_scale_factor=1.0 + 0.5 * k))
        pos = np.array([x.position for x in gs])
        assert len(gs) == len(g[f"lift{k}_pos"])
        want = g[f"lift{k}_pos"].astype(np.float32).astype(np.float64)
        # the reference's BLAS unprojection may differ in the last fp64 bit:
        # at most a 1-ulp float32 rounding difference
        assert np.abs(pos - want).max() <= 1e-6 * (1 + np.abs(want).max())
        assert (pos == want).mean() > 0.99
        assert np.array_equal(np.array([x.scale for x in gs]), g[f"lift{k}_scale"].astype(np.float32).astype(np.float64))
        assert np.array_equal(np.array([x.sh[[0, 16, 32]] for x in gs]),
                              g[f"lift{k}_sh0"].astype(np.float32).astype(np.float64))
        assert all(x.opacity == float(np.float32(0.1)) for x in gs)
        assert all(np.array_equal(x.rotation, [1.0, 0, 0, 0]) for x in gs)


def test_ingest_keyframe_matches_reference_replay(cuda, golden, tmp_path):
    """Two ingests (empty map, then a map the first one populated and the
    second renders) through MappingEngine.ingest_keyframe insert the
    reference replay's Gaussians: same count, chunks and f32 records."""
    from paper_2511_23030_b200.core import CameraIntrinsics, Pose
    from paper_2511_23030_b200.mapping import MappingEngine
    from paper_2511_23030_b200.sample import SampleConfig
    from paper_2511_23030_b200.store import ChunkStore, StoreConfig
    g = golden("sample.npz")
    intr = CameraIntrinsics(fx=50.0, fy=50.0, cx=31.5, cy=23.5, width=64, height=48, near=0.2, far=100.0)
    store = ChunkStore(StoreConfig(disk_root=tmp_path, chunk_size_m=2.0, gaussian_budget=100_000,
                                   keyframe_budget=16, io_ns_per_byte=1.0, device="cuda"))
    eng = MappingEngine(store, intr, seed=7, sample=SampleConfig(samples_per_keyframe=800))
    for k in range(2):
        n = eng.ingest_keyframe(k, Pose(translation=g[f"ingest{k}_t"]), g[f"ingest{k}_rgb"], g[f"ingest{k}_depth"])
        assert n == int(g[f"ingest{k}_n"]), k
    rows, cids = [], []
    for cid, gs in store.iter_map():
        for x in gs:
            cids.append(cid)
            rows.append(list(x.position) + list(x.scale) + [x.opacity] + list(x.sh[[0, 16, 32]]))
    assert np.array_equal(np.array(cids, dtype=np.uint64), g["ingest_cids"])
    got, want = np.array(rows), g["ingest_map"]
    assert got.shape == want.shape
    assert np.abs(got - want).max() <= 1e-6 * (1 + np.abs(want).max())
    assert (got == want).all(axis=1).mean() > 0.99
