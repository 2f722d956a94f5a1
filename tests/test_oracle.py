"""Pin the CPU oracle (oracle/render_oracle.c) against the reference's own outputs.

The golden fixtures were produced by running the reference splatmap package
(tests/golden/make_golden.py).  CPU-only; no GPU needed.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_cases import oracle_args, render_case


def test_forward_matches_reference(golden):
    g = golden("render_small.npz")
    for k in range(int(g["count"])):
        scene, pose, intr, (rgb, depth, alpha) = render_case(g, k)
        r, d, a = O.render_arrays(*oracle_args(scene, pose, intr))
        # fp64 restatement: only matmul summation order differs from NumPy/BLAS
        assert np.abs(r - rgb).max() < 1e-12, k
        assert np.abs(a - alpha).max() < 1e-12, k
        assert np.abs(d - depth).max() < 1e-11, k


def test_single_gaussian_known_answer(golden):
    g = golden("render_small.npz")
    k = int(g["count"]) - 1
    scene, pose, intr, ref = render_case(g, k)
    r, d, a = O.render_arrays(*oracle_args(scene, pose, intr))
    cy, cx = int(intr.cy), int(intr.cx)
    assert np.abs(r[cy, cx] - 0.999 * np.array([0.9, 0.3, 0.6])).max() < 1e-6
    assert abs(d[cy, cx] - 2.0) / 2.0 < 0.01
    assert a[cy, cx] > 0.99
    assert np.array_equal(r, ref[0])


def _fd_case(golden):
    f = golden("render_fd.npz")
    it = f["intr"]
    args = (f["positions"], f["rotations"], f["scales"], f["opacities"], f["sh0"], f["pose_q"],
            f["pose_t"], it[0], it[1], it[2], it[3], it[4], 32, 32)
    return f, args


FIELDS = ["positions", "rotations", "scales", "opacities", "sh0"]


def test_backward_matches_reference_finite_differences(golden):
    f, args = _fd_case(golden)
    gr = O.render_backward(*args, d_rgb=f["w_rgb"], d_depth=f["w_depth"], d_alpha=f["w_alpha"])
    for fld in FIELDS:
        an = gr[fld][f["picks"]].reshape(len(f["picks"]), -1)
        fd = f[f"lin_{fld}"]
        scale = np.abs(fd).max()
        assert np.abs(an - fd).max() <= 1e-6 * scale + 1e-6, fld


def test_loss_gradient_chain_matches_reference_fd(golden):
    f, args = _fd_case(golden)
    rgb, depth, alpha = O.render_arrays(*args)
    loss, d_rgb, d_depth = O.total_loss(rgb, depth, f["gt_rgb"], f["gt_depth"], grad=True)
    assert abs(loss - float(f["loss"])) < 1e-12
    gl = O.render_backward(*args, d_rgb=d_rgb, d_depth=d_depth)
    for fld in FIELDS:
        an = gl[fld][f["picks"]].reshape(len(f["picks"]), -1)
        fd = f[f"loss_{fld}"]
        assert np.abs(an - fd).max() <= 1e-6 * np.abs(fd).max() + 1e-9, fld


def test_total_loss_matches_reference(golden):
    g = golden("loss.npz")
    for k in range(int(g["count"])):
        for j in range(3):
            ls, ld, ref = g[f"c{k}_total_{j}"]
            v = O.total_loss(g[f"c{k}_rgb"], g[f"c{k}_depth"], g[f"c{k}_gt_rgb"],
                             g[f"c{k}_gt_depth"], ls, ld)
            assert abs(v - ref) < 1e-12, (k, j)


def test_adam_matches_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    p0 = rng.normal(size=50)
    grads = [rng.normal(size=50) for _ in range(5)]
    tp = torch.tensor(p0.copy(), requires_grad=True)
    opt = torch.optim.Adam([tp], lr=0.01, betas=(0.9, 0.999), eps=1e-8)
    p, m, v = p0.copy(), np.zeros(50), np.zeros(50)
    for step, g in enumerate(grads, start=1):
        tp.grad = torch.tensor(g)
        opt.step()
        O.adam(p, m, v, g, 0.01, 0.9, 0.999, 1e-8, step)
    assert np.abs(p - tp.detach().numpy()).max() < 1e-12
