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


def _ref_projection(scene, pose, intr):
    """renderloss.py:170-212 in NumPy (the reference's own op sequence)."""
    r_wc = O.quat_to_matrix(pose.rotation)
    cam = (scene["positions"] - pose.translation) @ r_wc
    keep = cam[:, 2] >= intr.near
    idx = np.flatnonzero(keep)
    cam = cam[keep]
    x, y, z = cam[:, 0], cam[:, 1], cam[:, 2]
    means = np.stack([intr.fx * x / z + intr.cx, intr.fy * y / z + intr.cy], axis=1)
    q = scene["rotations"][keep]
    w_, x_, y_, z_ = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    rot = np.empty((len(q), 3, 3))
    rot[:, 0, 0] = 1 - 2 * (y_ * y_ + z_ * z_)
    rot[:, 0, 1] = 2 * (x_ * y_ - w_ * z_)
    rot[:, 0, 2] = 2 * (x_ * z_ + w_ * y_)
    rot[:, 1, 0] = 2 * (x_ * y_ + w_ * z_)
    rot[:, 1, 1] = 1 - 2 * (x_ * x_ + z_ * z_)
    rot[:, 1, 2] = 2 * (y_ * z_ - w_ * x_)
    rot[:, 2, 0] = 2 * (x_ * z_ - w_ * y_)
    rot[:, 2, 1] = 2 * (y_ * z_ + w_ * x_)
    rot[:, 2, 2] = 1 - 2 * (x_ * x_ + y_ * y_)
    s2 = scene["scales"][keep] ** 2
    sw = (rot * s2[:, None, :]) @ rot.transpose(0, 2, 1)
    wm = r_wc.T
    sc = (wm @ sw) @ wm.T
    jac = np.zeros((len(z), 2, 3))
    jac[:, 0, 0] = intr.fx / z
    jac[:, 0, 2] = -intr.fx * x / z ** 2
    jac[:, 1, 1] = intr.fy / z
    jac[:, 1, 2] = -intr.fy * y / z ** 2
    cov2 = (jac @ sc) @ jac.transpose(0, 2, 1)
    abc = np.stack([cov2[:, 0, 0] + 0.3, cov2[:, 0, 1], cov2[:, 1, 1] + 0.3], axis=1)
    colors = np.clip(0.28209479177 * scene["sh0"][keep] + 0.5, 0.0, 1.0)
    full = lambda a: np.zeros((len(scene["positions"]),) + a.shape[1:])  # noqa: E731
    out = {k: full(v) for k, v in (("means", means), ("abc", abc), ("z", z), ("colors", colors))}
    out["means"][idx], out["abc"][idx], out["z"][idx], out["colors"][idx] = means, abc, z, colors
    return out


def test_bin_oracle_tile_lists_reproduce_reference_images(golden):
    """The binning restatement (oracle/bin_oracle.c, the device's K2/K3
    arithmetic) loses no (pixel, Gaussian) pair and keeps the reference
    order: compositing each 16x16 tile over its key list -- depth ranks in
    key order, the reference's per-pair math (renderloss.py:106-152) -- gives
    the reference's own images (tests/golden/render_small.npz) to 1e-12."""
    g = golden("render_small.npz")
    for k in range(int(g["count"])):
        scene, pose, intr, (rgb_ref, depth_ref, alpha_ref) = render_case(g, k)
        n = len(scene["positions"])
        rec = np.zeros((n, 16), np.float32)
        rec[:, 0:3], rec[:, 3:7], rec[:, 7:10] = scene["positions"], scene["rotations"], scene["scales"]
        rec[:, 10], rec[:, 11:14] = scene["opacities"], scene["sh0"]
        order, keys, ranges = O.bin_tiles(rec, pose.rotation, pose.translation, intr.fx, intr.fy, intr.cx,
                                          intr.cy, intr.near, intr.width, intr.height)
        rb = max(1, int(np.ceil(np.log2(max(n, 2)))))
        pr = _ref_projection(scene, pose, intr)
        h, w = intr.height, intr.width
        rgb, dacc, trans = np.zeros((h, w, 3)), np.zeros((h, w)), np.ones((h, w))
        tx = (w + 15) // 16
        for t in range(len(ranges)):
            ys, xs = np.mgrid[(t // tx) * 16:(t // tx) * 16 + 16, (t % tx) * 16:(t % tx) * 16 + 16]
            inside = (ys < h) & (xs < w)
            ys, xs = ys[inside], xs[inside]
            for key in keys[ranges[t, 0]:ranges[t, 1]]:
                i = int(order[int(key) & ((1 << rb) - 1)])
                a, b, c = pr["abc"][i]
                det = a * c - b * b
                u, v = pr["means"][i]
                rx, ry = 3.0 * np.sqrt(a), 3.0 * np.sqrt(c)
                x0, x1 = max(int(np.ceil(u - rx)), 0), min(int(np.floor(u + rx)), w - 1)
                y0, y1 = max(int(np.ceil(v - ry)), 0), min(int(np.floor(v + ry)), h - 1)
                m = (xs >= x0) & (xs <= x1) & (ys >= y0) & (ys <= y1)
                dx, dy = xs - u, ys - v
                qq = (c / det) * dx * dx + 2.0 * (-b / det) * dx * dy + (a / det) * dy * dy
                tt = trans[ys, xs]
                m &= (qq <= 9.0) & (tt >= 1e-10)
                al = scene["opacities"][i] * np.exp(-0.5 * qq)
                con = np.where(m, tt * al, 0.0)
                rgb[ys, xs] += con[:, None] * pr["colors"][i]
                dacc[ys, xs] += con * pr["z"][i]
                trans[ys, xs] = np.where(m, tt * (1.0 - al), tt)
        alpha = 1.0 - trans
        assert np.abs(np.clip(rgb, 0, 1) - rgb_ref).max() <= 1e-12, k
        assert np.abs(np.clip(alpha, 0, 1) - alpha_ref).max() <= 1e-12, k
