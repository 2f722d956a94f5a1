"""Helpers to unpack the committed golden fixtures (tests/golden/*.npz)."""
import numpy as np

from paper_2511_23030_b200.core import CameraIntrinsics, Pose


def render_case(g, k):
    it = g[f"c{k}_intr"]
    intr = CameraIntrinsics(fx=float(it[0]), fy=float(it[1]), cx=float(it[2]), cy=float(it[3]),
                            near=float(it[4]), far=float(it[5]), width=int(it[6]), height=int(it[7]))
    scene = dict(positions=g[f"c{k}_positions"], rotations=g[f"c{k}_rotations"],
                 scales=g[f"c{k}_scales"], opacities=g[f"c{k}_opacities"], sh0=g[f"c{k}_sh0"])
    pose = Pose(rotation=g[f"c{k}_pose_q"], translation=g[f"c{k}_pose_t"])
    ref = (g[f"c{k}_rgb"], g[f"c{k}_depth"], g[f"c{k}_alpha"])
    return scene, pose, intr, ref


def oracle_args(scene, pose, intr):
    return (scene["positions"], scene["rotations"], scene["scales"], scene["opacities"],
            scene["sh0"], pose.rotation, pose.translation, intr.fx, intr.fy, intr.cx, intr.cy,
            intr.near, intr.width, intr.height)


def f32(scene):
    return {k: np.asarray(v, dtype=np.float32).astype(np.float64) for k, v in scene.items()}


def edge_scene():
    """The tiling / cutoff edge cases (test_edge_cases_match_oracle): a ragged
    97x61 image, splats straddling the near plane, far off-screen boxes
    reaching in, needles and near-points, an opaque stack saturating T."""
    from paper_2511_23030_b200.core import CameraIntrinsics, Pose, quat_normalize
    rng = np.random.default_rng(17)
    intr = CameraIntrinsics(fx=60.0, fy=60.0, cx=48.3, cy=30.1, width=97, height=61, near=0.2)
    pose = Pose(rotation=quat_normalize([1.0, 0.01, -0.02, 0.005]), translation=[0.0, 0.0, 0.0])
    parts = []

    def add(pos, scales, op, quats=None):
        m = len(pos)
        q = quats if quats is not None else rng.normal(size=(m, 4))
        q = q / np.linalg.norm(q, axis=1, keepdims=True)
        parts.append((np.asarray(pos, float), q, np.asarray(scales, float), np.asarray(op, float),
                      (rng.uniform(0.05, 0.95, (m, 3)) - 0.5) / 0.28209479177))

    m = 300   # background
    add(np.stack([rng.uniform(-3, 3, m), rng.uniform(-2, 2, m), rng.uniform(1, 8, m)], 1),
        rng.uniform(0.03, 0.4, (m, 3)), rng.uniform(0.2, 0.95, m))
    m = 40    # straddling / behind the near plane
    add(np.stack([rng.uniform(-0.3, 0.3, m), rng.uniform(-0.2, 0.2, m), rng.uniform(-0.1, 0.5, m)], 1),
        rng.uniform(0.02, 0.2, (m, 3)), rng.uniform(0.2, 0.9, m))
    m = 40    # far off screen, large: boxes clipped to the image
    add(np.stack([rng.choice([-1, 1], m) * rng.uniform(4, 9, m), rng.uniform(-2, 2, m), rng.uniform(2, 6, m)], 1),
        rng.uniform(0.5, 2.5, (m, 3)), rng.uniform(0.3, 0.9, m))
    m = 60    # needles and near-points
    sc = np.exp(rng.uniform(np.log(1e-4), np.log(0.5), (m, 3)))
    sc[: m // 2, 1:] = 1e-4
    add(np.stack([rng.uniform(-1.5, 1.5, m), rng.uniform(-1, 1, m), rng.uniform(1, 4, m)], 1), sc,
        rng.uniform(0.3, 0.95, m))
    m = 30    # opaque stack in front of the centre: saturates T
    add(np.stack([rng.normal(0, 0.05, m), rng.normal(0, 0.05, m), np.linspace(1.0, 1.6, m)], 1),
        np.full((m, 3), 0.25), np.full(m, 0.999), np.tile([1.0, 0, 0, 0], (m, 1)))
    pos, q, sc, op, sh0 = (np.concatenate(x) for x in zip(*parts))
    scene = f32(dict(positions=pos, rotations=q, scales=sc, opacities=op, sh0=sh0))
    return scene, pose, intr, rng
