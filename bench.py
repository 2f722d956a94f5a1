#!/usr/bin/env python
"""Mapping-step benchmark (BASELINE.json metric: mapping iters/s, Gaussians/s).

Workload = BASELINE.json configs[1] ("C2"): 1M-Gaussian Replica-shaped room,
640x480, 8x8x2 chunks (s = 1 m), single-GPU mapping loop; synthetic data
(paper_2511_23030_b200.synthetic), random-init-free: the map is the scene and
the keyframes' ground truth renders a perturbed copy of it.

One step = paper_2511_23030_b200.mapping.MappingEngine.optimization_step:
the reference's host policy (keyframe draw, visibility, residency, metrics)
+ device render fwd, fused loss fwd/bwd, render bwd, fused Adam, one loss
readback.  N > 1 (torchrun): data-parallel over keyframes, one keyframe per
rank per step, NCCL all-reduce of the gradient slab, replicated Adam
(weak scaling: value = keyframe-iterations/s over all ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "mapping iters/sec (render fwd+bwd+Adam)"
UNIT = "it/s"
WORKLOAD = "C2: 1M-Gaussian Replica-shaped room, 640x480, 8x8x2 chunks (s=1 m), 16 keyframes"
WORKLOAD_C3 = ("C3: C2's 1M room at 640x480, K keyframes per mapping step (default 8), data-parallel over the "
               "GPUs (keyframe j on rank j mod G), packed union gradients summed with one NCCL all-reduce, "
               "replicated Adam; value = keyframe iterations/s over all ranks")


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.lines: list[str] = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.start_count = len(self.lines)
        except Exception:
            self.proc = None
            self.start_count = 0

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        rows = [l.split(", ") for l in self.lines[max(0, self.start_count - 1):] if l]
        sm = [float(r[0]) for r in rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 7 for i in range(4)
                          if r[3 + i].strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


# Algorithmic bytes per unit of each stage.
#   n = visible Gaussians, i = tile instances, p = pixels
# Algorithmic bytes per step and stage (n visible Gaussians, i tile instances,
# p pixels, v instances the compositing revisits = the backward's horizon sum):
STAGE_BYTES = {
    "project_fwd": lambda n, i, p, v: n * (4 + 64 + 64 + 40 + 8 + 4 + 4),
    "depth_sort": lambda n, i, p, v: n * 8 * 4 * 2 + n * 8,
    "bin_emit": lambda n, i, p, v: n * (4 + 4 + 64 + 64 + 4 * 4) + i * 4,
    "tile_sort": lambda n, i, p, v: i * 2 * 12 + i * 8,
    "composite_fwd": lambda n, i, p, v: v * (4 + 64) + p * (20 + 28),
    "loss": lambda n, i, p, v: p * (16 + 7 + 36 * 2 + 16),
    "composite_bwd": lambda n, i, p, v: v * (4 + 64 + 48) + p * (28 + 16),
    "project_bwd": lambda n, i, p, v: n * (4 + 4 + 4 + 64 + 40 + 2 * 64),
    "adam": lambda n, i, p, v: n * (4 + 7 * 64),
    "grad_gather": lambda n, i, p, v: n * (4 + 4 + 64 + 48) + v * (48 + 4),
}
NCU_SUMMARY = Path(__file__).resolve().parent / "profiles" / "r02_ncu_full.json"


def _ncu_kernel(name: str):
    """Counters of `name` from the committed `ncu --set full` summary (same build)."""
    try:
        return json.loads(NCU_SUMMARY.read_text())["kernels"].get(name)
    except (OSError, ValueError, KeyError):
        return None


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _ensure_ranks(args) -> None:
    """`bench.py --gpus N` outside torchrun re-executes itself under
    torch.distributed.run with N ranks (one per GPU, 127.0.0.1); under a
    launcher whose world size is not N it refuses to run."""
    env = os.environ.get("WORLD_SIZE")
    if env is None:
        if args.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                   f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
            sys.exit(subprocess.call(cmd))
        return
    if int(env) != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env}; refusing to report\n")
        sys.exit(2)


def _dist():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("SM_BENCH_ONE_GPU"):
        # plumbing check of the N-rank path on a one-GPU box: every rank on
        # cuda:0, exchanging through gloo (host copies), so no rank's kernels
        # wait on another's; never a measurement (the line says so)
        local = 0
        if world > 1 and not dist.is_initialized():
            dist.init_process_group("gloo")
        return world, rank, local
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def cpu_baseline_step(eng, kf_id: int, seconds: float = 20.0, threads: int | None = None):
    """Oracle (CPU, fp64) mapping iteration on the same active set; bounded sample."""
    from oracle import oracle as O
    store = eng.store
    kf = store.keyframe_get(kf_id)
    visible, _ = eng._visible_for_pose(kf.pose)
    ids = sorted(visible)
    rows = np.concatenate([np.arange(o, o + c) for o, c in store.segments(ids)]) if ids else np.zeros(0, int)
    p = store.slab.params[rows].cpu().numpy().astype(np.float64)
    st = O.TrainState(p[:, 0:3], p[:, 3:7], p[:, 7:10], p[:, 10], p[:, 11:14])
    a = eng.adam
    lr = [a.lr_position] * 3 + [a.lr_rotation] * 4 + [a.lr_scale] * 3 + [a.lr_opacity] + [a.lr_sh0] * 3
    gt = kf.rgb.astype(np.float64)
    threads = threads or os.cpu_count() or 1
    times = []
    t_end = time.perf_counter() + seconds
    while True:
        t0 = time.perf_counter()
        st.step(kf.pose.rotation, kf.pose.translation, kf.intrinsics, gt, kf.depth, eng.weights.lambda_s,
                eng.weights.lambda_depth, lr, a.beta1, a.beta2, a.eps, a.min_scale, threads=threads)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end or len(times) >= 5:
            break
    per = sum(times) / len(times)
    return {"value": 1.0 / per, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{len(times)} full oracle mapping iteration(s) (fp64 fwd+loss+bwd+Adam, "
                      f"oracle/render_oracle.c) on keyframe {kf_id}'s active set of {len(rows)} "
                      f"Gaussians at 640x480, {per:.2f} s each, {threads} threads"}


def workload_config(args) -> dict:
    """The benchmarked configuration -- identical in both arms' lines."""
    c3 = args.gpus > 1 or args.keyframes_per_step > 1
    return {"workload": WORKLOAD_C3 if c3 else WORKLOAD, "keyframes_per_step": args.keyframes_per_step,
            "gaussians_total": args.n, "keyframes": args.keyframes, "resolution": [640, 480],
            "parallelism": f"dp{args.gpus}",
            "l2": "inputs larger than L2 (slab params+Adam+grads 256 MB/1M Gaussians)"}


def run_reference(args, world, rank):
    """--impl reference: the reference algorithm's CPU path on this host.

    The like-for-like arm (oracle/ref_arm.py OracleMappingLoop): the
    reference's own policy code (baseline/_ref/splatmap select / culling,
    unmodified) draws the same keyframe sequence as the GPU arm -- one
    iteration per keyframe (the GPU arm's graph warm-up), W warm-up steps,
    then exactly K timed steps of K keyframes each -- and each keyframe
    iteration (render, loss + gradient, backward, Adam on the active set)
    runs in the fp64 oracle on all host threads.  Two more measurements
    travel in the line: the same iteration on 1 thread (BASELINE.md 3's
    primary denominator) and, for context, the unmodified reference
    sim._Replay.optimization_step (forward + nudge only) on the same scene.
    """
    if rank != 0:
        return
    from oracle.ref_arm import OracleMappingLoop, reference_replay_leg
    from paper_2511_23030_b200.synthetic import C2_INTR, perturbed, room_poses, room_scene
    threads = os.cpu_count() or 1
    kps = args.keyframes_per_step
    scene = room_scene(args.n, seed=42)
    poses = room_poses(args.keyframes, seed=42)
    target = perturbed(scene, 49)
    loop = OracleMappingLoop(scene, target, poses, C2_INTR, threads=threads)
    loop.warm()
    for _ in range(args.warmup * kps):
        loop.step()
    n0 = len(loop.n_active)
    t0 = time.perf_counter()
    for _ in range(args.steps * kps):   # C3: K keyframe iterations per step, in sequence
        loop.step()
    dt = time.perf_counter() - t0
    seq = loop.selected[-args.steps * kps:]
    n_act = float(np.mean(loop.n_active[n0:]))
    value = args.steps * kps / dt
    t1 = time.perf_counter()
    loop.train(seq[-1], threads=1)
    one = 1.0 / (time.perf_counter() - t1)
    ctx = None
    if not args.no_context:
        try:
            ctx = reference_replay_leg(scene, target, poses, C2_INTR, steps=2, warmup=1, gts=loop.gt)
        except Exception as exc:   # report, never fake
            ctx = {"value": None, "sample": f"failed: {type(exc).__name__}: {exc}"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args),
        "kf_sequence": seq,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} steps x {kps} keyframe iteration(s) after {len(poses)} "
                                   f"warm-up iterations + {args.warmup} warm-up steps: reference policy "
                                   f"(baseline/_ref/splatmap select/culling) + fp64 oracle fwd+loss+bwd+Adam "
                                   f"(oracle/render_oracle.c) on ~{int(n_act)} active of {args.n} Gaussians, "
                                   f"640x480, {threads} threads",
                         "single_thread": {"value": one, "unit": UNIT, "cores": 1,
                                           "sample": "1 keyframe iteration of the same loop, 1 thread"}},
        "reference_replay": ctx,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--keyframes", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-context", action="store_true", help="reference arm: skip the _Replay context leg")
    ap.add_argument("--fused-adam", action="store_true", help="A/B: Adam fused into the backward")
    ap.add_argument("--keyframes-per-step", type=int, default=None,
                    help="K keyframes per mapping step (default 1 on one GPU = C2, 8 on N > 1 = C3)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = (1, 0, 0)
    if args.impl != "reference":
        _ensure_ranks(args)
    if args.keyframes_per_step is None:
        args.keyframes_per_step = 1 if args.gpus == 1 else 8
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, world, rank)
        return
    import torch
    world, rank, local = _dist()
    torch.cuda.set_device(local)
    from paper_2511_23030_b200 import _lib
    from paper_2511_23030_b200.workloads import build_c2
    lib = _lib.load()
    eng = build_c2(args.n, args.keyframes, store_dir=tempfile.mkdtemp(prefix=f"bench_r{rank}_"),
                   device=f"cuda:{local}")
    eng.fused_adam = args.fused_adam
    dist = None
    if world > 1:
        import torch.distributed as dist
    kps = args.keyframes_per_step
    c3 = world > 1 or kps > 1
    step_fn = (lambda f, s: eng.optimization_step(f, s)) if not c3 else \
        (lambda f, s: eng.optimization_step_dp(f, s, world, rank, keyframes=kps))
    def timed(frame: int, clocks_gpu=None, fn=None):
        """barrier + sync, CUDA events around exactly args.steps steps, max over ranks."""
        fn = fn or step_fn
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        sampler = ClockSampler(clocks_gpu) if clocks_gpu is not None else None
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for s in range(args.steps):
            fn(frame, s)
        b.record()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        clk = sampler.stop() if sampler else None
        t_ms = a.elapsed_time(b)
        if dist is not None:
            t = torch.tensor([t_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_ms = float(t.item())
        return t_ms, clk

    eng.warm_graphs()
    for s in range(args.warmup):
        step_fn(0, s)
    torch.cuda.synchronize()
    # ------------------------------------------------------------ timed (device-resident)
    eng.reset_counters()
    launches0 = lib.sm_launch_count()
    te0 = eng.counter_eager
    ms, clk = timed(1, clocks_gpu=local)
    timed_eager = eng.counter_eager - te0
    launches = lib.sm_launch_count() - launches0
    kf_seq = [r.selected_kf for r in eng.rows[-args.steps * (kps if c3 else 1):]]
    ms_step = ms / args.steps
    units = args.steps * (kps if c3 else 1)   # keyframe iterations, all ranks
    value = units / (ms / 1e3)
    n_vis = eng.counter_gaussians / max(eng.counter_steps, 1)
    n_inst = eng.counter_instances / max(eng.counter_steps, 1)
    n_visit = eng.counter_visited / max(eng.counter_steps, 1)
    gauss_s = eng.counter_gaussians * world / (ms / 1e3)
    c3_g1 = None
    if rank == 0 and world == 1 and not c3:
        # C3 at G = 1 (K = 8 keyframes per step on this GPU): the T_1(K) of the
        # scaling runs, where N > 1 lines report the same K split over N ranks
        dp = lambda f, s: eng.optimization_step_dp(f, s, 1, 0, keyframes=8)  # noqa: E731
        for s in range(3):
            dp(5, s)
        n3 = max(args.steps // 8, 20)
        torch.cuda.synchronize()
        a3, b3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a3.record()
        for s in range(n3):
            dp(6, s)
        b3.record()
        torch.cuda.synchronize()
        t3 = a3.elapsed_time(b3)
        c3_g1 = {"workload": WORKLOAD_C3, "keyframes_per_step": 8, "n_gpus": 1, "steps": n3,
                 "ms_per_step": t3 / n3, "value": 8 * n3 / (t3 / 1e3), "unit": UNIT}
    # ------------------------------------------------------------ e2e through the public API
    eng.upload_keyframes_each_step = True
    eng.warm_graphs()
    eng.reset_counters()
    h2d0, d2h0 = eng.h2d_bytes, eng.d2h_bytes
    e0, r0 = eng.counter_eager, eng.counter_replays
    ems, _ = timed(3)
    e2e = {"value": units / (ems / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int((eng.h2d_bytes - h2d0) / args.steps),
           "d2h_bytes_per_step": int((eng.d2h_bytes - d2h0) / args.steps),
           # the pass's own work (it trains later steps of the same run)
           "visible_gaussians_per_step": eng.counter_gaussians / max(eng.counter_steps, 1),
           "revisited_instances_per_step": eng.counter_visited / max(eng.counter_steps, 1),
           "eager_steps": eng.counter_eager - e0, "graph_replays": eng.counter_replays - r0,
           "kf_sequence_distinct": len(set(r.selected_kf for r in eng.rows[-units:]))}
    eng.upload_keyframes_each_step = False
    # ------------------------------------------------------------ per-kernel timing pass
    # Same steps again with CUDA-event pairs around every stage (external event
    # nodes inside the step graphs); kept out of the headline region because
    # the extra nodes cost ~5%.
    lib.sm_profile_enable(1)
    eng.drop_graphs()
    eng.warm_graphs()
    _lib.profile_collect()
    # (C3: single-keyframe steps -- the same per-keyframe kernels; the K-keyframe
    # step's per-stage events are not all recorded inside its graphs)
    if c3:
        eng.reset_counters()
    pms, _ = timed(4, fn=(lambda f, s: eng.optimization_step(f, s)) if c3 else None)
    prof = _lib.profile_collect()
    lib.sm_profile_enable(0)
    if c3:   # the per-keyframe work of the profiled (single-keyframe) steps
        n_vis = eng.counter_gaussians / max(eng.counter_steps, 1)
        n_inst = eng.counter_instances / max(eng.counter_steps, 1)
        n_visit = eng.counter_visited / max(eng.counter_steps, 1)
    # ------------------------------------------------------------ roofline of the dominant kernel
    peaks = _peaks()
    px = eng.intr.width * eng.intr.height
    stages = {k: {"ms_per_step": v[0] / args.steps, "calls": v[1]} for k, v in prof.items() if v[1]}
    dom = max(stages, key=lambda k: stages[k]["ms_per_step"]) if stages else None
    roof = None
    if dom:
        per_launch_ms = prof[dom][0] / prof[dom][1]
        launches_per_step = prof[dom][1] / args.steps
        byt = STAGE_BYTES.get(dom, lambda *a: 0)(n_vis, n_inst, px, n_visit) / max(launches_per_step, 1)
        achieved = byt / (per_launch_ms / 1e3) / 1e9
        nk = _ncu_kernel(dom)
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                "traffic": nk.get("traffic_bytes") if nk else None,
                "traffic_source": f"profiles/{NCU_SUMMARY.name} (ncu --set full, dram read+write per launch)",
                "algorithmic_bytes_per_launch": byt, "ms_per_launch": per_launch_ms,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if "_fallback" not in peaks
                else "fallback 6.65 TB/s",
                # the compositing kernels are issue / FP32-pipe bound, not HBM bound
                "issue_active_pct": nk.get("issue_pct") if nk else None,
                "fma_pipe_active_pct": nk.get("fma_pipe_pct") if nk else None,
                "sm_throughput_pct": nk.get("sm_pct") if nk else None}
        for k, v in stages.items():
            f = STAGE_BYTES.get(k)
            if f and v["calls"]:
                b = f(n_vis, n_inst, px, n_visit) / (v["calls"] / args.steps)
                v["gbs"] = b / (v["ms_per_step"] / (v["calls"] / args.steps) / 1e3) / 1e9
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_step(eng, eng.latest_kf, seconds=args.cpu_seconds)
        except Exception as exc:  # report, never fake
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "port", "sample": f"failed: {exc}"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args),
        "measured": {"visible_gaussians_per_step": n_vis, "tile_instances_per_step": n_inst,
                     "revisited_instances_per_step": n_visit, "eager_steps": timed_eager},
        "kf_sequence": kf_seq,
        "gaussians_per_s": gauss_s,
        "e2e": e2e, "gpu_launches": int(launches), "clocks": clk, "roofline": roof,
        "stages": stages, "stages_pass_ms_per_step": pms / args.steps, "cpu_baseline": cpu,
        "stages_mode": "single-keyframe steps" if c3 else "the timed steps",
        "c3_g1": c3_g1,
    }
    if os.environ.get("SM_BENCH_ONE_GPU"):
        line["plumbing_check"] = "all ranks on one GPU over gloo: not a measurement"
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
