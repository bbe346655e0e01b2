#!/usr/bin/env python
"""Benchmark of the MGPBD hot path (BASELINE.json metric: ms/frame @20 AMG-PCG iterations on the
1.67M-tet block, plus the HBM GB/s of the level-0 matrix pass).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]
                  [--precision fp32|fp64] [--level0-operator 0|1] [--partitioned]

One step = one frame of Algorithm 1 (20 outer iterations x 10 MGPCG iterations; the lazy setup runs
every 20 frames and after an indefinite PCG step, reading c13, and its cost is inside the timed
frames).  Rank 0 prints one JSON line.  `--gpus N` (N > 1) without torchrun re-launches itself under
`torch.distributed.run` with N ranks; under torchrun WORLD_SIZE must equal N.
--impl reference times the CPU oracle (the tier's reference arm) on the same workload: each step is
one outer Algorithm-1 iteration of the full configuration after the frame-0 setup (timed on its own),
and the value is setup/setup_interval + n_iters x the mean iteration time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms/frame @20 AMG-PCG iters (1.7M-tet block) at 1/2/4/8 B200; SpMV HBM GB/s"
UNIT = "ms/frame"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def traffic_per_launch(op=1):
    """dram__bytes_read.sum + dram__bytes_write.sum per level-0 pass (both kernels of the matrix-free
    pass, or the CSR k_rows pass for op=0), from the committed ncu --set full capture summary
    (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return d.get("bytes_per_launch") if op == 1 else d.get("previous_csr_k_rows_bytes_per_launch")
        except Exception:
            return None
    return None


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def oracle_at_config(sc, iters):
    """The oracle (1 core, fp64) on the configured workload itself: frame 0 with `iters` outer
    iterations (setup at ite 0, timed inside the oracle).  Returns (ms/frame = setup/setup_interval +
    n_iters x mean iteration, mean iteration ms, setup ms, the Sim for the parity comparison)."""
    import oracle as O
    sim = O.Sim(sc)                      # pattern of A (creation, not part of a frame)
    t0 = time.perf_counter()
    sim.step(sc.dt, iters)
    total = (time.perf_counter() - t0) * 1e3
    setup = sim.setup_ms()
    per_iter = (total - setup) / iters
    return setup / sim.cfg.setup_interval + sc.n_iters * per_iter, per_iter, setup, sim


def frame_errors(ctx, sim, sc):
    """GPU-vs-oracle error of the same frame: relative 2-norm and max-abs/max of lambda and of the
    displacement x - x_start."""
    import numpy as np
    xo, _, lo = sim.state()
    x, lam = ctx.positions(), ctx.lambdas()
    dx, dxo = x - sc.pos, xo - sc.pos
    return {"lambda_rel2": float(np.linalg.norm(lam - lo) / np.linalg.norm(lo)),
            "lambda_maxabs_over_max": float(np.abs(lam - lo).max() / np.abs(lo).max()),
            "dx_rel2": float(np.linalg.norm(dx - dxo) / np.linalg.norm(dxo)),
            "dx_maxabs_over_max": float(np.abs(dx - dxo).max() / np.abs(dxo).max())}


def config_dict(sc, args, world, extra=None):
    d = {"workload": sc.name, "n_cons": sc.n_cons, "n_verts": sc.n_verts, "n_iters": sc.n_iters,
         "k_nullspace": args.k_nullspace,
         "pcg_iters": sc.pcg_iters, "setup_interval": 20, "precision": args.precision,
         "accumulation": "fp64", "l2": "inputs larger than L2 (level-0 matrix streamed from HBM every pass)",
         "parallelism": (f"level-0 rows partitioned over {world} GPUs (NCCL halos + allreduce), coarse "
                         f"levels replicated") if world > 1 else "single GPU"}
    if extra:
        d.update(extra)
    return d


def run_reference(args):
    """The tier's reference arm: the CPU oracle, as it stands, on the configured workload.  Each step is
    one outer Algorithm-1 iteration (constraint evaluation, assembly, Galerkin refresh, 10 MGPCG
    iterations, update) of the full configuration; frame 0's setup runs once before the warm-up steps
    and is timed on its own."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2505_13390_b200 import scenes
    import oracle as O
    sc = scenes.make(args.config)
    t0 = time.perf_counter()
    sim = O.Sim(sc)
    t_create = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    sim.step(sc.dt, 1)                   # frame 0: predict, setup (timed inside), first outer iteration
    first = (time.perf_counter() - t0) * 1e3
    setup = sim.setup_ms()
    times = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        sim.step(sc.dt, 1)               # one outer iteration (setup_interval 20: no setup in frames 1..19)
        dt_ms = (time.perf_counter() - t0) * 1e3
        if sim.setup_ms() > 0:           # an off-schedule setup (indefinite event / frame % 20): count apart
            dt_ms -= sim.setup_ms()
        if k >= args.warmup:
            times.append(dt_ms)
    per_iter = statistics.mean(times)
    ms = setup / sim.cfg.setup_interval + sc.n_iters * per_iter
    sample = (f"oracle (fp64, 1 core) on the full {sc.name} ({sc.n_cons} constraints): each step = one outer "
              f"Alg.-1 iteration ({args.steps} timed after {args.warmup} warm-up, mean {per_iter:.0f} ms); frame-0 "
              f"setup {setup:.0f} ms timed once and amortised /{sim.cfg.setup_interval}; value = setup/20 + "
              f"{sc.n_iters} x iteration (pattern creation {t_create:.0f} ms excluded)")
    cores = 1
    out = {"impl": "reference", "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": sc.name, "n_cons": sc.n_cons, "n_verts": sc.n_verts, "n_iters": sc.n_iters,
                      "pcg_iters": sc.pcg_iters, "setup_interval": 20, "precision": "fp64 (oracle)",
                      "same_config": True},
           "cpu_baseline": {"value": ms, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                            "measured_at_config": True, "iteration_ms": per_iter, "setup_ms": setup,
                            "first_frame_ms": first},
           "e2e": {"value": ms, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def run_ours(args):
    # NCCL's banner / debug lines go to stderr: stdout carries exactly one JSON line
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    import numpy as np
    import torch
    from paper_2505_13390_b200 import mgpbd, scenes

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sc = scenes.make(args.config)
    prec = 1 if args.precision == "fp32" else 0
    stream = torch.cuda.Stream()
    part = {}
    if world > 1:
        # one process per GPU; level-0 rows partitioned over NCCL (rank 0 creates the unique id)
        obj = [mgpbd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        part = dict(rank=rank, world=world, nccl_id=obj[0])
    elif args.partitioned:
        part = dict(rank=0, world=1, nccl_id=mgpbd.nccl_unique_id())   # partitioned path, 1-rank NCCL
    # k > 1: coarse DOFs shrink by ~k/aggregate size per level, the stall rule (c7) leaves a larger coarsest level
    kx = dict(max_dense_coarse=8192) if args.k_nullspace > 1 else {}
    ctx = mgpbd.Context.from_scene(sc, precision=prec, device=local, stream=stream.cuda_stream, profile=0,
                                   level0_operator=args.level0_operator, k_nullspace=args.k_nullspace, **part, **kx)
    for _ in range(args.warmup):
        ctx.step(sc.dt, sc.n_iters)
    st0 = ctx.stats()
    levels = [(int(st0.n[l]), int(st0.nnz[l])) for l in range(st0.n_levels)]

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    launches = 0
    indef = 0
    frames_ms, setup_ms, steady_ms = [], [], []
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            ctx.step(sc.dt, sc.n_iters)
            s = ctx.stats()
            launches += s.kernel_launches
            indef += s.indefinite_events
            frames_ms.append(s.ms_frame)
            if s.setup_ran:
                setup_ms.append(s.ms_setup)
            else:
                steady_ms.append(s.ms_frame)
        e1.record(stream)
        barrier()
    t_ms = e0.elapsed_time(e1)
    st1 = ctx.stats()   # the hierarchy the window ended on (re-setups inside the window change it)
    levels_end = [(int(st1.n[l]), int(st1.nnz[l])) for l in range(st1.n_levels)]
    # phase breakdown + eager pass timing: the same frames again with CUDA events around every level-0 pass
    # and phase (the per-iteration graphs are bypassed; kernels are identical)
    ctx.set_profiling(True)
    l0_ms = l0_bytes = 0.0
    prof_frames_ms = 0.0
    phases = {"assemble": 0.0, "galerkin_refresh": 0.0, "vcycle": 0.0, "pcg_other": 0.0, "update": 0.0}
    for _ in range(args.profile_frames):
        ctx.step(sc.dt, sc.n_iters)
        s = ctx.stats()
        l0_ms += s.l0_pass_ms
        l0_bytes += s.l0_pass_bytes
        prof_frames_ms += s.ms_frame - s.ms_setup
        for k, v in zip(phases, (s.ms_assemble, s.ms_galerkin, s.ms_vcycle, s.ms_pcg_other, s.ms_update)):
            phases[k] += v / max(args.profile_frames, 1)
    # the same passes timed INSIDE the replayed per-iteration graphs (the launch configuration of the timed
    # frames): event-record nodes around every level-0 pass, the last replay standing for all iterations
    ctx.set_profiling(2)
    g_ms = g_bytes = g_frames_ms = 0.0
    for _ in range(args.profile_frames):
        ctx.step(sc.dt, sc.n_iters)
        s = ctx.stats()
        g_ms += s.l0_pass_ms
        g_bytes += s.l0_pass_bytes
        g_frames_ms += s.ms_frame - s.ms_setup
    ctx.set_profiling(False)
    burst = None
    if world == 1 and not args.partitioned:  # the same pass replayed as one CUDA graph: no launch gaps
        b_ms, b_bytes = ctx.pass_burst(50)
        burst = (b_bytes / 1e9) / (b_ms / 1e3)
    if dist:
        tt = torch.tensor([t_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
        ll = torch.tensor([launches], device="cuda", dtype=torch.int64)
        dist.all_reduce(ll)
        launches = int(ll.item())
    ms_per_step = t_ms / args.steps
    value = ms_per_step              # one block, all ranks together: time per frame (max over ranks)

    # e2e: through the public API with host buffers (pinned), H2D of the state + D2H of the result
    n, m = sc.n_verts, sc.n_cons
    pos_h = torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy()
    vel_h = torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy()
    lam_h = torch.empty((m,), dtype=torch.float64, pin_memory=True).numpy()
    ctx.positions(pos_h)
    vel_h[:] = ctx.velocities()
    barrier()
    e2e_setups = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ctx.set_state(pos_h, vel_h)
        ctx.step(sc.dt, sc.n_iters)
        e2e_setups += int(ctx.stats().setup_ran)   # the device-timed loop reads stats every frame too
        ctx.positions(pos_h)
        ctx.velocities(vel_h)
        ctx.lambdas(lam_h)
    barrier()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    if dist:
        tt = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())

    peak, peak_kind = measured_peaks()
    achieved = (g_bytes / 1e9) / (g_ms / 1e3) if g_ms > 0 else None
    achieved_eager = (l0_bytes / 1e9) / (l0_ms / 1e3) if l0_ms > 0 else None
    clocks = clk.summary()
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if prec else "f64", "data": "synthetic",
        "config": config_dict(sc, args, world, {
            "nnz_A0": levels[0][1] if levels else None, "levels": levels_end, "levels_at_window_start": levels,
            "op_complexity": st1.op_complexity,
            "ms_setup_frame_extra": (statistics.mean(setup_ms) if setup_ms else None),
            "setups_in_window": len(setup_ms),
            "indefinite_events_in_window": indef,
            "ms_frame_median": statistics.median(frames_ms),
            "ms_frame_steady_median": statistics.median(steady_ms) if steady_ms else None,
            "sweep_criterion": "ms_frame_steady_median (frames without a setup) and ms_setup_frame_extra"}),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic_per_launch(args.level0_operator),
                     "kernel": ("level-0 matrix-free passes (k_mf_vgather + k_mf_rows: omega-Jacobi / residual*P / "
                                "SpMV+dot / Jacobi+r.z)") if args.level0_operator == 1 else
                               "level-0 CSR passes (k_rows: omega-Jacobi / residual*P / SpMV+dot / Jacobi+r.z)",
                     "peak_kind": peak_kind, "profiled_frames": args.profile_frames,
                     "method": "CUDA events captured around every level-0 pass inside the replayed per-iteration "
                               "graphs (mgpbd_set_profiling(2)), frames after the timed window",
                     "l0_pass_share_of_frame": (g_ms / g_frames_ms) if g_frames_ms else None},
        "roofline_eager": {"achieved": achieved_eager, "frac": (achieved_eager / peak) if achieved_eager else None,
                           "l0_pass_share_of_frame": (l0_ms / prof_frames_ms) if prof_frames_ms else None,
                           "method": "the same passes launched eagerly between event records (launch gaps included)"},
        "roofline_graph_burst": None if burst is None else {
            "achieved": burst, "peak": peak, "unit": "GB/s", "frac": burst / peak, "passes": 50,
            "method": "50 level-0 SpMV+dot passes on the frame's state captured as one CUDA graph, CUDA "
                      "events around its replay (the kernel timed alone: no launch gaps)"},
        "e2e": {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": 2 * 3 * n * 8,
                "d2h_bytes_per_step": (2 * 3 * n + m) * 8, "setups_in_window": e2e_setups,
                "note": "frames after the device-timed window; the lazy / indefinite-step re-setups "
                        "(45 ms each) fall differently across the two windows"},
        "phase_ms_per_frame": {**{k: round(v, 3) for k, v in phases.items()},
                               "note": "profiled (eager) frames; graphs are faster"},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    ctx.close()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the oracle on the configured workload itself (frame 0, setup + cpu_iters outer iterations),
        # and the GPU's error on that same frame (a fresh context in the bench configuration)
        ms_o, per_iter, setup, sim = oracle_at_config(sc, args.cpu_iters)
        ctx0 = mgpbd.Context.from_scene(sc, precision=prec, device=local, stream=stream.cuda_stream,
                                        level0_operator=args.level0_operator, k_nullspace=args.k_nullspace)
        ctx0.step(sc.dt, args.cpu_iters)
        err = frame_errors(ctx0, sim, sc)
        ctx0.close()
        out["cpu_baseline"] = {
            "value": ms_o, "unit": UNIT, "cores": 1, "kind": "oracle", "measured_at_config": True,
            "iteration_ms": per_iter, "setup_ms": setup,
            "sample": (f"oracle (fp64, 1 core) on the full {sc.name}: frame 0 with setup + {args.cpu_iters} of "
                       f"{sc.n_iters} outer iterations timed ({setup:.0f} ms setup, {per_iter:.0f} ms per "
                       f"iteration); value = setup/20 + {sc.n_iters} x iteration"),
            "gpu_vs_oracle_same_frame": {"frame": 0, "outer_iterations": args.cpu_iters, **err}}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    # 20 warm-up frames: the timed window (frames 20..39) starts with the scheduled lazy setup of frame 20 on
    # the state after the initial release transient, i.e. exactly one scheduled setup per window (SURVEY.md
    # §8(d)) on a hierarchy of the running simulation; frames 0..19 run on the hierarchy of the squashed
    # initial state, which is 20-30 % more expensive
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="block1.67M")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=1,
                    help="outer iterations of the oracle's frame-0 sample at the full configuration")
    ap.add_argument("--k-nullspace", type=int, default=1,
                    help="near-kernel vectors per aggregate (SURVEY.md §8(f) f2; 1 = the paper's hierarchies, reading c1)")
    ap.add_argument("--level0-operator", type=int, default=1, choices=[0, 1],
                    help="1: matrix-free level 0 (default), 0: assembled-CSR level-0 passes")
    ap.add_argument("--partitioned", action="store_true",
                    help="N=1 only: run the row-partitioned (NCCL) code path on a 1-rank communicator")
    ap.add_argument("--profile-frames", type=int, default=2, help="frames timed per level-0 pass for the roofline")
    ap.add_argument("--dry-run", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    ws = os.environ.get("WORLD_SIZE")
    if ws is None and args.gpus > 1:
        return spawn(args.gpus)
    if int(ws or 1) != args.gpus:
        print(f"error: --gpus {args.gpus} but WORLD_SIZE={ws or 1}", file=sys.stderr)
        return 2
    if args.dry_run:  # launcher check only (tests): what each rank sees, no CUDA
        rank, world, local = dist_env()
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": world, "gpus_arg": args.gpus, "local_rank": local}),
                  flush=True)
        return 0
    return run_ours(args)


def spawn(n):
    """`--gpus N` without a launcher: run this script under torch.distributed.run with N ranks (one per
    GPU, rendezvous on 127.0.0.1); rank 0's JSON line passes through."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
