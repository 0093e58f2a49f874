#!/usr/bin/env python
"""Benchmark of the PBD-R substep loop (BASELINE.json metric: particle-substeps/s
at 1/2/4/8 B200; achieved HBM GB/s vs peak).

A "step" is one frame: cfg.substeps substeps, each = integrate + hash grid
(cell keys, onesweep sort, cell ranges, contact candidates) + cfg.solver_iterations
fused iteration kernels, replayed from one CUDA graph.

Default workload (N=1): config 4 (BASELINE.json configs[3]) -- 4096 batched
independent scenes of 16 cubes (14,155,776 particles), the largest config the
metric's 1/2/4/8-GPU scaling is quoted on that shards with no communication.
Under torchrun each rank simulates its own 4096 scenes (weak scaling). Other
configs: --config 1..5. --config 5 under torchrun runs the single giant scene
split into x-slabs (paper_2603_14634_b200/slab.py): each rank owns the bodies
whose com lies in its slab, ghosts are refreshed over NCCL after every
iteration, bodies migrate at frame boundaries (strong scaling: the scene is
fixed as N grows). C1-C3 run replicas under torchrun.

--impl reference times the oracle restatement of the reference's CPU solver
(the reference's own solver.cpp is absent from /root/reference, so the port is
the reference arm) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_ITERATION = 96    # read pos4, vel4, rest4, init4 (64 B) + write pos4, vel4 (32 B)
BYTES_PER_SUBSTEP = 1120    # 10 x 96 + integrate 80 + hash 80


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--scale", type=int, default=0, help="config size knob (0 = BASELINE size)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--preroll", type=int, default=0,
                    help="untimed frames simulated before the warm-up (measure a later, contact-rich window)")
    ap.add_argument("--tile-kp", type=int, default=0, help="force the iteration tile shape (2, 4, 8; 0 = automatic)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-slices", type=int, default=16,
                    help="batched config: drive the e2e leg as this many handles/streams (1 = one handle)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.3)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[4:8]))
            except ValueError:
                continue
        if not rows:
            return None
        sm = np.array([r[0] for r in rows])
        mx = max(r[1] for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        loaded = sm[sm >= 0.5 * sm.max()] if sm.max() > 0 else sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config_id):
    """Per-launch DRAM bytes of the iteration kernel from the committed ncu
    --set full summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_iteration_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        entry = d.get(f"c{config_id}")
        return None if entry is None else float(entry["dram_bytes_per_launch"])
    except (OSError, ValueError, KeyError):
        return None


def workload(args, rank, world):
    from paper_2603_14634_b200 import pbdr as P
    cid = args.config
    if cid == 4:
        from paper_2603_14634_b200 import shard as S
        sh = S.c4_shard(rank, world, args.scale if args.scale > 0 else 4096)
        g = S.generate_c4_shard(sh, seed=args.seed)
        name = P.CONFIG_NAMES[4]
        extra = {"scenes_per_gpu": sh.scenes_per_rank, "scenes_total": sh.total_scenes,
                 "parallelism": f"scene-shard x{world} (no collective in the data path)"}
    else:
        g = P.GeneratedScene(cid, seed=args.seed, scale=args.scale)
        name = P.CONFIG_NAMES[cid]
        extra = {"parallelism": f"replicas x{world}" if world > 1 else "single-gpu"}
    return g, name, extra


def cpu_sample_scene(args):
    """Bounded sample of the same workload for the CPU arm (about 10-30 s)."""
    from paper_2603_14634_b200 import pbdr as P
    if args.config == 4:
        return P.GeneratedScene(4, seed=args.seed, scale=64), "64 of the 4096 scenes (221,184 particles)"
    if args.config == 3:
        return P.GeneratedScene(3, seed=args.seed, scale=512), "first 512 of the 8192 bodies"
    if args.config == 5:
        return P.GeneratedScene(5, seed=args.seed, scale=16), "16x16x8 cubes of the 64x64x32 grid"
    return P.GeneratedScene(args.config, seed=args.seed), "the whole scene"


def run_cpu(args, substeps_per_step):
    """Oracle port on all host threads; returns (rate, cores, sample, seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    g, sample = cpu_sample_scene(args)
    threads = os.cpu_count() or 1
    o = pyoracle.Oracle(g.desc, g.cfg, threads=threads)
    assert o.step(1) == 0  # warm-up substep
    t0 = time.perf_counter()
    done = 0
    while True:
        assert o.step(substeps_per_step) == 0
        done += substeps_per_step
        if time.perf_counter() - t0 > 12.0:  # about 10-30 s of CPU work
            break
    dt = time.perf_counter() - t0
    rate = g.num_particles * done / dt
    return rate, threads, f"{sample}, {done} substeps after 1 warm-up substep", dt


def reference_arm(args, rank, world):
    if rank != 0:
        return
    from paper_2603_14634_b200 import pbdr as P
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    g, sample = cpu_sample_scene(args)
    threads = os.cpu_count() or 1
    o = pyoracle.Oracle(g.desc, g.cfg, threads=threads)
    for _ in range(args.warmup):
        assert o.step(1) == 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        assert o.step(1) == 0  # each step: one substep of the bounded sample
    dt = time.perf_counter() - t0
    rate = g.num_particles * args.steps / dt
    name = P.CONFIG_NAMES[args.config]
    line = {
        "impl": "reference", "metric": "particle-substeps/s", "value": rate, "unit": "particle-substeps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded BASELINE.json config)",
        "config": {"workload": name, "particles_sampled": g.num_particles, "step": "1 substep of the sample"},
        "cpu_baseline": {"value": rate, "unit": "particle-substeps/s", "cores": threads, "kind": "port",
                         "sample": f"{sample}; oracle/pbdr_oracle.cpp restatement (reference solver.cpp absent)"},
        "e2e": {"value": rate, "unit": "particle-substeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_e2e(args, solver, g, rank, world, local, total_particles, subs, barrier):
    """End to end through the C-ABI with host buffers: every step uploads the
    state from pinned host memory, advances one frame and reads it back. For
    the batched config the rank's scenes are driven as `--e2e-slices` slices
    (one handle and CUDA stream each, asynchronous calls), so one slice's
    transfers overlap another's compute; otherwise one handle, synchronous."""
    import torch
    import torch.distributed as dist
    from paper_2603_14634_b200 import pbdr as P
    steps = max(1, min(args.steps, 5))
    slices = []
    if args.config == 4 and args.e2e_slices > 1:
        from paper_2603_14634_b200 import shard as S
        per_rank = args.scale if args.scale > 0 else 4096
        k = args.e2e_slices
        per = per_rank // k
        for i in range(k):
            sh = S.SceneShard(rank * k + i, world * k, per)
            gi = S.generate_c4_shard(sh, seed=args.seed)
            # shard() numbers scenes rank-major, so slice i of rank r holds the
            # same scenes as rows [i*per, (i+1)*per) of that rank's batch.
            slices.append(P.GpuSolver(gi.desc, gi.cfg, device=local))
    else:
        slices.append(solver)
    bufs = []
    for s in slices:
        hp = torch.empty((s.n, 4), dtype=torch.float32, pin_memory=True).numpy()
        hv = torch.empty((s.n, 4), dtype=torch.float32, pin_memory=True).numpy()
        s.read_f32(hp, hv)
        s.step_frames(1)  # graphs built, warm
        s.read_f32(hp, hv)
        bufs.append((hp, hv))
    barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        for s, (hp, hv) in zip(slices, bufs):
            s.write_f32_async(hp, hv)
            s.step_frames_async(1)
            s.read_f32_async(hp, hv)
        for s in slices:
            s.sync()
    dt = time.perf_counter() - t0
    te = torch.tensor([dt], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    n_e2e = sum(s.n for s in slices) * world
    nbytes = sum(hp.nbytes + hv.nbytes for hp, hv in bufs)
    out = {"value": n_e2e * subs * steps / float(te.item()), "unit": "particle-substeps/s",
           "h2d_bytes_per_step": int(nbytes), "d2h_bytes_per_step": int(nbytes), "steps": steps,
           "slices": len(slices), "timer": "host wall clock, max over ranks"}
    for s in slices:
        if s is not solver:
            s.close()
    return out


def slab_bench(args, rank, world, local):
    """Config 5 split into x-slabs across the ranks (one scene, NCCL halo)."""
    import torch
    import torch.distributed as dist
    from paper_2603_14634_b200 import pbdr as P
    from paper_2603_14634_b200 import slab as S

    g = P.GeneratedScene(5, seed=args.seed, scale=args.scale)
    nb = g.desc.num_bodies
    off = g.array("body_offsets", nb + 1, np.int64)
    rho, h = S.body_reach(g.array("rest_offsets", 3 * g.num_particles), off, g.array("radius", g.num_particles))
    solver = P.GpuSolver(g.desc, g.cfg, device=local)
    eng = S.GpuEngine(solver, g.cfg)
    run = S.SlabRunner(eng, rank, world, S.TorchComm(), off, rho=rho, h=h, margin=0.1)
    run.start()
    run.step_frames(max(3, args.warmup))
    dist.barrier()
    torch.cuda.synchronize(local)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(eng.stream)
        run.step_frames(args.steps)
        ev1.record(eng.stream)
        ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    dist.barrier()
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    n_total = solver.n
    subs = g.cfg.substeps
    value = n_total * subs * args.steps / (ms_max / 1e3)
    owned = torch.tensor([sum(int(run.bcount[b]) for b in run.owned)], dtype=torch.int64, device=f"cuda:{local}")
    owned_max = owned.clone()
    dist.all_reduce(owned_max, op=dist.ReduceOp.MAX)
    ghosts = sum(len(v) for v in run.plan.recv_bodies.values())
    peak, peak_src = measured_peak()
    if rank == 0:
        line = {
            "metric": "particle-substeps/s", "value": value, "unit": "particle-substeps/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded BASELINE.json config 5, host generator)",
            "config": {"workload": P.CONFIG_NAMES[5], "particles_total": n_total, "bodies_total": nb,
                       "substeps_per_step": subs, "iterations": g.cfg.solver_iterations,
                       "parallelism": f"x-slab x{world}, NCCL halo after every iteration, migration per frame",
                       "max_owned_particles_per_gpu": int(owned_max.item()), "ghost_bodies_rank0": ghosts,
                       "ghost_band_m": run.geo.ghost_band,
                       "l2": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "achieved": (value / world) * BYTES_PER_SUBSTEP / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": (value / world) * BYTES_PER_SUBSTEP / (peak * 1e9),
                         "traffic": None, "kernel": "whole substep (per GPU)", "peak_source": peak_src},
            "cpu_baseline": None,
            "e2e": None,
            "gpu_launches": int(solver.info.launches_per_frame * args.steps),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    solver.close()
    dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if args.config == 5 and world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        slab_bench(args, rank, world, local)
        return

    import torch
    import torch.distributed as dist
    from paper_2603_14634_b200 import pbdr as P

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    g, name, extra = workload(args, rank, world)
    if args.tile_kp:
        g.desc.tile_kp = args.tile_kp
    solver = P.GpuSolver(g.desc, g.cfg, device=local)
    n = solver.n
    subs = g.cfg.substeps
    iters = g.cfg.solver_iterations

    if args.preroll > 0:
        solver.step_frames(args.preroll)
    # Warm-up (also instantiates the per-frame CUDA graphs).
    solver.step_frames(max(3, args.warmup))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(local)

    barrier()
    with ClockSampler(local) as clocks:
        ms = solver.time_frames(args.steps)  # CUDA events on the library's stream
    barrier()
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_particles = n * world
    value = total_particles * subs * args.steps / (ms_max / 1e3)

    # End-to-end through the C-ABI with host buffers: every step uploads the
    # state from pinned host memory, advances one frame and reads it back.
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, solver, g, rank, world, local, total_particles, subs, barrier)

    # Roofline of the dominant kernel (the fused iteration) from per-launch
    # CUDA events on the library's stream, separate run of the same workload.
    prof = solver.profile_frames(1)
    frame_ms = sum(v[0] for v in prof.values())
    it_ms, it_launches = prof["iteration"]
    it_avg_ms = it_ms / max(1, it_launches)
    # Scenes without candidate pairs run a substep's iterations in one launch.
    iters_per_launch = max(1, (subs * iters) // max(1, it_launches))
    alg_bytes = n * BYTES_PER_ITERATION * iters_per_launch
    achieved = alg_bytes / (it_avg_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": ncu_traffic(args.config), "kernel": "k_iteration",
                "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": it_avg_ms,
                "share_of_frame": it_ms / frame_ms if frame_ms > 0 else None, "peak_source": peak_src,
                "whole_substep_frac": (value / world) * BYTES_PER_SUBSTEP / (peak * 1e9),
                "per_kernel_ms_per_frame": {k: round(v[0], 4) for k, v in prof.items()}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, cores, sample, secs = run_cpu(args, 1)
        cpu = {"value": rate, "unit": "particle-substeps/s", "cores": cores, "kind": "port",
               "sample": f"{sample} ({secs:.1f} s)"}

    info = solver.info
    if rank == 0:
        line = {
            "metric": "particle-substeps/s", "value": value, "unit": "particle-substeps/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded BASELINE.json config, host generator)",
            "config": {"workload": name, "particles_per_gpu": n, "bodies_per_gpu": info.num_bodies,
                       "substeps_per_step": subs, "iterations": iters, "frame_rate_hz": g.cfg.frame_rate,
                       "l2": f"inputs larger than L2 ({n * 64 / 1e6:.0f} MB particle state per GPU)"
                       if n * 64 > 126e6 else "state fits in L2 (latency-bound config)",
                       "timed_frames": f"{args.preroll + max(3, args.warmup) + 1}..{args.preroll + max(3, args.warmup) + args.steps}",
                       **extra},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(info.launches_per_frame * args.steps),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
