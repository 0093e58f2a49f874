#!/usr/bin/env python
"""Benchmark of the PBD-R substep loop (BASELINE.json metric: particle-substeps/s
at 1/2/4/8 B200; achieved HBM GB/s vs peak).

A "step" is one frame: cfg.substeps substeps, each = integrate + hash grid
(cell keys, onesweep sort, cell ranges, contact candidates) + cfg.solver_iterations
fused iteration kernels, replayed from one CUDA graph.

Default workload (N=1): config 5 (BASELINE.json configs[4]) -- the single giant
scene of 131,072 cubes (67,108,864 particles), the largest config, which fits
one B200 (25 GB of the 180). The timed window is the LAST K frames of the
config's own run (frames F-K .. F-1 of F = 100): the warm-up frames and the
frames before the window are simulated untimed-by-contract but measured too,
so the line also carries the whole-run rate (frames W .. F-1) and the
free-flight rate of its first frames. `--window head` times frames W .. W+K-1
instead (free flight). C4 (4096 batched scenes) rides along as a `secondary`
entry (whole run and tail window), `--config N` runs any other config.

Under torchrun: C4 shards scenes per rank (weak scaling, no collective);
C5 runs as x-slabs of a grid that grows with the rank count (weak scaling:
--slab-columns x-columns of 64 x 32 cubes per GPU, 64 = a whole config 5 per
GPU) through the native C++ slab driver with an NCCL halo (csrc/pbdr_slab.cu);
C1-C3 run replicas.

--impl reference times the oracle restatement of the reference's CPU solver
(the reference's own solver.cpp is absent from /root/reference, so the port is
the reference arm) on the host cores, rank 0 only, on a bounded
sample of the same workload. It maps only the host-only scene generator
(libpbdr_host.so) and the oracle -- never the CUDA library.
"""
from __future__ import annotations

import argparse
import hashlib
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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--scale", type=int, default=0, help="config size knob (0 = BASELINE size)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--window", choices=["tail", "head"], default="tail",
                    help="timed K frames: the last K of the config's run (tail) or the first after warm-up (head)")
    ap.add_argument("--tile-kp", type=int, default=0, help="force the iteration tile shape (2, 4, 8; 0 = automatic)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the C4 secondary entry")
    ap.add_argument("--slab-columns", type=int, default=64,
                    help="config 5 under torchrun: x-columns of cubes per rank (weak scaling; 64 = a whole "
                         "BASELINE config 5 per GPU, 8 = BASELINE.md's 1/8 of it per GPU)")
    ap.add_argument("--halo-refresh", type=int, default=0, choices=[0, 1],
                    help="config 5 slabs: 0 = ghost positions after every iteration (exact), 1 = once per substep")
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


def build_id():
    """Hash of the CUDA sources the library is built from: an ncu capture is
    quoted as `traffic` only for the build it was taken on."""
    d = os.path.join(ROOT, "paper_2603_14634_b200", "csrc")
    h = hashlib.sha1()
    for name in sorted(os.listdir(d)):
        if name.endswith((".cu", ".cuh", ".h")):
            with open(os.path.join(d, name), "rb") as f:
                h.update(name.encode() + f.read())
    return h.hexdigest()[:16]


def ncu_traffic(workload_name, window):
    """DRAM bytes per iteration launch (ncu --set full: dram__bytes_read.sum +
    dram__bytes_write.sum, averaged over one substep's iteration launches) from
    profiles/ncu_iteration_summary.json, if it was captured on this build for
    this workload and window; else None."""
    path = os.path.join(ROOT, "profiles", "ncu_iteration_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(f"{workload_name}:{window}")
        if e is None or e.get("build") != build_id():
            return None, None
        return float(e["dram_bytes_per_launch"]), e
    except (OSError, ValueError, KeyError):
        return None, None


def config_frames(cid):
    return {1: 1000, 2: 1000, 3: 500, 4: 200, 5: 100}[cid]


def workload_size(args, rank, world):
    """(particles, bodies) per GPU of the workload, without building it on
    the device (the reference arm quotes the same config block)."""
    from paper_2603_14634_b200 import pbdr as P
    cid = args.config
    if cid == 4:
        s = args.scale if args.scale > 0 else 4096
        return s * 3456, s * 16
    if cid == 5:
        gx = args.scale if args.scale > 0 else 64
        nb = gx * gx * max(1, gx // 2)
        return nb * 512, nb
    g = P.GeneratedScene(cid, seed=args.seed, scale=args.scale)
    return int(g.num_particles), int(g.num_bodies)


def window_frames(args):
    """(first timed frame, last timed frame) -- 0-based frame indices."""
    F = config_frames(args.config)
    W = max(3, args.warmup)
    K = args.steps
    first = max(W, F - K) if args.window == "tail" else W
    return first, first + K - 1


def config_block(args, rank, world):
    """The `config` object both arms print (same workload, same window)."""
    from paper_2603_14634_b200 import pbdr as P
    n, nb = workload_size(args, rank, world)
    first, last = window_frames(args)
    block = {"workload": P.CONFIG_NAMES[args.config], "particles_per_gpu": n, "bodies_per_gpu": nb,
             "substeps_per_step": 10, "iterations": 10, "frame_rate_hz": 240.0,
             "run_frames": config_frames(args.config),
             "timed_frames": f"{first}..{last} ({args.window} of the run; frames 0..{first - 1} simulated before)",
             "l2": (f"inputs larger than L2 ({n * 64 / 1e6:.0f} MB particle state per GPU)" if n * 64 > 126e6
                    else "state fits in L2 (latency-bound config)")}
    if args.config == 4:
        block.update({"scenes_per_gpu": nb // 16, "scenes_total": world * (nb // 16),
                      "parallelism": f"scene-shard x{world} (no collective in the data path)"})
    else:
        block["parallelism"] = f"replicas x{world}" if world > 1 else "single-gpu"
    if args.tile_kp:
        block["tile_kp"] = args.tile_kp
    return block


def workload(args, rank, world):
    from paper_2603_14634_b200 import pbdr as P
    cid = args.config
    if cid == 4:
        from paper_2603_14634_b200 import shard as S
        sh = S.c4_shard(rank, world, args.scale if args.scale > 0 else 4096)
        return S.generate_c4_shard(sh, seed=args.seed)
    return P.GeneratedScene(cid, seed=args.seed, scale=args.scale)


def cpu_sample_scene(args):
    """Bounded sample of the same workload for the CPU arms (about 10-30 s),
    built by the host-only generator (no CUDA library is mapped)."""
    from paper_2603_14634_b200 import pbdr as P
    if args.config == 4:
        return P.GeneratedScene(4, seed=args.seed, scale=64), "64 of the 4096 scenes (221,184 particles)"
    if args.config == 3:
        return P.GeneratedScene(3, seed=args.seed, scale=512), "first 512 of the 8192 bodies"
    if args.config == 5:
        return (P.GeneratedScene(5, seed=args.seed, scale=16),
                "16x16x8 of the 64x64x32 cubes (1,048,576 particles), same generator, frame 0")
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
    """The reference's CPU implementation of the path (the oracle restatement:
    the reference's solver.cpp is absent) on all host threads, one substep of
    the bounded sample per step. Maps libpbdr_host.so + oracle only."""
    if rank != 0:
        return
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
    line = {
        "impl": "reference", "metric": "particle-substeps/s", "value": rate, "unit": "particle-substeps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded BASELINE.json config, host generator)",
        "config": config_block(args, rank, world),
        "cpu_baseline": {"value": rate, "unit": "particle-substeps/s", "cores": threads, "kind": "port",
                         "sample": f"{sample}; one substep per step; oracle/pbdr_oracle.cpp restatement "
                                   f"(the reference's solver.cpp is absent)"},
        "e2e": {"value": rate, "unit": "particle-substeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_e2e(args, solver, g, rank, world, local, subs, barrier):
    """End to end through the C-ABI with host buffers, continuing the run.

    Headline leg: every step uploads the state (pos4 + vel4, fp32, from
    pinned host memory), advances one frame and reads it back. For the batched
    config the rank's scenes are driven as `--e2e-slices` slices (one handle and
    CUDA stream each, asynchronous calls), so one slice's transfers overlap
    another's compute; otherwise one handle.

    `api_fp64` leg: the reference-shaped calls -- pbdr_gpu_write_particles
    (fp64, caller order) + one frame + pbdr_gpu_read_particles."""
    import torch
    import torch.distributed as dist
    from paper_2603_14634_b200 import pbdr as P
    steps = max(1, min(args.steps, 3))
    slices = []
    if args.config == 4 and args.e2e_slices > 1:
        from paper_2603_14634_b200 import shard as S
        per_rank = args.scale if args.scale > 0 else 4096
        k = args.e2e_slices
        per = per_rank // k
        for i in range(k):
            sh = S.SceneShard(rank * k + i, world * k, per)
            gi = S.generate_c4_shard(sh, seed=args.seed)
            slices.append(P.GpuSolver(gi.desc, gi.cfg, device=local))
    else:
        slices.append(solver)
    bufs = []
    for s in slices:
        hp = torch.empty((s.n, 4), dtype=torch.float32, pin_memory=True).numpy()
        hv = torch.empty((s.n, 4), dtype=torch.float32, pin_memory=True).numpy()
        s.read_f32(hp, hv)
        if s is not solver:
            s.step_frames(1)  # graphs built, warm
            s.read_f32(hp, hv)
        bufs.append((hp, hv))

    def timed(fn):
        barrier()
        t0 = time.perf_counter()
        fn()
        dt = time.perf_counter() - t0
        te = torch.tensor([dt], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        return float(te.item())

    def f32_leg():
        for _ in range(steps):
            for s, (hp, hv) in zip(slices, bufs):
                s.write_f32_async(hp, hv)
                s.step_frames_async(1)
                s.read_f32_async(hp, hv)
            for s in slices:
                s.sync()

    dt = timed(f32_leg)
    n_e2e = sum(s.n for s in slices) * world
    nbytes = sum(hp.nbytes + hv.nbytes for hp, hv in bufs)
    out = {"value": n_e2e * subs * steps / dt, "unit": "particle-substeps/s",
           "h2d_bytes_per_step": int(nbytes), "d2h_bytes_per_step": int(nbytes), "steps": steps,
           "slices": len(slices), "timer": "host wall clock, max over ranks",
           "calls": "pbdr_gpu_write_f32_async + pbdr_gpu_step_frames_async(1) + pbdr_gpu_read_f32_async, pinned"}
    for s in slices:
        if s is not solver:
            s.close()
    del bufs

    # Reference-shaped fp64 transfer (Scene::particles order) on the main handle.
    pos, vel = solver.read_particles()

    def api_leg():
        for _ in range(steps):
            solver.write_particles(pos, vel)
            solver.step_frames(1)
            p2, v2 = solver.read_particles()
            pos[:] = p2
            vel[:] = v2

    dt_api = timed(api_leg)
    out["api_fp64"] = {"value": solver.n * world * subs * steps / dt_api, "unit": "particle-substeps/s",
                       "h2d_bytes_per_step": int(pos.nbytes + vel.nbytes),
                       "d2h_bytes_per_step": int(pos.nbytes + vel.nbytes), "steps": steps,
                       "calls": "pbdr_gpu_write_particles + pbdr_gpu_step_frames(1) + pbdr_gpu_read_particles "
                                "(fp64, caller order, pageable host arrays)"}
    return out


def roofline_block(args, solver, name, value, world):
    """Dominant kernel (the fused iteration, all its launches in one frame):
    algorithmic bytes (n x 96 B per particle-iteration) over its
    device time from per-launch CUDA events on the library's stream."""
    prof = solver.profile_frames(1)
    frame_ms = sum(v[0] for v in prof.values())
    it_ms, it_launches = prof["iteration"]
    subs, iters = 10, 10
    alg_total = solver.n * BYTES_PER_ITERATION * subs * iters  # every particle, every iteration
    alg_per_launch = alg_total / max(1, it_launches)
    avg_ms = it_ms / max(1, it_launches)
    achieved = alg_per_launch / (avg_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()
    traffic, ncu = ncu_traffic(name, args.window)
    out = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "traffic": traffic, "kernel": "k_iteration (all launches of a frame)",
           "algorithmic_bytes_per_launch": alg_per_launch, "avg_launch_ms": avg_ms, "launches_per_frame": it_launches,
           "share_of_frame": it_ms / frame_ms if frame_ms > 0 else None, "peak_source": peak_src,
           "frac_basis": "algorithmic bytes (SURVEY 8d); measured DRAM bytes in `traffic` (ncu, same build)",
           "whole_substep_frac": (value / world) * BYTES_PER_SUBSTEP / (peak * 1e9),
           "per_kernel_ms_per_frame": {k: round(v[0], 4) for k, v in prof.items()},
           "build": build_id()}
    if ncu is not None:
        out["ncu"] = {k: ncu[k] for k in ("limiter", "sm_throughput_pct", "dram_gbs", "capture") if k in ncu}
    return out


def secondary_c4(args, local):
    """C4 (4096 batched scenes) on the same GPU: whole run and tail window."""
    from paper_2603_14634_b200 import pbdr as P
    g = P.GeneratedScene(4, seed=args.seed)
    s = P.GpuSolver(g.desc, g.cfg, device=local)
    F, K, W = config_frames(4), args.steps, max(3, args.warmup)
    s.step_frames(W)
    with ClockSampler(local) as clocks:
        pre = s.time_frames(F - K - W)
        tail = s.time_frames(K)
    n = s.n
    s.close()
    return {"workload": P.CONFIG_NAMES[4], "particles": n,
            "tail_value": n * 10 * K / (tail / 1e3), "tail_frames": f"{F - K}..{F - 1}",
            "whole_run_value": n * 10 * (F - W) / ((pre + tail) / 1e3), "whole_run_frames": f"{W}..{F - 1}",
            "unit": "particle-substeps/s", "clocks": clocks.summary()}


def native_slab_bench(args, rank, world, local):
    """Config 5 as x-slabs, one rank per GPU, weak scaling: each rank generates
    and holds only its slab (args.slab_columns x-columns of 64 x 32 cubes) plus
    3 ghost columns per side, and the C++ driver (csrc/pbdr_slab.cu) runs the
    substeps with the ghost halo over NCCL send/recv, overlapped with the
    interior tiles. Device time (CUDA events on the handle's stream around the
    K frames, including the per-frame repartition), max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2603_14634_b200 import pbdr as P
    from paper_2603_14634_b200 import slab_native as S

    spec = S.c5_slab_spec(rank, world, columns_per_rank=args.slab_columns)
    g = S.generate(spec, seed=args.seed)
    solver = P.GpuSolver(g.desc, g.cfg, device=local)
    ids = [P.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    S.attach(solver, spec, refresh=args.halo_refresh, overlap=1, nccl_id=ids[0])
    solver.slab_start()
    W = max(3, args.warmup)
    first, last = window_frames(args)
    solver.slab_step_frames(W)
    if first > W:
        solver.slab_step_frames(first - W)
    stream = torch.cuda.ExternalStream(solver.stream_handle(), device=torch.device("cuda", local))
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize(local)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        solver.slab_step_frames(args.steps)
        ev1.record(stream)
        ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    dist.barrier()
    info = solver.slab_info()
    t = torch.tensor([ms, info["owned_particles"], info["ghost_bodies"], info["halo_bytes_per_iteration"],
                      info["migrations"]], dtype=torch.float64, device=f"cuda:{local}")
    tmax = t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    tsum = t.clone()
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    ms_max = float(tmax[0].item())
    n_total = int(tsum[1].item())
    subs = g.cfg.substeps
    value = n_total * subs * args.steps / (ms_max / 1e3)
    peak, peak_src = measured_peak()
    if rank == 0:
        line = {
            "metric": "particle-substeps/s", "value": value, "unit": "particle-substeps/s", "n_gpus": world,
            "steps": args.steps, "warmup": W, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded BASELINE.json config 5 grid, rank-local generation)",
            "config": {"workload": P.CONFIG_NAMES[5], "grid": [spec.gx, spec.gy, spec.gz],
                       "columns_per_gpu": args.slab_columns, "particles_total": n_total,
                       "particles_per_gpu": n_total // world, "substeps_per_step": subs,
                       "iterations": g.cfg.solver_iterations, "frame_rate_hz": 240.0,
                       "timed_frames": f"{first}..{last} ({args.window} of the run)",
                       "parallelism": f"x-slab x{world}: native driver, NCCL halo "
                                      f"({'every iteration' if args.halo_refresh == 0 else 'once per substep'}),"
                                      " overlapped with interior tiles, migration per frame",
                       "max_ghost_bodies_per_gpu": int(tmax[2].item()),
                       "max_halo_bytes_per_iteration": int(tmax[3].item()),
                       "migrations": int(tsum[4].item()), "l2": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "achieved": (value / world) * BYTES_PER_SUBSTEP / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": (value / world) * BYTES_PER_SUBSTEP / (peak * 1e9),
                         "traffic": None, "kernel": "whole substep (per GPU, algorithmic 1120 B)",
                         "peak_source": peak_src},
            "cpu_baseline": None,
            "e2e": None,
            # graph-mode count of the same scene plus, per iteration, the halo's
            # gather / scatter launches (4 per peer at the last iteration)
            "gpu_launches": int((solver.info.launches_per_frame + subs * g.cfg.solver_iterations * 4) * args.steps),
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
        native_slab_bench(args, rank, world, local)
        return

    import torch
    import torch.distributed as dist
    from paper_2603_14634_b200 import pbdr as P

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    g = workload(args, rank, world)
    name = P.CONFIG_NAMES[args.config]
    if args.tile_kp:
        g.desc.tile_kp = args.tile_kp
    solver = P.GpuSolver(g.desc, g.cfg, device=local)
    n = solver.n
    subs = g.cfg.substeps
    W = max(3, args.warmup)
    first, last = window_frames(args)
    F = config_frames(args.config)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(local)

    # Warm-up: frames 0..W-1 (also instantiates the per-frame CUDA graphs).
    solver.step_frames(W)
    # Frames W..first-1: outside the contract's timed region, measured with the
    # same device events for the whole-run figure.
    pre_ms = solver.time_frames(first - W) if first > W else 0.0
    barrier()
    with ClockSampler(local) as clocks:
        ms = solver.time_frames(args.steps)  # CUDA events on the library's stream
    barrier()
    t = torch.tensor([ms, pre_ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, pre_max = float(t[0].item()), float(t[1].item())
    total_particles = n * world
    value = total_particles * subs * args.steps / (ms_max / 1e3)
    runs = {}
    if args.window == "tail" and last >= F - 1:
        runs["whole_run"] = {"value": total_particles * subs * (last + 1 - W) / ((pre_max + ms_max) / 1e3),
                             "frames": f"{W}..{last}", "note": "device time of every frame after the warm-up"}
    if pre_max > 0 and first - W >= 1:
        runs["before_window"] = {"value": total_particles * subs * (first - W) / (pre_max / 1e3),
                                 "frames": f"{W}..{first - 1}"}

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, solver, g, rank, world, local, subs, barrier)

    roofline = roofline_block(args, solver, name, value, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, cores, sample, secs = run_cpu(args, 1)
        cpu = {"value": rate, "unit": "particle-substeps/s", "cores": cores, "kind": "port",
               "sample": f"{sample} ({secs:.1f} s)"}

    info = solver.info
    solver.close()
    del g
    secondary = None
    if rank == 0 and world == 1 and args.config == 5 and not args.no_secondary and args.scale == 0:
        secondary = secondary_c4(args, local)
    if rank == 0:
        line = {
            "metric": "particle-substeps/s", "value": value, "unit": "particle-substeps/s", "n_gpus": world,
            "steps": args.steps, "warmup": W, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded BASELINE.json config, host generator)",
            "config": config_block(args, rank, world),
            "runs": runs,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(info.launches_per_frame * args.steps),
            "clocks": clocks.summary(),
        }
        if secondary is not None:
            line["secondary"] = secondary
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
