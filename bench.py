#!/usr/bin/env python
"""Benchmark of the hybrid-snapshot step (BASELINE.json metric, BJ:2):
hybrid-step cell-updates/s (fp64) at 2D 2048^2, with the fill pass's fraction of the
measured HBM roofline.

python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 4] [--fraction 0.1]

One step = one hybrid step of Algorithm 1: H1 dt, H3 masked RK3, H4-H5 gappy
solve, H6 fill + indicator (+H9/H10 window Gram row), H7 seam filter, H10-H12 basis update,
H8 sampling -- every row of SURVEY §8(a).  The w-1 warm-up full steps that fill the window
are set-up, outside the timed region.  Multi-GPU: one independent problem per rank (seed
+ rank), no data-path collective ("scaling": "weak").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "hybrid-step cell-updates/s (fp64) at 2D 2048²; % of HBM / FP64-TC roofline"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.path = f"/tmp/hrom_clocks_{os.getpid()}.csv"
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 8:
                try:
                    rows.append((float(f[0]), float(f[1]), f[4], f[5], f[6], f[7]))
                except ValueError:
                    pass
        if not rows:
            return None
        sm = sorted(r[0] for r in rows)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": rows[0][1], "reasons": sorted(reasons), "samples": len(rows)}


def rank_seed(config: int, rank: int) -> int:
    """Each rank runs an independent problem of the same shape (weak scaling)."""
    return config + 1000 * rank


def reduce_max_over_ranks(vals, dist=None, device="cpu"):
    """Max over ranks of the per-rank device times (the only collective of the bench)."""
    if dist is None:
        return [float(v) for v in vals]
    import torch
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def whole_job_value(cells_per_rank: int, world: int, ms_step: float) -> float:
    """Whole-job cell-updates/s: the cells of all ranks over the slowest rank's step time."""
    return cells_per_rank * world / (ms_step / 1000.0)


def fill_bytes(wl, n_s: int) -> int:
    """Algorithmic bytes of one fill-pass launch: read the w+1 window
    columns and the Gram shift, write gamma_k; read the partial-HDM values and write the
    squared errors on the c*n_s S-hat DOFs; two N-bit masks."""
    D = wl.D
    return 8 * D * (wl.w + 1 + 1 + 1) + 16 * wl.c * n_s + 2 * (wl.N // 8)


def run_hrom(args, rank, world, local_rank):
    import numpy as np
    import torch
    from paper_2301_01718_b200 import inputs
    from paper_2301_01718_b200.hrom import HybridROM, SECTIONS
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    wl = inputs.config(args.config, f=args.fraction, seed=rank_seed(args.config, rank))
    q0 = inputs.initial_condition(wl)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        rom = HybridROM(wl, stream=stream, gram_mode=args.gram_mode)
        rom.set_state(torch.from_numpy(q0).cuda())
        # set-up: w-1 full steps + bootstrap (not timed)
        for _ in range(wl.w - 1):
            rom.step()
        # full-step throughput for contrast (separate context state is not needed: time 5 steps on a copy)
        rom.sync()
        # warm-up hybrid steps
        for _ in range(args.warmup):
            rom.step()
        rom.sync()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        clocks = ClockSampler(local_rank) if rank == 0 else None
        l0 = rom.launch_count()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/ selects these launches
        ev0.record(stream)
        for _ in range(args.steps):
            rom.step()
        rom.join()  # the last step's eigen-solve runs on the library's side stream: inside the timed region
        ev1.record(stream)
        torch.cuda.nvtx.range_pop()
        ev1.synchronize()
        rom.sync()
        launches = rom.launch_count() - l0
        ms_total = ev0.elapsed_time(ev1)
        ck = clocks.stop() if clocks else None
        # second pass over the next K steps with the library's per-section CUDA events on (they
        # serialise the side stream's overlap a little, so the headline pass above runs without
        # them): the fill pass's average launch time of the roofline object and the section split
        rom.profile(True)
        pv0 = torch.cuda.Event(enable_timing=True)
        pv1 = torch.cuda.Event(enable_timing=True)
        pv0.record(stream)
        for _ in range(args.steps):
            rom.step()
        rom.join()
        pv1.record(stream)
        pv1.synchronize()
        rom.sync()
        sec = rom.profile_read()
        rom.profile(False)
        ms_total_prof = pv0.elapsed_time(pv1)
        # S-hat size and mask stats (outside the timed region)
        n_s = int(H_count(rom, wl))
        # end-to-end through the C ABI with host buffers: put gamma_{k-1} from pinned host
        # memory, step, read gamma_k back (D2H) every step
        host = torch.empty((wl.c, wl.N), dtype=torch.float64, pin_memory=True)
        rom.get_state(host)
        rom.sync()
        e2e_steps = max(2, min(args.steps, 10))
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            rom.put_state(host)
            rom.step()
            rom.get_state(host)
        rom.join()
        e1.record(stream)
        e1.synchronize()
        rom.sync()
        ms_e2e = e0.elapsed_time(e1) / e2e_steps
        # full-step throughput for contrast
        fs = HybridROM(wl, stream=stream)
        fs.set_state(torch.from_numpy(q0).cuda())
        fs.full_step()
        fs.sync()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(5):
            fs.full_step()
        f1.record(stream)
        f1.synchronize()
        ms_full = f0.elapsed_time(f1) / 5
        fs.close()
    # max over ranks
    ms_step = ms_total / args.steps
    ms_step, ms_e2e = reduce_max_over_ranks([ms_step, ms_e2e], dist, "cuda")
    out = None
    if rank == 0:
        value = whole_job_value(wl.N, world, ms_step)
        peak, peak_src = measured_peaks()
        fill_ms, fill_n = sec["fill_pass"]
        fb = fill_bytes(wl, n_s)
        fill_avg_ms = fill_ms / max(fill_n, 1)
        achieved = fb / (fill_avg_ms / 1000.0) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "fill_traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        split = {k: round(v[0] / max(args.steps, 1), 4) for k, v in sec.items() if v[1]}
        out = {
            "metric": METRIC,
            "value": value,
            "unit": "cell-updates/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded config-4 blasts, BASELINE.json configs[3]; DESIGN.md §3)",
            "config": {"workload": wl.name, "grid": f"{wl.nx}x{wl.ny}", "cells": wl.N, "dofs": wl.D,
                       "window_w": wl.w, "rank_r": wl.r, "sample_fraction": wl.f, "halo": wl.h, "band_W": wl.W,
                       "gram_mode": "incremental-shifted" if args.gram_mode == 0 else "full-dmma",
                       "n_s_last": n_s, "l2": "inputs larger than L2 (window %.1f GB)" % ((wl.w + 2) * wl.D * 8 / 1e9),
                       "parallelism": f"independent problem per GPU x{world}"},
            "roofline": {"kernel": "fill_pass (H6+H9+H10 row)", "bound": "hbm", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": fb, "avg_launch_ms": fill_avg_ms,
                         "share_of_step": fill_ms / ms_total_prof if ms_total_prof > 0 else None,
                         "peak_source": peak_src,
                         "timed_in": "second pass of K steps with per-section CUDA events on the library's stream"},
            "section_ms_per_step": split,
            "section_pass_ms_per_step": ms_total_prof / args.steps,
            "full_step": {"ms": ms_full, "cell_updates_per_s": wl.N / (ms_full / 1000.0)},
            "clocks": ck,
            "e2e": {"value": whole_job_value(wl.N, world, ms_e2e), "unit": "cell-updates/s",
                    "h2d_bytes_per_step": wl.D * 8, "d2h_bytes_per_step": wl.D * 8, "ms_per_step": ms_e2e,
                    "steps": e2e_steps},
            "gpu_launches": int(launches),
        }
    rom.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return out


def run_slab(args, rank, world, local_rank):
    """--shard slab: ONE config-4 problem cut into row slabs, one per rank:
    halo rows to the neighbours and the small all-reduces of csrc/slab.cu over NCCL every step;
    strong scaling (the grid is fixed, value = N / step time).  The driver's default run is the
    replica mode; this mode exists for multi-GPU boxes and is exercised with one rank on one GPU."""
    import torch
    import torch.distributed as dist
    from paper_2301_01718_b200 import inputs, slab
    torch.cuda.set_device(local_rank)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world)
    wl = inputs.config(args.config, f=args.fraction, seed=rank_seed(args.config, 0))  # the same problem on every rank
    q0 = torch.from_numpy(inputs.initial_condition(wl)).cuda()
    comm = slab.DistComm()
    rom = slab.SlabROM(wl, rank, world)
    rom.set_state(q0)
    for _ in range(wl.w - 1 + args.warmup):
        rom.step(comm)
    rom.sync()
    dist.barrier()
    torch.cuda.synchronize()
    l0 = int(rom.lib.hrom_launch_count(rom.h))
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        rom.step(comm)
    ev1.record()
    ev1.synchronize()
    rom.sync()
    launches = int(rom.lib.hrom_launch_count(rom.h)) - l0
    (ms_step,) = reduce_max_over_ranks([ev0.elapsed_time(ev1) / args.steps], dist if world > 1 else None, "cuda")
    out = None
    if rank == 0:
        out = {"metric": METRIC, "value": wl.N / (ms_step / 1000.0), "unit": "cell-updates/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded config-4 blasts, BASELINE.json configs[3]; DESIGN.md §3)",
               "config": {"workload": wl.name, "grid": f"{wl.nx}x{wl.ny}", "cells": wl.N, "window_w": wl.w,
                          "rank_r": wl.r, "sample_fraction": wl.f,
                          "parallelism": f"row slabs x{world} (halo {int(rom.info.halo)} rows, {int(rom.info.rows_own)} own rows on rank 0)",
                          "l2": "inputs larger than L2"},
               "gpu_launches": launches}
    rom.close()
    dist.barrier()
    dist.destroy_process_group()
    return out


def H_count(rom, wl):
    from paper_2301_01718_b200.hrom import cells_from_mask
    return int(cells_from_mask(wl, rom.mask()).sum())


def host_cpu():
    """The GPU box's host: logical CPUs and model name (the oracle runs on one of them)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"host_nproc": os.cpu_count(), "cpu_model": model}


def cpu_sample(steps: int = 1, side: int = 256):
    """The oracle (oracle/, untuned) on a bounded sample of the config-4 workload: a
    side x side periodic tile with the config-4 method parameters (w = 64, r = 32,
    f = 10 %, W = 3, MUSCL-Rusanov), window seeded by the shared generator, one hybrid
    step of Algorithm 1 per sample, single thread."""
    import numpy as np
    import oracle
    from paper_2301_01718_b200 import inputs
    wl = inputs.config(4, nx=side, ny=side)
    snaps = inputs.smooth_window(wl, wl.w + 1, seed=7, amp=0.03)
    rng = np.random.default_rng(7)
    S = (rng.random(wl.N) < wl.f).astype(np.uint8)
    times = []
    for _ in range(steps):
        R = oracle.Run(wl, snaps[0])
        R.set_window(wl.w + 1, snaps, S)
        t0 = time.perf_counter()
        R.step()
        t1 = time.perf_counter()
        times.append(t1 - t0)
    t = float(np.median(times))
    return {"value": wl.N / t, "unit": "cell-updates/s", "cores": 1, "kind": "oracle", **host_cpu(),
            "sample": f"one oracle hybrid step (H1-H12, incl. POD of the 65-column window) on a {side}x{side} periodic tile "
                      f"with config-4 parameters (w=64, r=32, f=10%), median of {steps}; per-cell work is size-independent",
            "seconds_per_step": t}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64,
                    help="timed hybrid steps; the default w = 64 spans one Gram re-base period (amortised in)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hrom", choices=["hrom", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--fraction", type=float, default=0.10)
    ap.add_argument("--gram-mode", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--shard", default="replicas", choices=["replicas", "slab"],
                    help="replicas: one independent problem per GPU (default, weak scaling); slab: one problem cut "
                         "into row slabs across the GPUs (strong scaling, DESIGN.md §6)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        if rank != 0:
            return
        # each timed step: one oracle hybrid step on a 128^2 tile (~1 s), so that the default
        # K = 64 run ends within a few minutes
        side = 128
        samples = []
        for _ in range(args.warmup):
            cpu_sample(1, side)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            samples.append(cpu_sample(1, side)["seconds_per_step"])
        ms = 1000.0 * sum(samples) / len(samples)
        value = side * side / (ms / 1000.0)
        base = {"value": value, "unit": "cell-updates/s", "cores": 1, "kind": "oracle", **host_cpu(),
                "sample": f"one oracle hybrid step on a {side}x{side} periodic tile with config-4 parameters per step"}
        print(json.dumps({"impl": "reference", "metric": METRIC, "value": value, "unit": "cell-updates/s",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic", "config": {"workload": "config4-blasts-2048",
                                                                     "sample": f"one oracle hybrid step on a {side}x{side} tile per step"},
                          "cpu_baseline": base,
                          "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0},
                          "wall_s": time.perf_counter() - t0}))
        return
    if args.shard == "slab":
        out = run_slab(args, rank, world, local_rank)
        if rank == 0 and out is not None:
            print(json.dumps(out))
        return
    out = run_hrom(args, rank, world, local_rank)
    if rank == 0 and out is not None:
        if world == 1 and not args.no_cpu:
            out["cpu_baseline"] = cpu_sample(3)  # ~13 s of single-thread oracle work
        print(json.dumps(out))


if __name__ == "__main__":
    main()
