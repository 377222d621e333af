"""Per-config measurements of SURVEY.md §8(d) D.1 (reported in DESIGN.md §8; not the driver's
bench line, which is bench.py on config 4 at f = 10 %).

python tools/bench_configs.py [--configs 1,2,3,4,5] [--out profiles/r1_configs.json]

  1-3  whole Algorithm-1 runs (full warm-up + hybrid steps), mean hybrid / full step time
  4    f in {5, 10, 15, 20} % (incremental Gram) and f = 10 % with the full DMMA Gram every step
  5    4096^2 x 4 vars, window of 129 smooth columns streamed into the ring: SᵀS Gram (DMMA) +
       128 x 128 eigen (rebuild_basis), lift to r = 64, and per f in {2, 5, 10, 20} %: gappy
       gather/normal equations, solve, fill of a held-out column, seam filter.
All times are CUDA-event times on the context stream (hrom_profile sections or explicit events).
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM, mask_from_cells


def _sec(d, name):
    v = d.get(name)
    return (v[0] / v[1]) if v and v[1] else None


def _peak():
    import bench
    return bench.measured_peaks()[0]


def _roofline(wl, fill_ms, step_ms):
    """north_star's per-config GB/s and roofline fraction: the fill pass's algorithmic bytes
    (bench.fill_bytes) over its mean launch time against the measured HBM
    copy bandwidth, and the same bytes over the whole step (the step's HBM floor is the fill)."""
    import bench
    n_s = int(np.ceil(wl.f * wl.N))
    fb = bench.fill_bytes(wl, n_s)
    peak = _peak()
    return {"fill_ms_mean": fill_ms, "fill_algorithmic_bytes": fb, "fill_GBs": fb / (fill_ms / 1e3) / 1e9,
            "fill_frac_of_hbm_peak": fb / (fill_ms / 1e3) / 1e9 / peak, "step_GBs": fb / (step_ms / 1e3) / 1e9,
            "step_frac_of_hbm_peak": fb / (step_ms / 1e3) / 1e9 / peak, "hbm_peak_GBs": peak}


def run_trajectory(cfg, steps=None, f=None):
    wl = inputs.config(cfg, **({"f": f} if f else {}))
    if steps:
        wl = inputs.config(cfg, steps=steps, **({"f": f} if f else {}))
    rom = HybridROM(wl)
    rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
    full_ms, hyb_ms, fill_ms = [], [], []
    t0 = time.perf_counter()
    for k in range(1, wl.steps + 1):
        rom.profile(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rom.step()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        sec = rom.profile_read()
        if k >= wl.w and sec.get("fill_pass") and sec["fill_pass"][1]:
            fill_ms.append(sec["fill_pass"][0] / sec["fill_pass"][1])
        if os.environ.get("HROM_CFG_DEBUG"):
            rom.sync()
        (hyb_ms if k >= wl.w else full_ms).append(ms)
    rom.sync()
    wall = time.perf_counter() - t0
    out = {"workload": wl.name, "grid": f"{wl.nx}x{wl.ny}", "steps": wl.steps, "w": wl.w, "r": wl.r, "f": wl.f,
           "full_step_ms_mean": float(np.mean(full_ms[1:])) if len(full_ms) > 1 else None,
           "hybrid_step_ms_mean": float(np.mean(hyb_ms[3:])) if len(hyb_ms) > 3 else None,
           "hybrid_step_ms_median": float(np.median(hyb_ms[3:])) if len(hyb_ms) > 3 else None,
           "hybrid_steps_w_to_w+99_ms_mean": float(np.mean(hyb_ms[:100])) if hyb_ms else None,
           "wall_s": wall}
    if out["hybrid_step_ms_mean"]:
        out["hybrid_cell_updates_per_s"] = wl.N / (out["hybrid_step_ms_mean"] / 1e3)
        if len(fill_ms) > 3:
            out["roofline"] = _roofline(wl, float(np.mean(fill_ms[3:])), out["hybrid_step_ms_mean"])
    rom.close()
    return out


def run_config4(f, gram_mode=0, steps=20, warmup=3):
    wl = inputs.config(4, f=f)
    rom = HybridROM(wl, gram_mode=gram_mode)
    rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
    for _ in range(wl.w - 1 + warmup):
        rom.step()
    rom.sync()
    rom.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        rom.step()
    e1.record()
    e1.synchronize()
    sec = rom.profile_read()
    rom.profile(False)
    ms = e0.elapsed_time(e1) / steps
    res = {"f": f, "gram_mode": "full-dmma" if gram_mode else "incremental-shifted", "ms_per_step": ms,
           "cell_updates_per_s": wl.N / (ms / 1e3),
           "sections_ms": {k: round(v[0] / steps, 4) for k, v in sec.items() if v[1]}}
    if sec.get("fill_pass") and sec["fill_pass"][1]:
        res["roofline"] = _roofline(wl, sec["fill_pass"][0] / sec["fill_pass"][1], ms)
    rom.close()
    return res


def smooth_column(nx, ny, j, gamma=1.4, seed=5, nmodes=32, dev="cuda"):
    """Config-5 column j (A30): primitive base + 32 Fourier modes (amplitude 2^{-i/4}) + two
    tanh fronts, converted to conservative; generated on the device with separable products."""
    g = torch.Generator(device="cpu").manual_seed(seed * 1000003 + j)
    x = (torch.arange(nx, dtype=torch.float64, device=dev) + 0.5) / nx
    y = (torch.arange(ny, dtype=torch.float64, device=dev) + 0.5) / ny
    prims = []
    base = (1.0, 0.0, 0.0, 1.0)
    for v in range(4):
        fld = torch.full((ny, nx), base[v], dtype=torch.float64, device=dev)
        kl = torch.randint(-8, 9, (nmodes, 2), generator=g)
        zeta = torch.rand(nmodes, generator=g) * 2 - 1
        phi = torch.rand(nmodes, 2, generator=g) * 2 * math.pi
        for i in range(nmodes):
            k, l = int(kl[i, 0]), int(kl[i, 1])
            if k == 0 and l == 0:
                k = 1
            a = 0.05 * 2.0 ** (-(i + 1) / 4.0) * float(zeta[i])
            cx = torch.cos(2 * math.pi * k * x + float(phi[i, 0]))
            sx = torch.sin(2 * math.pi * k * x + float(phi[i, 0]))
            cy = torch.cos(2 * math.pi * l * y + float(phi[i, 1]))
            sy = torch.sin(2 * math.pi * l * y + float(phi[i, 1]))
            fld += a * (torch.outer(cy, cx) - torch.outer(sy, sx))
        for q in range(2):
            ang = float(torch.rand(1, generator=g)) * 2 * math.pi
            s0 = 0.2 + 0.6 * float(torch.rand(1, generator=g))
            d = math.cos(ang) * x[None, :] + math.sin(ang) * y[:, None] - s0
            fld += 0.05 * torch.tanh(d / (4.0 / nx))
        prims.append(fld)
    rho = prims[0].clamp(min=0.3)
    p = prims[3].clamp(min=0.3)
    u, v = prims[1], prims[2]
    E = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v)
    return torch.stack([rho, rho * u, rho * v, E]).reshape(4, nx * ny).contiguous()


def run_config5(fracs=(0.02, 0.05, 0.10, 0.20), side=4096):
    wl = inputs.Workload("config5-stress", dim=2, nx=side, ny=side, bc=1, recon=2, cfl=0.4, w=128, r=64, f=0.1,
                         h=2, W=3, seed=5)
    rom = HybridROM(wl)
    res = {"workload": wl.name, "grid": f"{side}x{side}", "D": wl.D, "w": wl.w, "r": wl.r}
    k = wl.w
    t0 = time.perf_counter()
    for j in range(wl.w + 1):
        rom.put_snapshot(j, smooth_column(side, side, j))
    torch.cuda.synchronize()
    res["generate_window_s"] = time.perf_counter() - t0
    # Gram of the 129 window columns (full DMMA) + 128 x 128 eigen-solve
    rom.profile(True)
    rom.rebuild_basis(k)
    rom.sync()
    sec = rom.profile_read()
    res["gram_STS_ms"] = _sec(sec, "rebase_gram")
    res["eigen_ms"] = _sec(sec, "basis_eigen_side_stream")
    ncol = wl.w + 1
    flops = wl.D * ncol * (ncol + 1)  # symmetric count, FMA = 2
    if res["gram_STS_ms"]:
        res["gram_STS_tflops_symmetric"] = flops / (res["gram_STS_ms"] / 1e3) / 1e12
        res["gram_STS_bytes_GBs"] = 8 * wl.D * (ncol + 2) / (res["gram_STS_ms"] / 1e3) / 1e9
    res["r_eff"] = rom.effective_rank()
    res["log10_lambda"] = [round(math.log10(max(x, 1e-300)), 2) for x in rom.eigenvalues().cpu().numpy()[:80:4]]
    # lift Phi = X A (D x r_eff)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    phi, psi = rom.basis()
    e1.record()
    e1.synchronize()
    res["lift_ms"] = e0.elapsed_time(e1)
    res["lift_bytes_GBs"] = 8 * wl.D * (ncol + res["r_eff"] + 1) / (res["lift_ms"] / 1e3) / 1e9
    res["lift_tflops"] = 2.0 * wl.D * wl.w * res["r_eff"] / (res["lift_ms"] / 1e3) / 1e12
    # projection Phi^T S of the window (r_eff x (w+1)) on the FP64 tensor cores
    phi = phi.contiguous()
    pt = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rom.project(phi)
        e1.record()
        e1.synchronize()
        pt.append(e0.elapsed_time(e1))
    res["project_PhiTS_ms"] = min(pt)
    res["project_PhiTS_tflops"] = 2.0 * wl.D * res["r_eff"] * (wl.w + 1) / (res["project_PhiTS_ms"] / 1e3) / 1e12
    del phi, psi
    torch.cuda.empty_cache()
    # held-out column q* and its projection-error indicator (reconstruct with S-hat = all cells)
    qs = smooth_column(side, side, 10_000)
    allmask = mask_from_cells(wl, np.ones(wl.N, np.uint8))
    eps = torch.empty(wl.N, dtype=torch.float64, device="cuda")
    v = qs.clone()
    rom.reconstruct(v, mask=allmask, eps_out=eps)  # S-hat = all cells: per-cell projection error
    rom.sync()
    res["per_fraction"] = []
    for f in fracs:
        rom.sample(fraction=f, eps=eps)
        v = qs.clone()
        rom.profile(True)
        rom.reconstruct(v)
        rom.sync()
        sec = rom.profile_read()
        F = qs
        vf = v.clone()
        rom.filter(vf, F)
        rom.sync()
        sec2 = rom.profile_read()
        rom.profile(False)
        res["per_fraction"].append({"f": f, "gather_normal_eq_ms": _sec(sec, "gathered_gram"),
                                    "solve_ms": _sec(sec, "pinv_solve"), "fill_ms": _sec(sec, "fill_pass"),
                                    "seam_filter_ms": _sec(sec2, "seam_filter"),
                                    "fill_GBs": 8 * wl.D * (ncol + 2) / (_sec(sec, "fill_pass") / 1e3) / 1e9})
    rom.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--out", default="gpurun_out/configs.json")
    args = ap.parse_args()
    which = [int(x) for x in args.configs.split(",")]
    out = {"device": torch.cuda.get_device_name(0)}
    for cfg in which:
        t0 = time.perf_counter()
        if cfg in (1, 2, 3):
            out[f"config{cfg}"] = run_trajectory(cfg)
        elif cfg == 4:
            out["config4"] = [run_config4(f) for f in (0.05, 0.10, 0.15, 0.20)] + [run_config4(0.10, gram_mode=1)]
        elif cfg == 5:
            out["config5"] = run_config5()
        print(f"config {cfg} done in {time.perf_counter() - t0:.1f} s", flush=True)
        os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
        json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
