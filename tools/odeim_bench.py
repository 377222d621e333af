"""Algorithm 1 with ODEIM points (NEXT-1) on config 4 (2048^2, w = 64, r = 32, f = 10 %) with
n_p = 2r = 64: mean step time over hybrid steps, and the ODEIM part alone (lift of Phi_{k+1} +
64 greedy points) timed with CUDA events.  python tools/odeim_bench.py [--steps 8]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--cfg", type=int, default=4)
args = ap.parse_args()
base = inputs.config(args.cfg)
wl = inputs.config(args.cfg, n_p=2 * base.r)
rom = HybridROM(wl)
rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
for _ in range(wl.w + 2):
    rom.step()
torch.cuda.synchronize()
ts = []
for _ in range(args.steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rom.step()
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
phi, _ = rom.basis()
phi = phi.contiguous()
torch.cuda.synchronize()
to = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rom.odeim(phi, wl.n_p)
    e1.record()
    e1.synchronize()
    to.append(e0.elapsed_time(e1))
print(json.dumps({"config": args.cfg, "n_p": wl.n_p, "r_eff": int(phi.shape[0]), "step_ms_mean": sum(ts) / len(ts),
                  "step_ms_all": ts, "odeim_points_ms": min(to)}))
