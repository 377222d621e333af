"""Projection Phi^T S of the window (hrom_project, DMMA cross Gram) on config 4 (D = 16.8 M,
m = r_eff, w + 1 = 65 columns): best-of-3 CUDA-event time and TF/s vs the measured DMMA peak.
python tools/project_bench.py [cfg]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
wl = inputs.config(cfg)
rom = HybridROM(wl)
rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
for _ in range(wl.w + 1):
    rom.step()
phi, _ = rom.basis()
phi = phi.contiguous()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rom.project(phi)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = min(ts)
fl = 2.0 * wl.D * phi.shape[0] * (wl.w + 1)
print(json.dumps({"config": cfg, "m": int(phi.shape[0]), "ncol": wl.w + 1, "ms": ms, "tflops": fl / ms / 1e9,
                  "frac_dmma_peak": fl / ms / 1e9 / 37.107}))
