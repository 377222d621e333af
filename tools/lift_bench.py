"""Lift Phi = X V_r Lambda_r^{-1/2} (hrom_get_basis, DMMA) on config 4 (D = 16.8 M, w = 64,
r_eff): best-of-3 CUDA-event time and TF/s.  python tools/lift_bench.py [cfg]"""
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
rom.basis()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    phi, _ = rom.basis()
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = min(ts)
r = phi.shape[0]
fl = 2.0 * wl.D * wl.w * r
print(json.dumps({"config": cfg, "r_eff": r, "ms": ms, "tflops": fl / ms / 1e9, "GBs": 8 * wl.D * (wl.w + 2 + r) / ms / 1e6}))
