"""Phase timings (kcycles) of the one-CTA eigen-solve of the basis update (eig.cuh): [0]
tridiagonalisation, [1] Sturm multisection, [2] inverse iteration, [3] CGS2, [4] back-transform,
after a few config-4 steps (debug counters 10..14)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_01718_b200 import inputs  # noqa: E402
from paper_2301_01718_b200 import hrom as H  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
wl = inputs.config(cfg)
rom = H.HybridROM(wl)
rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
for _ in range(wl.w + 3):
    rom.step()
rom.sync()
print("config", cfg, "eigen phases (kcycles):", rom.debug_counters(16)[10:15])
