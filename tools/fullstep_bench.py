"""Full HDM step (H1 + H2) time at a config's grid: mean of N steps with CUDA events.
python tools/fullstep_bench.py [config] [steps]   (HROM_LIB=<path> selects another build of libhrom)"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_01718_b200 import inputs  # noqa: E402
from paper_2301_01718_b200 import hrom as H  # noqa: E402

if os.environ.get("HROM_LIB"):
    H.LIB_PATH = os.environ["HROM_LIB"]
    H.load_library(H.LIB_PATH)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
wl = inputs.config(cfg)
rom = H.HybridROM(wl)
rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
for _ in range(3):
    rom.full_step()
rom.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    rom.full_step()
e1.record()
e1.synchronize()
rom.sync()
ms = e0.elapsed_time(e1) / n
print(json.dumps({"config": cfg, "lib": os.path.basename(H.LIB_PATH), "full_step_ms": ms,
                  "cell_updates_per_s": wl.N / (ms / 1e3)}))
