"""Host-side cost of hrom_step (enqueue time, no sync) vs device time per step (CUDA events):
tells whether a config is launch(CPU)-bound.  python tools/host_probe.py [cfg]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
wl = inputs.config(cfg)
rom = HybridROM(wl)
rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
for _ in range(wl.w + 3):
    rom.step()
torch.cuda.synchronize()
K = 20
host = []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    t = time.perf_counter()
    rom.step()
    host.append(time.perf_counter() - t)
e1.record()
e1.synchronize()
print({"config": cfg, "host_enqueue_ms_per_step": 1e3 * sum(host) / K, "device_ms_per_step": e0.elapsed_time(e1) / K,
       "launches_per_step": None})
