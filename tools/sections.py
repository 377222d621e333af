"""Mean per-section times (ms/step, hrom_profile CUDA events) of the hybrid steps of a config.
python tools/sections.py <config> [hybrid steps] [skip]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_01718_b200 import inputs  # noqa: E402
from paper_2301_01718_b200.hrom import HybridROM  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 3
wl = inputs.config(cfg)
rom = HybridROM(wl)
rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
for _ in range(wl.w - 1 + skip):
    rom.step()
rom.sync()
rom.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    rom.step()
rom.join()
e1.record()
e1.synchronize()
rom.sync()
sec = rom.profile_read()
cnt = rom.debug_counters(8)
print(json.dumps({"config": cfg, "steps": n, "ms_per_step": e0.elapsed_time(e1) / n,
                  "sections_ms": {k: round(v[0] / n, 4) for k, v in sec.items() if v[1]},
                  "last_filter_sweeps": cnt[4:7]}))
