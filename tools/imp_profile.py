"""Per-kernel breakdown of NEXT-4 hybrid steps (run under ncu --metrics gpu__time_duration.sum):
the implosion preset to step w + 8, then 7 timed steps (one full, six hybrid) marked by an NVTX range."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_01718_b200 import inputs  # noqa: E402
from paper_2301_01718_b200 import hrom as H  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "implosion"
wl = inputs.preset(name)
rom = H.ImplicitROM(wl)
rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
for _ in range(wl.w + 8):
    rom.step()
torch.cuda.synchronize()
rom.debug_timers()
torch.cuda.nvtx.range_push("timed")
t0 = time.perf_counter()
stats = []
for _ in range(7):
    rom.step()
    stats.append(rom.stats())
torch.cuda.synchronize()
t1 = time.perf_counter()
torch.cuda.nvtx.range_pop()
print("wall ms/step", 1e3 * (t1 - t0) / 7, stats)
tm = rom.debug_timers()
ghz = 1.965
print("Newton per step (ms): products %.3f  GS %.3f  norms+Givens %.3f  line search %.3f  kernels %.3f;  products %d  solves %d"
      % tuple([x / 7 / ghz / 1e6 for x in tm[:5]] + [tm[5] / 7, tm[6] / 7]))
print("per product (us): own face task %.2f, wait for the slowest task + barrier %.2f"
      % (tm[7] / max(tm[5], 1) / ghz / 1e3, tm[8] / max(tm[5], 1) / ghz / 1e3))
