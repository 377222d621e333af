"""Small-grid Algorithm-1 run with config-4 window/rank (debug helper for compute-sanitizer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
wl = inputs.config(4, nx=n, ny=n)
rom = HybridROM(wl)
rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
for k in range(wl.w + 3):
    rom.step()
rom.sync()
print("ok", rom.k, rom.effective_rank())
