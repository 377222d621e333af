"""How much of S-hat changes from one hybrid step to the next (config 4)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM, cells_from_mask
wl = inputs.config(4)
rom = HybridROM(wl)
rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
for _ in range(wl.w - 1):
    rom.step()
prev = cells_from_mask(wl, rom.mask()).astype(bool)
for k in range(40):
    rom.step()
    cur = cells_from_mask(wl, rom.mask()).astype(bool)
    if k % 4 == 0:
        print(f"step {k}: |S|={cur.sum()} added {(cur & ~prev).sum()} removed {(prev & ~cur).sum()}", flush=True)
    prev = cur
