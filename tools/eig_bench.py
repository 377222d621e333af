"""Time the one-CTA eigen-solve of the basis update in isolation (set_window -> update_basis)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM
w = int(sys.argv[1]) if len(sys.argv) > 1 else 64
wl = inputs.config(4, nx=256, ny=256, w=w, r=min(32, w))
snaps = inputs.smooth_window(wl, wl.w + 1, seed=3, amp=0.03)
rom = HybridROM(wl)
S = torch.zeros(rom.mask_words, dtype=torch.int32, device="cuda")
for rep in range(3):
    rom.profile(True)
    rom.set_window(wl.w + 5, torch.from_numpy(snaps.reshape(wl.w + 1, -1)).cuda(), S)
    sec = rom.profile_read()
    print({k: round(v[0], 4) for k, v in sec.items() if v[1]}, "counters", rom.debug_counters(12))
