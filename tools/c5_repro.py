import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM
side = int(sys.argv[1]) if len(sys.argv) > 1 else 256
wl = inputs.Workload("c5", dim=2, nx=side, ny=side, bc=1, recon=2, cfl=0.4, w=128, r=64, f=0.1, h=2, W=3, seed=5)
rom = HybridROM(wl)
cols = inputs.smooth_window(wl, wl.w + 1, seed=5)
for j in range(wl.w + 1):
    rom.put_snapshot(j, torch.from_numpy(cols[j]).cuda())
rom.rebuild_basis(wl.w)
rom.sync()
print("rebuild ok, reff", rom.effective_rank())
phi, psi = rom.basis()
torch.cuda.synchronize()
print("basis ok", phi.shape)
