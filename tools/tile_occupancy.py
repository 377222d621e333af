"""Active-tile statistics of the masked RK3 sets (config 4) after a few hybrid steps."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from scipy import ndimage
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM, cells_from_mask
wl = inputs.config(4)
rom = HybridROM(wl)
rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
for _ in range(wl.w - 1 + 25):
    rom.step()
S = cells_from_mask(wl, rom.mask()).reshape(wl.ny, wl.nx).astype(bool)
sq = np.ones((2 * wl.W + 1, 2 * wl.W + 1), bool)
T = ndimage.binary_dilation(S, structure=sq, mode="wrap") if False else S.copy()
T = S | ndimage.binary_dilation(S, structure=sq)
cross = ndimage.generate_binary_structure(2, 1)
def crossdil(M, h):
    out = M.copy()
    for a in range(1, h + 1):
        out |= np.roll(M, a, 0) | np.roll(M, -a, 0) | np.roll(M, a, 1) | np.roll(M, -a, 1)
    return out
A2 = crossdil(T, wl.h); A1 = crossdil(A2, wl.h)
for name, M in (("S", S), ("T", T), ("A2", A2), ("A1", A1)):
    for ty, tx in ((8, 32), (16, 16), (4, 32)):
        t = M.reshape(wl.ny // ty, ty, wl.nx // tx, tx).any(axis=(1, 3))
        print(f"{name}: cells {M.sum()} ({M.mean():.3f}) tiles {ty}x{tx}: {t.sum()} of {t.size} -> work inflation {t.sum()*ty*tx/M.sum():.2f}")
