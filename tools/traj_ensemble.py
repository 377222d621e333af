"""GPU trajectory drift vs the oracle's own sensitivity (ensemble of 1e-15-perturbed ICs)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200 import hrom as H

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nens = int(sys.argv[2]) if len(sys.argv) > 2 else 4
wl = inputs.config(cfg)
q0 = inputs.initial_condition(wl)
rom = H.HybridROM(wl)
rom.set_state(torch.from_numpy(q0).cuda())
R = oracle.Run(wl, q0)
ens = []
for s in range(nens):
    rng = np.random.default_rng(s)
    ens.append(oracle.Run(wl, q0 * (1.0 + 1e-15 * rng.standard_normal(q0.shape))))
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
for k in range(1, wl.steps + 1):
    rom.step(); R.step()
    for E in ens:
        E.step()
    o = R.state()
    g = rom.get_state().cpu().numpy()
    mo = R.mask()
    fg = int(k >= wl.w - 1 and not np.array_equal(H.cells_from_mask(wl, rom.mask()), mo))
    fe = [int(k >= wl.w - 1 and not np.array_equal(E.mask(), mo)) for E in ens]
    print(f"k={k} gpu={rel(g, o):.2e} flip={fg} ens=" + " ".join(f"{rel(E.state(), o):.2e}/{f}" for E, f in zip(ens, fe)), flush=True)
