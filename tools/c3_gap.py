"""Conditioning of POD_r for the full-size config-3 replay window: eigenvalues
around r_eff and the subspace bound eps * lambda_1 / gap used by test_replay_config3_fullsize."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as orc
from paper_2301_01718_b200 import inputs
wl = inputs.config(3)
q = inputs.initial_condition(wl)
snaps = [q]
for _ in range(wl.w):
    snaps.append(orc.full_step(wl, snaps[-1], orc.dt(wl, snaps[-1])))
snaps = np.stack(snaps)
S = (np.random.default_rng(33).random(wl.N) < wl.f).astype(np.uint8)
R = orc.Run(wl, snaps[0]); R.set_window(wl.w, snaps, S)
sig = R.sigma(); lam = sig**2
r = wl.r
print("reff", R.reff(), "lam1", lam[0], "lam r-1..r+1", lam[r-2:r+2], "gap ratio", lam[0]/(lam[r-1]-lam[r]))
print("predicted subspace sine", 2.2e-16*lam[0]/(lam[r-1]-lam[r]))
