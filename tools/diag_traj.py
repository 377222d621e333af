"""Lock-step GPU vs oracle diagnostic of an Algorithm-1 trajectory (debug tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200 import hrom as H

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
wl = inputs.config(cfg, steps=steps)
q0 = inputs.initial_condition(wl)
rom = H.HybridROM(wl)
rom.set_state(torch.from_numpy(q0).cuda())
R = oracle.Run(wl, q0)
for k in range(1, steps + 1):
    rom.step(); kind = R.step()
    g = rom.get_state().cpu().numpy(); o = R.state()
    rel = np.linalg.norm(g - o) / np.linalg.norm(o)
    line = f"k={k} kind={kind} rel={rel:.2e}"
    if k >= wl.w - 1:
        eg = rom.indicator().cpu().numpy(); eo = R.eps()
        mg = H.cells_from_mask(wl, rom.mask()); mo = R.mask()
        nzg, nzo = (eg > 0).sum(), (eo > 0).sum()
        both = (eg > 0) & (eo > 0)
        erel = np.max(np.abs(eg[both] - eo[both]) / eo[both]) if both.any() else 0
        line += f" nz={nzg}/{nzo} nzdiff={(np.logical_xor(eg>0, eo>0)).sum()} epsrel={erel:.2e} maskdiff={(mg != mo).sum()} reff={rom.effective_rank()}/{R.reff()}"
        lam = rom.eigenvalues().cpu().numpy(); sig = R.sigma()
        line += f" lam0rel={abs(lam[0]-sig[0]**2)/sig[0]**2:.1e}"
        kept, sw = R.filter_stats()
        line += f" okept={kept} osw={sw}"
    print(line, flush=True)
