import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM
wl = inputs.config(1)
for prof in (False, True):
    rom = HybridROM(wl)
    rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
    bad = None
    for k in range(1, wl.steps + 1):
        if prof: rom.profile(True)
        rom.step()
        if prof: rom.profile_read()
        try:
            rom.sync()
        except Exception as e:
            bad = (k, str(e)); break
    g = rom.get_state().cpu().numpy()
    print("prof", prof, "first failure", bad, "min rho", g[0].min())
    rom.close()
