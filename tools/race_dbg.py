import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM
wl = inputs.config(1)
q0 = torch.from_numpy(inputs.initial_condition(wl)).cuda()
def run(nsteps, prof, events):
    rom = HybridROM(wl)
    rom.set_state(q0)
    for k in range(1, nsteps + 1):
        if prof: rom.profile(True)
        if events:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True); e0.record()
        rom.step()
        if events:
            e1.record(); e1.synchronize()
        if prof: rom.profile_read()
    try:
        rom.sync(); ok = True
    except Exception as e:
        ok = str(e)
    g = rom.get_state().cpu().numpy()
    rom.close()
    return ok, float(g[0].min())
for prof in (False, True):
    for events in (False, True):
        print("prof", prof, "events", events, run(200, prof, events), flush=True)
