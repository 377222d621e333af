"""Two contexts (eager/eager or eager/graph) in lock step, compared every `every` steps (debug)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200 import hrom as H
cfg, graph, every = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
wl = inputs.config(cfg)
q0 = torch.from_numpy(inputs.initial_condition(wl)).cuda()
a = H.HybridROM(wl); b = H.HybridROM(wl)
if graph:
    b.set_graph(True)
a.set_state(q0); b.set_state(q0)
steps = wl.w + 2 * (wl.w + 2) + 7
for k in range(1, steps + 1):
    a.step(); b.step()
    if k % every == 0 or k == steps:
        same = torch.equal(a.get_state(), b.get_state()) and torch.equal(a.mask(), b.mask())
        if not same:
            print(f"cfg {cfg} graph {graph} every {every}: differ at k={k}")
            break
else:
    print(f"cfg {cfg} graph {graph} every {every}: identical through k={steps}")
