"""First step where a graph-mode context departs from an eager one (debug)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200 import hrom as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = inputs.config(cfg)
q0 = torch.from_numpy(inputs.initial_condition(wl)).cuda()
a = H.HybridROM(wl); b = H.HybridROM(wl)
b.set_graph(True)
a.set_state(q0); b.set_state(q0)
for k in range(1, wl.w + 3 * (wl.w + 2)):
    a.step(); b.step()
    sa, sb = a.get_state(), b.get_state()
    ma, mb = a.mask(), b.mask()
    ea, eb = a.indicator(), b.indicator()
    if not (torch.equal(sa, sb) and torch.equal(ma, mb) and torch.equal(ea, eb)):
        print("first difference at k", k, "state", torch.equal(sa, sb), "mask", torch.equal(ma, mb), "eps", torch.equal(ea, eb),
              "graph launches", b.graph_launches(), "max state diff", (sa - sb).abs().max().item())
        break
else:
    print("no difference", b.graph_launches())
