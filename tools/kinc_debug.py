"""Lock-step gather_mode 0 (incremental) vs 1 (full) contexts: first divergence."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = inputs.config(cfg)
q0 = torch.from_numpy(inputs.initial_condition(wl)).cuda()
a = HybridROM(wl, gather_mode=0); b = HybridROM(wl, gather_mode=1)
a.set_state(q0); b.set_state(q0)
for k in range(1, wl.w + 12):
    a.step(); b.step()
    ga, gb = a.get_state(), b.get_state()
    d = (torch.linalg.norm(ga - gb) / torch.linalg.norm(gb)).item()
    ca = a.debug_counters(24)
    print(f"k={k} rel={d:.2e} |S|={ca[16]} add={ca[22]} rem={ca[23]} y_a={a.y()[:3].tolist()} y_b={b.y()[:3].tolist()}", flush=True)
