"""Hunt a rare eager-vs-graph (or eager-vs-eager) divergence without synchronising between steps:
every step's state / S-hat / indicator / y / eigenvalues are copied on the streams into device
buffers and compared after the run.  python tools/flake_probe.py [config] [runs] [mode]
mode: eg = eager vs graph (default), ee = eager vs eager, gg = graph vs graph"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_01718_b200 import inputs  # noqa: E402
from paper_2301_01718_b200 import hrom as H  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 20
mode = sys.argv[3] if len(sys.argv) > 3 else "eg"
wl = inputs.config(cfg)
steps = wl.w + 2 * (wl.w + 2) + 7
q0 = torch.from_numpy(inputs.initial_condition(wl)).cuda()


def grab(rom):
    y = torch.zeros(wl.r, dtype=torch.float64, device="cuda")
    rom.lib.hrom_get_y(rom.h, y.data_ptr())
    out = [rom.get_state().clone(), rom.mask().clone(), rom.indicator().clone(), y]
    if os.environ.get("PROBE_JOIN") == "1":  # also the eigenvalues: joins the side-stream eigen-solve every step
        lam = torch.zeros(wl.w, dtype=torch.float64, device="cuda")
        rom.lib.hrom_get_eigen(rom.h, lam.data_ptr())
        out.append(lam)
        for which, n in ((0, 130 * 130), (1, 130 * 130), (2, 2 * 130 * 130), (3, wl.w * wl.w), (4, wl.w * wl.r)):
            t = torch.zeros(n, dtype=torch.float64, device="cuda")
            rom.lib.hrom_debug_read(rom.h, which, t.data_ptr(), n)
            out.append(t)
    return out


bad = 0
for run in range(runs):
    a, b = H.HybridROM(wl), H.HybridROM(wl)
    if mode[0] == "g":
        a.set_graph(True)
    if mode[1] == "g":
        b.set_graph(True)
    a.set_state(q0)
    b.set_state(q0)
    ra, rb = [], []
    for k in range(1, steps + 1):
        a.step()
        b.step()
        ra.append(grab(a))
        rb.append(grab(b))
    a.sync()
    b.sync()
    first = None
    for k, (x, z) in enumerate(zip(ra, rb), start=1):
        eq = [torch.equal(p, q) for p, q in zip(x, z)]
        if not all(eq):
            first = (k, dict(zip(["state", "mask", "eps", "y", "lam", "C", "Clo", "Mdd", "Zf", "A"], eq)),
                     float((x[0] - z[0]).abs().max()), float((x[3] - z[3]).abs().max()))
            break
    if first:
        bad += 1
        print("run", run, "first difference at step", first, "graph launches", a.graph_launches(), b.graph_launches(), flush=True)
    a.close()
    b.close()
print(f"mode {mode} config {cfg}: {bad} of {runs} runs diverged")
