"""NEXT-4 measurement: Algorithm 1 with the paper's implicit HDM on its own presets (Sod's shock
tube P:737-767, the model implosion P:906-921), on the GPU through hrom_imp_*.

For each preset: the AROM trajectory (the preset's z, delta, w, m, n_p) and the full-HDM
trajectory (z = 1) side by side; per step the wall time of hrom_imp_step (the step synchronises
once per subiteration, so the host clock brackets the device work) and the paper's metrics:
e_k = sum|gamma_k - q_k| / sum|q_k|, e-bar, s-bar, s-bar* (P:715-727), p-bar
(P:728-731), J-bar and S = t_H / t_R (Eq. speedup).

python tools/next4_bench.py [sod|implosion|all] [steps] -> JSON on stdout
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_01718_b200 import inputs  # noqa: E402
from paper_2301_01718_b200 import hrom as H  # noqa: E402

PAPER = {"implosion": {"J_bar": 2.73, "p_bar_pct": 0.23, "s_bar_pct": 18.35, "s_star_pct": 4.07, "S": 4.52,
                       "source": "P:919-921 (laptop CPU, single core, P:890)"}}


def run(name, steps=None):
    wl = inputs.preset(name)
    steps = steps or wl.steps
    q0 = torch.from_numpy(inputs.initial_condition(wl)).cuda()
    rom = H.ImplicitROM(wl)
    hdm = H.ImplicitROM(inputs.preset(name, z=1))
    rom.set_state(q0)
    hdm.set_state(q0)
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    t_r, t_h, e, s, kinds, Js, pts, its = [], [], [], [], [], [], [], []
    for _ in range(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rom.step(cnt)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        hdm.step()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        kind, J, nit, prods, np_used = rom.stats()
        kinds.append(kind)
        Js.append(J)
        pts.append(np_used)
        its.append(nit)
        s.append(int(cnt.item()))
        t_r.append(t1 - t0)
        t_h.append(t2 - t1)
        g = rom.get_state()
        q = hdm.get_state()
        e.append(float((g - q).abs().sum() / q.abs().sum()))
    hyb = [i for i, k in enumerate(kinds) if k == 1]
    N = wl.N
    out = {
        "preset": wl.name, "steps": steps, "N": N, "w": wl.w, "m": wl.r, "z": wl.z, "delta": wl.delta,
        "n_p": wl.n_p, "dt": wl.dt,
        "e_bar": float(np.mean(e)), "e_last": e[-1],
        "s_bar_pct": 100.0 * float(np.mean(s)) / N,
        "s_star_pct": 100.0 * float(np.mean([s[i] for i in hyb])) / N if hyb else None,
        "p_bar_pct": 100.0 * float(np.mean([pts[i] for i in hyb])) / N if hyb else None,
        "J_bar": float(np.mean([Js[i] for i in hyb])) if hyb else None,
        "J_range": [int(min(Js[i] for i in hyb)), int(max(Js[i] for i in hyb))] if hyb else None,
        "hybrid_steps": len(hyb), "escalated": kinds.count(2), "full_steps": kinds.count(0),
        "newton_its_per_step": float(np.mean(its)),
        "t_R_ms": 1e3 * float(np.mean(t_r)), "t_H_ms": 1e3 * float(np.mean(t_h)),
        "t_hybrid_step_ms": 1e3 * float(np.mean([t_r[i] for i in hyb])) if hyb else None,
        "S": float(np.mean(t_h) / np.mean(t_r)),
        "paper": PAPER.get(name),
    }
    return out


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else None
    names = ["sod", "implosion"] if which == "all" else [which]
    res = [run(n, steps) for n in names]
    print(json.dumps({"gpu": torch.cuda.get_device_name(0), "results": res}, indent=1))


if __name__ == "__main__":
    main()
