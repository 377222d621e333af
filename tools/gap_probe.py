"""Spectral-gap probe of the POD window on a config (default: the bench workload, config 4,
f = 10 %): for each hybrid step after the bootstrap, the eigenvalues of the window Gram give
kappa = eps * lambda_1 / (lambda_reff - lambda_{reff+1}) (the fp64-Gram subspace error bound,
DESIGN.md G11) and the smallest relative gap among the retained modes.

python tools/gap_probe.py [config] [steps_after_bootstrap] -> JSON on stdout"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2301_01718_b200 import inputs
    from paper_2301_01718_b200.hrom import HybridROM
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    nst = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    wl = inputs.config(cfg, f=0.1) if cfg == 4 else inputs.config(cfg)
    rom = HybridROM(wl)
    rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
    for _ in range(wl.w - 1):
        rom.step()
    eps = np.finfo(np.float64).eps
    rows = []
    for s in range(nst):
        rom.step()
        rom.sync()
        lam = np.sort(rom.eigenvalues().cpu().numpy())[::-1]
        r = rom.effective_rank()
        l1 = lam[0]
        tail = lam[r] if r < len(lam) else 0.0
        gap_r = lam[r - 1] - tail
        gaps = [lam[i] - lam[i + 1] for i in range(r - 1)]
        rows.append({"k": rom.k, "reff": int(r), "lam1": float(l1), "lam_r": float(lam[r - 1]),
                     "kappa_subspace": float(eps * l1 / max(gap_r, 1e-300)),
                     "min_rel_gap_retained": float(min(gaps) / l1) if gaps else None})
    print(json.dumps({"config": cfg, "rows": rows,
                      "kappa_max": max(x["kappa_subspace"] for x in rows)}, indent=1))


if __name__ == "__main__":
    main()
