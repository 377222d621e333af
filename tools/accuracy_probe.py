"""Per-step GPU-vs-oracle errors of the replays in tests/test_gpu_accuracy.py, printed as JSON
(DESIGN.md §7 table): relative L2, per-element max error, the SVD-class bar, indicator error.

python tools/accuracy_probe.py [c3] [c4] [c4full]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as orc  # noqa: E402
from paper_2301_01718_b200 import inputs  # noqa: E402
import test_gpu_accuracy as T  # noqa: E402


def row(tag, rec):
    g, o = rec["g"], rec["o"]
    eg, eo = rec["eg"], rec["eo"]
    both = eo > 0
    return {"case": tag, "rel_l2": T.rel(g, o), "max_elem": T.maxerr(g, o), "bar": rec["bar"],
            "eps_rel": T.rel(eg, eo), "eps_max_elem": float(np.max(np.abs(eg - eo)) / np.max(eo)),
            "eps_support_flips": int(((eg > 0) ^ (eo > 0)).sum()),
            "eps_flip_max": float(np.max(np.maximum(eg, eo)[(eg > 0) ^ (eo > 0)], initial=0.0) / np.max(eo))}


def main():
    which = sys.argv[1:] or ["c3", "c4"]
    out = []
    t0 = time.time()
    if "c3" in which:
        wl, snaps = T.hdm_trajectory(orc, inputs, 3, inputs.config(3).w + 50)
        for ko in (0, 1, 50):
            S = (np.random.default_rng(33 + ko).random(wl.N) < wl.f).astype(np.uint8)
            out.append(row(f"config3 k=w+{ko}", T.replay(orc, inputs, wl, snaps, wl.w + ko, S)[0]))
            print(json.dumps(out[-1]), flush=True)
    if "c4" in which:
        wl, snaps = T.hdm_trajectory(orc, inputs, 4, inputs.config(4).w + 50, nx=512, ny=512)
        for ko in (0, 1, 50):
            S = (np.random.default_rng(44 + ko).random(wl.N) < wl.f).astype(np.uint8)
            for st, rec in enumerate(T.replay(orc, inputs, wl, snaps, wl.w + ko, S, steps=2)):
                out.append(row(f"config4-512 k=w+{ko} step {st + 1}", rec))
                print(json.dumps(out[-1]), flush=True)
    if "c4full" in which:
        wl = inputs.config(4)
        snaps = inputs.smooth_window(wl, wl.w + 1, seed=404, amp=0.03)
        S = (np.random.default_rng(404).random(wl.N) < wl.f).astype(np.uint8)
        out.append(row("config4 2048 smooth window", T.replay(orc, inputs, wl, snaps, wl.w + 3, S)[0]))
        print(json.dumps(out[-1]), flush=True)
    print(json.dumps({"rows": out, "seconds": time.time() - t0}))


if __name__ == "__main__":
    main()
