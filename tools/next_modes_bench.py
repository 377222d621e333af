"""Mean hybrid-step time of the NEXT modes against the default (fraction rule, seam band) on
configs 2 and 4: RRE-delta selection (delta = 0.99), ODEIM points (n_p = 2r,
P:282-290) and the whole-domain filter (W = -1).  CUDA events around hrom_step, steps
w+3 .. w+3+K after the full warm-up.  python tools/next_modes_bench.py [--configs 2,4] [--steps 8]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200.hrom import HybridROM


def run(cfg, steps, **kw):
    wl = inputs.config(cfg, **kw)
    rom = HybridROM(wl)
    rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
    for _ in range(wl.w + 3):
        rom.step()
    torch.cuda.synchronize()
    ts, cnt = [], torch.zeros(1, dtype=torch.int32, device="cuda")
    sizes = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rom.step(count_out=cnt)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
        sizes.append(int(cnt.item()))
    rom.sync()
    return {"ms_mean": sum(ts) / len(ts), "ms_min": min(ts), "s_hat_mean": sum(sizes) / len(sizes)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,4")
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--out", default="gpurun_out/next_modes.json")
    a = ap.parse_args()
    out = {}
    for cfg in [int(x) for x in a.configs.split(",")]:
        r = inputs.config(cfg).r
        modes = {"default": {}, "rre_delta_0.99": {"delta": 0.99}, "odeim_np_2r": {"n_p": 2 * r},
                 "whole_domain_filter": {"W": -1}}
        out[f"config{cfg}"] = {name: run(cfg, a.steps, **kw) for name, kw in modes.items()}
        print(json.dumps({f"config{cfg}": out[f"config{cfg}"]}), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
