"""Steady-state hybrid-step throughput per config, eager launches vs CUDA-graph replay (G12):
w + warm-up steps untimed (graph mode: two ring periods so every phase is captured), then K
steps back to back timed with CUDA events on the context stream; the side-stream work of the
last step is joined inside the timed region.

python tools/config_throughput.py [--configs 1,2,3,4] [--steps 64] [--out profiles/r2_throughput.json]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_01718_b200 import inputs  # noqa: E402
from paper_2301_01718_b200.hrom import HybridROM  # noqa: E402


def measure(cfg, steps, graph):
    wl = inputs.config(cfg)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        rom = HybridROM(wl, stream=stream)
        if graph:
            rom.set_graph(True)
        rom.set_state(torch.from_numpy(inputs.initial_condition(wl)).cuda())
        warm = wl.w + 3 + (2 * (wl.w + 2) if graph else 0)
        for _ in range(warm):
            rom.step()
        rom.sync()
        g0 = rom.graph_launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            rom.step()
        rom.join()
        e1.record(stream)
        e1.synchronize()
        rom.sync()
        ms = e0.elapsed_time(e1) / steps
        out = {"config": cfg, "workload": wl.name, "cells": wl.N, "mode": "graph" if graph else "eager",
               "ms_per_step": ms, "cell_updates_per_s": wl.N / (ms / 1e3),
               "graph_steps": rom.graph_launches() - g0, "steps": steps}
        rom.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for cfg in [int(x) for x in args.configs.split(",")]:
        for graph in (False, True):
            rows.append(measure(cfg, args.steps, graph))
            print(json.dumps(rows[-1]), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
