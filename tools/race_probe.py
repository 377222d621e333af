"""Bitwise-determinism probe: config 4 (or a given config) run twice from the same IC, the states
compared after every step; prints the first step where the runs differ and where (variable, cells).
Repeats R times.  python tools/race_probe.py [config] [extra_steps] [repeats]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_01718_b200 import inputs  # noqa: E402
from paper_2301_01718_b200 import hrom as H  # noqa: E402


def pollute(seed, gb=24):
    """fill freed device memory with garbage (RACE_POLLUTE=1): a context allocated afterwards gets
    memory whose previous contents differ from run to run"""
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    x = torch.empty(int(gb * 2 ** 30 / 8), dtype=torch.float64, device="cuda")
    x.uniform_(-1e3, 1e3, generator=g)
    del x
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def run(wl, q0, steps, every=True, seed=0):
    """every = False: no reads between steps (the overlap of a free-running trajectory), only the
    final state is kept"""
    if os.environ.get("RACE_POLLUTE") == "1":
        pollute(seed)
    rom = H.HybridROM(wl)
    rom.set_state(q0)
    out = []
    for k in range(steps):
        rom.step()
        if every or k == steps - 1:
            out.append((rom.get_state().clone(), rom.mask().clone(), rom.indicator().clone()))
    rom.sync()
    rom.close()
    return out


def main():
    if os.environ.get("HROM_LIB"):
        H.load_library(os.environ["HROM_LIB"])
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    extra = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    wl = inputs.config(cfg)
    q0 = torch.from_numpy(inputs.initial_condition(wl)).cuda()
    steps = wl.w + extra
    every = os.environ.get("RACE_EVERY", "0") == "1"
    ref = run(wl, q0, steps, every)
    bad = 0
    for rep in range(reps):
        cur = run(wl, q0, steps, every, seed=rep + 1)
        for k, ((a, ma, ea), (b, mb, eb)) in enumerate(zip(ref, cur)):
            same = torch.equal(a, b) and torch.equal(ma, mb) and torch.equal(ea, eb)
            if not same:
                bad += 1
                d = (a != b).reshape(wl.c, -1)
                cells = torch.nonzero(d.any(0)).flatten()
                print(f"rep {rep}: first difference after step {k + 1} (w = {wl.w}): state cells {cells.numel()} "
                      f"(first {cells[:8].tolist()}), mask equal {torch.equal(ma, mb)}, eps equal {torch.equal(ea, eb)}, "
                      f"max |diff| {float((a - b).abs().max()):.3e}")
                break
        else:
            print(f"rep {rep}: identical over {steps} steps")
    print("mismatching repetitions", bad, "of", reps)


if __name__ == "__main__":
    main()
