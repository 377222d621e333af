"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
config 1 or 2 (BJ:7-8) through Algorithm 1 for w + 6 steps -- full warm-up steps, bootstrap,
hybrid steps with the masked RK3, gathered Gram (full and incremental), solve, fill, seam filter,
sampling, basis update and eigen refinement -- plus the standalone calls (reconstruct, filter,
RRE sampling, ODEIM points, projection, Gram).

compute-sanitizer --tool racecheck python tools/sanitize_run.py 2
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_01718_b200 import inputs  # noqa: E402
from paper_2301_01718_b200 import hrom as H  # noqa: E402


def implicit(name, extra):
    """NEXT-4: Algorithm 1 with the implicit HDM (Newton-Krylov, partial HDM subiterations,
    implicit-residual filter) on a preset, plus the standalone residual / Newton calls."""
    wl = inputs.preset(name)
    q0 = torch.from_numpy(inputs.initial_condition(wl)).cuda()
    rom = H.ImplicitROM(wl)
    rom.set_state(q0)
    for _ in range(wl.w + extra):
        rom.step()
    rom.sync()
    q = rom.get_state()
    rom.residual(q, q0, q0)
    qq = q.clone()
    rom.newton(qq, q, q, order=2, mask=rom.mask())
    rom.sync()
    print("ok", name, rom.stats())


def main():
    if len(sys.argv) > 1 and sys.argv[1] in ("sod", "implosion"):
        implicit(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 4)
        return
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    extra = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    wl = inputs.config(cfg)
    q0 = torch.from_numpy(inputs.initial_condition(wl)).cuda()
    rom = H.HybridROM(wl)
    rom.set_state(q0)
    for _ in range(wl.w + extra):
        rom.step()
    rom.sync()
    # standalone calls of the ABI on the current basis / sets
    v = rom.get_state().clone()
    rom.reconstruct(v)
    rom.filter(v, rom.get_state())
    rom.sample_rre(0.99)
    phi, _ = rom.basis()
    rom.odeim(phi.contiguous(), min(2 * phi.shape[0], 32))
    rom.project(phi.contiguous())
    rom.gram(torch.stack([q0.reshape(-1), v.reshape(-1)]))
    rom.sync()
    # ODEIM mode and the whole-domain filter for a few steps
    import dataclasses
    for kw in (dict(n_p=2 * wl.r), dict(W=-1)):
        r2 = H.HybridROM(dataclasses.replace(wl, **kw))
        r2.set_state(q0)
        for _ in range(wl.w + 3):
            r2.step()
        r2.sync()
        r2.close()
    print("sanitize run ok", cfg, rom.k)


if __name__ == "__main__":
    main()
