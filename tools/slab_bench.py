"""Row-slab sharding measured on ONE GPU at the bench workload (config 4, 2048^2):

  unsharded eager / CUDA-graph replay        -- the reference step times
  slab, 1 rank  (LocalComm)                   -- cost of the phase protocol itself (one context does all
                                                 the work, every exchange is a no-op copy)
  slab, 2 and 4 ranks on this one GPU         -- the ranks' kernels run one after the other, so the step
                                                 time is the SUM of the ranks' work + the exchanges: an
                                                 upper bound of per-rank work x ranks, not a scaling number
  slab, 1 rank through torch.distributed NCCL -- the DistComm transport (world size 1)

and the sharded state against the unsharded one after the same number of steps (full size).
python tools/slab_bench.py [--steps 20] [--config 4] [--nx 2048 --ny 2048] > gpurun_out/slab_bench.json
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_01718_b200 import inputs, slab  # noqa: E402
from paper_2301_01718_b200.hrom import HybridROM  # noqa: E402


def timed(fn, steps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warm", type=int, default=4)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--nx", type=int, default=0)
    ap.add_argument("--ny", type=int, default=0)
    ap.add_argument("--ranks", type=int, nargs="*", default=[1, 2, 4])
    a = ap.parse_args()
    over = {}
    if a.nx:
        over = {"nx": a.nx, "ny": a.ny or a.nx}
    wl = inputs.config(a.config, **over)
    q0 = torch.from_numpy(inputs.initial_condition(wl)).cuda()
    out = {"workload": wl.name, "grid": f"{wl.nx}x{wl.ny}", "w": wl.w, "r": wl.r, "f": wl.f, "steps": a.steps}
    nset = wl.w - 1 + a.warm

    def run_unsharded(graph):
        rom = HybridROM(wl)
        rom.set_state(q0)
        if graph:
            rom.set_graph(True)
        for _ in range(nset + (wl.w + 2 if graph else 0)):  # graph mode: one ring period of captures first
            rom.step()
        rom.sync()
        full = None
        ms = timed(rom.step, a.steps)
        rom.join()
        rom.sync()
        k = rom.k
        st = rom.get_state().clone()
        rom.close()
        return ms, k, st, full

    ms_e, k_e, st_e, _ = run_unsharded(False)
    out["unsharded_eager_ms"] = ms_e
    ms_g, k_g, _, _ = run_unsharded(True)
    out["unsharded_graph_ms"] = ms_g
    for P in a.ranks:
        roms = [slab.SlabROM(wl, r, P) for r in range(P)]
        comm = slab.LocalComm(P)
        for r in roms:
            r.set_state(q0)
        full_ms = timed(lambda: slab.step_all(roms, comm), wl.w - 2) if wl.w > 3 else None
        for _ in range(nset - (wl.w - 2)):
            slab.step_all(roms, comm)
        ms = timed(lambda: slab.step_all(roms, comm), a.steps)
        for r in roms:
            r.sync()
        assert roms[0].k == k_e
        b = slab.assemble(roms, "state")
        scale = st_e.abs().amax(dim=1, keepdim=True)
        err = float(((b - st_e).abs() / scale).max())
        out[f"slab_{P}ranks_one_gpu"] = {"hybrid_ms": ms, "full_step_ms": full_ms, "max_rel_err_vs_unsharded": err,
                                         "halo_rows": int(roms[0].info.halo), "rows_own": int(roms[0].info.rows_own),
                                         "max_message_bytes": int(roms[0].info.max_message_bytes)}
        for r in roms:
            r.close()
        del roms
        torch.cuda.empty_cache()
    # the NCCL transport with one rank
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("nccl", rank=0, world_size=1)
    rom = slab.SlabROM(wl, 0, 1)
    comm = slab.DistComm()
    rom.set_state(q0)
    for _ in range(nset):
        rom.step(comm)
    ms = timed(lambda: rom.step(comm), a.steps)
    rom.sync()
    b = rom.get_state()
    scale = st_e.abs().amax(dim=1, keepdim=True)
    out["slab_1rank_nccl"] = {"hybrid_ms": ms, "max_rel_err_vs_unsharded": float(((b - st_e).abs() / scale).max())}
    rom.close()
    dist.destroy_process_group()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
