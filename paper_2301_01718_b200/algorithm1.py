"""Algorithm 1 driver with the paper's accuracy and cost metrics.

Runs the adaptive model (hrom_step_ex: full HDM step when k+1 <= w or k mod z = 0, P:557;
refresh skipped before full steps) beside a full-HDM reference trajectory q_k
(a second context with z = 1, which is the HDM bitwise) and reports

  e_k  = sum |gamma_k - q_k| / sum |q_k|                       (uniform cells)
  e-bar = (1/N_t) sum_k e_k
  s-bar = (1/N_t) sum_k n_{gamma_k}, n = N (full) or |S-hat|
  s-bar* = the same mean over the hybrid steps only
  p-bar = mean ODEIM points (n_p)_k over the hybrid steps, from hrom_points_used:
          n_p in ODEIM mode (odeim_points > 0), 0 when S-hat = G (reading A11)
  S = t_H / t_R, the speed-up of Eq. (speedup), from CUDA-event times of the
      two trajectories' own steps on the shared stream.

Every number comes from the device path (libhrom); e_k is reduced on the device
(hrom_rel_l1_error).  Nothing here runs on the CPU beyond bookkeeping.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np
import torch

from . import inputs as _inputs
from .hrom import HybridROM


@dataclasses.dataclass
class Algorithm1Metrics:
    steps: int
    z: int
    e: list            # e_k, k = 1..N_t
    n_gamma: list      # n_{gamma_k}
    hybrid: list       # k has a partial HDM solve
    points: list       # (n_p)_k, ODEIM points used by step k
    t_R_ms: float      # mean adaptive step time
    t_H_ms: Optional[float]  # mean full-HDM step time (reference trajectory)

    @property
    def e_bar(self) -> float:
        return float(np.mean(self.e)) if self.e else 0.0

    @property
    def s_bar(self) -> float:
        return float(np.mean(self.n_gamma))

    @property
    def s_bar_star(self) -> Optional[float]:
        h = [n for n, hy in zip(self.n_gamma, self.hybrid) if hy]
        return float(np.mean(h)) if h else None

    @property
    def p_bar(self) -> float:
        h = [p for p, hy in zip(self.points, self.hybrid) if hy]
        return float(np.mean(h)) if h else 0.0

    @property
    def speedup(self) -> Optional[float]:
        return self.t_H_ms / self.t_R_ms if self.t_H_ms else None

    def summary(self) -> dict:
        return {"steps": self.steps, "z": self.z, "e_bar": self.e_bar, "e_last": self.e[-1] if self.e else None,
                "s_bar": self.s_bar, "s_bar_star": self.s_bar_star, "p_bar": self.p_bar,
                "t_R_ms": self.t_R_ms, "t_H_ms": self.t_H_ms, "S": self.speedup,
                "hybrid_steps": int(sum(self.hybrid))}


def run(wl, steps: Optional[int] = None, z: Optional[int] = None, reference: bool = True,
        q0: Optional[np.ndarray] = None) -> Algorithm1Metrics:
    """Algorithm 1 on workload wl for `steps` steps (default wl.steps) with period z (default wl.z)."""
    steps = wl.steps if steps is None else steps
    z = wl.z if z is None else z
    wl = dataclasses.replace(wl, z=z)
    q0 = _inputs.initial_condition(wl) if q0 is None else q0
    q0d = torch.from_numpy(np.ascontiguousarray(q0)).cuda()
    rom = HybridROM(wl)
    rom.set_state(q0d)
    ref = None
    if reference:
        ref = HybridROM(dataclasses.replace(wl, z=1))
        ref.set_state(q0d)
    counts = torch.zeros(steps, dtype=torch.int32, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t_r = t_h = 0.0
    es, hyb, pts = [], [], []
    ga = torch.empty((wl.c, wl.N), dtype=torch.float64, device="cuda")
    gb = torch.empty_like(ga)
    for k in range(1, steps + 1):
        ev[0].record()
        rom.step(count_out=counts[k - 1:k])
        ev[1].record()
        hyb.append(not (k + 1 <= wl.w or (z > 0 and k % z == 0)))
        pts.append(rom.points_used())
        if ref is not None:
            ev[2].record()
            ref.step()
            ev[3].record()
            rom.get_state(ga)
            ref.get_state(gb)
            es.append(rom.rel_l1_error(ga, gb))  # synchronises
            t_h += ev[2].elapsed_time(ev[3])
        else:
            ev[1].synchronize()
        t_r += ev[0].elapsed_time(ev[1])
    rom.sync()
    n_gamma = counts.cpu().tolist()
    out = Algorithm1Metrics(steps=steps, z=z, e=es, n_gamma=n_gamma, hybrid=hyb, points=pts, t_R_ms=t_r / steps,
                            t_H_ms=(t_h / steps) if ref is not None else None)
    rom.close()
    if ref is not None:
        ref.close()
    return out
