"""Seeded synthetic workloads shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the hybrid-snapshot method: it only draws
counter-based random numbers and lays out initial conditions (ICs) in the
exchange format (SoA, q[v*N + n], n = j*nx + i, v = rho, rho*u, [rho*v,] rho*E).
Both sides (oracle/ and the CUDA path) consume exactly these bits.

Workloads follow /root/repo/BASELINE.json ``configs`` (BJ:7-11) with the
readings recorded in DESIGN.md §3:

* A26  perturbation: each primitive (rho, u, v, p) * (1 + 1e-3 * xi),
       xi ~ U[-1, 1) i.i.d. per cell and variable (zero velocities stay 0).
* A27  config-2 quadrant order Q1 (x>=1/2, y>=1/2), Q2 (x<1/2, y>=1/2),
       Q3 (x<1/2, y<1/2), Q4 (x>=1/2, y<1/2), tested at cell centres.
* A28  config-3 random quadrant states rho~U[0.1,2], p~U[0.02,2], u,v~U[-1.3,1.3].
* A29  config-4 blasts: Pi~U[10,100], p_in=Pi, rho_in=Pi**(1/gamma),
       R~U[0.02,0.08], centres~U[0,1)^2, periodic minimum-image distance,
       overlaps take the largest Pi, u=v=0, background rho=p=1.

The random generator is SplitMix64 applied to a counter
(seed, stream, index) -> 64-bit word -> top 53 bits -> [0, 1).
The conversion primitive -> conservative, E = p/(gamma-1) + rho|u|^2/2, is
part of laying out the IC (the configs are stated in primitive variables,
BJ:7-10); it is not a step of the hot path.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Tuple

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_G1 = np.uint64(0x9E3779B97F4A7C15)
_G2 = np.uint64(0xBF58476D1CE4E5B9)
_G3 = np.uint64(0x94D049BB133111EB)

# named streams so that different draws never share counters
STREAM_PERTURB = 1
STREAM_QUADRANT = 2
STREAM_BLAST = 3
STREAM_FIELD = 4
STREAM_TEST = 5


def splitmix64(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Counter-based SplitMix64: word(seed, stream, idx) for an array of idx."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) * _G1 + np.uint64(stream) * _G2 + idx * _G3 + _G1) & _M64
        z = (z ^ (z >> np.uint64(30))) * _G2
        z = (z ^ (z >> np.uint64(27))) * _G3
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """U[0,1) doubles from the top 53 bits of the counter hash."""
    z = splitmix64(seed, stream, idx)
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def uniform(seed: int, stream: int, idx: np.ndarray, lo: float, hi: float) -> np.ndarray:
    return lo + (hi - lo) * uniform01(seed, stream, idx)


@dataclasses.dataclass
class Workload:
    """One synthetic workload: grid, IC and method parameters.

    Field names follow SURVEY.md §0.4: w = window (BASELINE "m"), r = POD rank
    (BASELINE "k"), f = HDM sample fraction, h = per-stage halo, W = seam band.
    """
    name: str
    dim: int
    nx: int
    ny: int
    x0: float = 0.0
    x1: float = 1.0
    y0: float = 0.0
    y1: float = 1.0
    bc: int = 0            # 0 transmissive, 1 periodic
    recon: int = 2         # 1 first-order, 2 MUSCL-minmod
    gamma: float = 1.4
    cfl: float = 0.4
    steps: int = 100
    w: int = 8
    r: int = 4
    f: float = 0.1
    h: int = 2
    W: int = 3
    seed: int = 0
    filter_orders: Tuple[int, ...] = (2, 4, 6)
    filter_max_sweeps: int = 10
    filter_eps: float = 1e-2
    eig_rel_cutoff: float = 1e-8
    lsq_rel_cutoff: float = 1e-12
    z: int = 0             # full-HDM period of Algorithm 1; 0 = infinity (A20)
    delta: float = 0.0     # > 0: RRE-delta selection instead of the fraction f
    n_p: int = 0           # > 0: ODEIM points added to S-hat; gappy rows = their DOF rows
    # NEXT-4, the paper's implicit HDM: BDF2 + MUSCL/Roe by Newton-Krylov with
    # partial-HDM subiterations; fixed time step dt
    hdm: str = "explicit"  # "explicit" (SSP-RK3, BASELINE configs) or "implicit"
    flux: int = 0          # 0 Rusanov (BASELINE, A2), 1 Roe
    dt: float = 0.0        # fixed step of the implicit HDM
    eps_y: float = 1e-4    # subiteration tolerance on ||y^(j+1) - y^(j)||_2
    j_max: int = 10        # maximum subiterations
    newton_tol: float = 1e-12   # Newton stop on ||R_k||_inf (reading A40)
    newton_maxit: int = 30

    @property
    def c(self) -> int:
        return self.dim + 2

    @property
    def N(self) -> int:
        return self.nx * self.ny

    @property
    def D(self) -> int:
        return self.c * self.N

    def cell_centres(self) -> Tuple[np.ndarray, np.ndarray]:
        dx = (self.x1 - self.x0) / self.nx
        dy = (self.y1 - self.y0) / self.ny
        xc = self.x0 + (np.arange(self.nx) + 0.5) * dx
        yc = self.y0 + (np.arange(self.ny) + 0.5) * dy
        X = np.broadcast_to(xc[None, :], (self.ny, self.nx)).reshape(-1)
        Y = np.broadcast_to(yc[:, None], (self.ny, self.nx)).reshape(-1)
        return X, Y


def primitive_to_conservative(dim: int, gamma: float, rho, u, v, p) -> np.ndarray:
    """Lay out an IC given in primitive variables as the SoA conservative array."""
    rho = np.asarray(rho, dtype=np.float64)
    N = rho.size
    c = dim + 2
    q = np.empty((c, N), dtype=np.float64)
    q[0] = rho
    q[1] = rho * u
    if dim == 2:
        q[2] = rho * v
        q[3] = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v)
    else:
        q[2] = p / (gamma - 1.0) + 0.5 * rho * (u * u)
    return q


def _perturb(seed: int, N: int, prims, amp: float = 1e-3):
    """A26: multiplicative (1 + amp*xi), xi ~ U[-1,1), per cell and variable."""
    out = []
    for k, a in enumerate(prims):
        idx = np.arange(N, dtype=np.uint64) * np.uint64(8) + np.uint64(k)
        xi = uniform(seed, STREAM_PERTURB, idx, -1.0, 1.0)
        out.append(a * (1.0 + amp * xi))
    return out


def config(idx: int, **overrides) -> Workload:
    """BASELINE.json configs 1..5 (BJ:7-11) with the DESIGN.md readings."""
    if idx == 1:
        wl = Workload("config1-sod1d-N1000", dim=1, nx=1000, ny=1, bc=0, recon=1,
                      cfl=0.5, steps=200, w=20, r=10, f=0.10, h=2, W=3, seed=1)
    elif idx == 2:
        wl = Workload("config2-quadrant-256", dim=2, nx=256, ny=256, bc=0, recon=2,
                      cfl=0.4, steps=500, w=32, r=16, f=0.15, h=2, W=3, seed=2)
    elif idx == 3:
        wl = Workload("config3-randquad-1024", dim=2, nx=1024, ny=1024, bc=0, recon=2,
                      cfl=0.4, steps=1000, w=48, r=24, f=0.10, h=2, W=3, seed=3)
    elif idx == 4:
        wl = Workload("config4-blasts-2048", dim=2, nx=2048, ny=2048, bc=1, recon=2,
                      cfl=0.4, steps=300, w=64, r=32, f=0.10, h=2, W=3, seed=4)
    elif idx == 5:
        wl = Workload("config5-stress-4096", dim=2, nx=4096, ny=4096, bc=1, recon=2,
                      cfl=0.4, steps=0, w=128, r=64, f=0.05, h=2, W=3, seed=5)
    else:
        raise ValueError(f"no config {idx}")
    return dataclasses.replace(wl, **overrides)


def preset(name: str, **overrides) -> Workload:
    """The paper's own experiments (NEXT-4): Sod's shock tube (N = 499, N_t = 999 on
    (0, 0.2), w = 5, m = 4, delta = 0.80, filters 2-4-6) and the model implosion (P:906-921:
    100 x 100 on (0, 0.3)^2, walls, N_t = 1650 on (0, 0.5), z = 7, delta = 0.90, w = 6, m = 4),
    implicit BDF2 + MUSCL/Roe HDM.  n_p (never printed by the paper): S:296 defaults 2m = 8
    for Sod and 23 for the implosion (p-bar = 0.23 % of 10 000 cells).  The filter acts on
    the whole hybrid state (W = -1, reading G9)."""
    if name == "sod":
        wl = Workload("next4-sod-499", dim=1, nx=499, ny=1, bc=0, recon=2, steps=999, w=5, r=4,
                      f=0.1, h=2, W=-1, delta=0.80, n_p=8, hdm="implicit", flux=1, dt=0.2 / 999)
    elif name == "implosion":
        wl = Workload("next4-implosion-100", dim=2, nx=100, ny=100, x1=0.3, y1=0.3, bc=2, recon=2,
                      steps=1650, w=6, r=4, f=0.1, h=2, W=-1, z=7, delta=0.90, n_p=23,
                      hdm="implicit", flux=1, dt=0.5 / 1650)
    else:
        raise ValueError(f"no preset {name}")
    return dataclasses.replace(wl, **overrides)


def initial_condition(wl: Workload, kind: Optional[str] = None) -> np.ndarray:
    """Seeded IC of a workload as SoA conservative (c, N) float64.

    kind selects the IC family; default by workload name prefix.
    """
    if kind is None:
        kind = {"config1": "sod", "config2": "quadrant", "config3": "randquad",
                "config4": "blasts", "config5": "blasts"}.get(wl.name.split("-")[0], "blasts")
        if wl.name.startswith("next4-sod"):
            kind = "sod_clean"
        elif wl.name.startswith("next4-implosion"):
            kind = "implosion"
    X, Y = wl.cell_centres()
    N = wl.N
    g = wl.gamma
    if kind in ("sod", "sod_clean"):
        left = X < 0.5
        rho = np.where(left, 1.0, 0.125)
        u = np.zeros(N)
        p = np.where(left, 1.0, 0.1)
        if kind == "sod":
            rho, u, p = _perturb(wl.seed, N, (rho, u, p))
        if wl.dim == 1:
            return primitive_to_conservative(1, g, rho, u, None, p)
        return primitive_to_conservative(2, g, rho, u, np.zeros(N), p)
    if kind in ("quadrant", "quadrant_clean", "randquad"):
        if kind == "randquad":
            k = np.arange(16, dtype=np.uint64)
            uu = uniform01(wl.seed, STREAM_QUADRANT, k).reshape(4, 4)
            states = np.empty((4, 4))
            states[:, 0] = 0.1 + 1.9 * uu[:, 0]
            states[:, 1] = -1.3 + 2.6 * uu[:, 1]
            states[:, 2] = -1.3 + 2.6 * uu[:, 2]
            states[:, 3] = 0.02 + 1.98 * uu[:, 3]
        else:
            states = np.array([[1.5, 0.0, 0.0, 1.5],
                               [0.5323, 1.206, 0.0, 0.3],
                               [0.138, 1.206, 1.206, 0.029],
                               [0.5323, 0.0, 1.206, 0.3]])
        xm = 0.5 * (wl.x0 + wl.x1)
        ym = 0.5 * (wl.y0 + wl.y1)
        q = np.where(X >= xm, np.where(Y >= ym, 0, 3), np.where(Y >= ym, 1, 2))
        rho, u, v, p = (states[q, i] for i in range(4))
        if kind != "quadrant_clean":
            rho, u, v, p = _perturb(wl.seed, N, (rho, u, v, p))
        return primitive_to_conservative(2, g, rho, u, v, p)
    if kind == "blasts":
        nb = 8
        k = np.arange(nb, dtype=np.uint64)
        Pi = uniform(wl.seed, STREAM_BLAST, k * np.uint64(4) + np.uint64(0), 10.0, 100.0)
        R = uniform(wl.seed, STREAM_BLAST, k * np.uint64(4) + np.uint64(1), 0.02, 0.08)
        cx = uniform01(wl.seed, STREAM_BLAST, k * np.uint64(4) + np.uint64(2))
        cy = uniform01(wl.seed, STREAM_BLAST, k * np.uint64(4) + np.uint64(3))
        Lx = wl.x1 - wl.x0
        Ly = wl.y1 - wl.y0
        best = np.zeros(N)
        for b in range(nb):
            ddx = np.abs(X - (wl.x0 + cx[b] * Lx))
            ddy = np.abs(Y - (wl.y0 + cy[b] * Ly))
            if wl.bc == 1:
                ddx = np.minimum(ddx, Lx - ddx)
                ddy = np.minimum(ddy, Ly - ddy)
            inside = np.sqrt(ddx * ddx + ddy * ddy) < R[b]
            best = np.where(inside, np.maximum(best, Pi[b]), best)
        p = np.where(best > 0, best, 1.0)
        rho = np.where(best > 0, best ** (1.0 / g), 1.0)
        zero = np.zeros(N)
        return primitive_to_conservative(2, g, rho, zero, zero, p)
    if kind == "implosion":
        # rho, p = 0.125, 0.14 inside D = {x_1 + x_2 <= 0.15}, 1, 1 outside, u = 0
        inside = (X + Y) <= 0.15
        rho = np.where(inside, 0.125, 1.0)
        p = np.where(inside, 0.14, 1.0)
        zero = np.zeros(N)
        return primitive_to_conservative(2, g, rho, zero, zero, p)
    if kind == "uniform":
        return primitive_to_conservative(wl.dim, g, np.full(N, 1.3), np.full(N, 0.4),
                                         np.full(N, -0.2), np.full(N, 2.1))
    if kind == "entropy_wave":
        # rho = 1 + 0.2 sin(2 pi (x + y)), u = 1 (v = 1 in 2D), p = 1: exact Euler solution
        arg = X if wl.dim == 1 else X + Y
        rho = 1.0 + 0.2 * np.sin(2.0 * np.pi * arg)
        return primitive_to_conservative(wl.dim, g, rho, np.ones(N),
                                         np.ones(N) if wl.dim == 2 else None, np.ones(N))
    if kind == "random":
        k = np.arange(N, dtype=np.uint64) * np.uint64(4)
        rho = uniform(wl.seed, STREAM_TEST, k, 0.5, 2.0)
        u = uniform(wl.seed, STREAM_TEST, k + np.uint64(1), -0.5, 0.5)
        v = uniform(wl.seed, STREAM_TEST, k + np.uint64(2), -0.5, 0.5)
        p = uniform(wl.seed, STREAM_TEST, k + np.uint64(3), 0.5, 2.0)
        return primitive_to_conservative(wl.dim, g, rho, u, v if wl.dim == 2 else None, p)
    raise ValueError(kind)


def random_matrix(seed: int, rows: int, cols: int, stream: int = STREAM_TEST,
                  lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Seeded dense test matrix (column-major semantics: returned as (rows, cols))."""
    idx = np.arange(rows * cols, dtype=np.uint64)
    return uniform(seed, stream, idx, lo, hi).reshape(cols, rows).T.copy()


def random_values(seed: int, n: int, lo: float = 0.0, hi: float = 1.0,
                  stream: int = STREAM_TEST, offset: int = 0) -> np.ndarray:
    idx = np.arange(n, dtype=np.uint64) + np.uint64(offset)
    return uniform(seed, stream, idx, lo, hi)


def smooth_window(wl: Workload, ncols: int, seed: Optional[int] = None,
                  nmodes: int = 32, amp: float = 0.05) -> np.ndarray:
    """Config-5-style snapshot columns (reading A30), also used to
    seed windows for replay tests: each column j is a smooth periodic field sum of
    ``nmodes`` Fourier modes with amplitudes a_i = 2^{-i/4} plus two tanh fronts,
    per primitive variable, converted to conservative.  Returns (ncols, c, N).
    """
    s = wl.seed if seed is None else seed
    X, Y = wl.cell_centres()
    N = wl.N
    c = wl.c
    out = np.empty((ncols, c, N))
    kk = np.arange(nmodes, dtype=np.uint64)
    kx = np.floor(uniform(s, STREAM_FIELD, kk * np.uint64(2), -8.0, 9.0))
    ky = np.floor(uniform(s, STREAM_FIELD, kk * np.uint64(2) + np.uint64(1), -8.0, 9.0))
    kx = np.where((kx == 0) & (ky == 0), 1.0, kx)
    if wl.dim == 1:
        ky = np.zeros_like(ky)
        kx = np.where(kx == 0, 1.0, kx)
    a = 2.0 ** (-(np.arange(nmodes) + 1) / 4.0)
    nv = 4 if wl.dim == 2 else 3
    base = [1.0, 0.0, 0.0, 1.0] if wl.dim == 2 else [1.0, 0.0, 1.0]
    ell = 4.0 / max(wl.nx, 1)
    for j in range(ncols):
        prims = []
        for v in range(nv):
            o = (j * nv + v) * nmodes
            zeta = uniform(s, STREAM_FIELD, np.uint64(1000 + 3 * o) + kk * np.uint64(3), -1.0, 1.0)
            phi = uniform(s, STREAM_FIELD, np.uint64(1001 + 3 * o) + kk * np.uint64(3), 0.0, 2 * math.pi)
            fld = np.full(N, base[v])
            for i in range(nmodes):
                fld += amp * a[i] * zeta[i] * np.cos(2 * math.pi * (kx[i] * X + ky[i] * Y) + phi[i])
            for qf in range(2):
                t = uniform(s, STREAM_FIELD, np.arange(3, dtype=np.uint64) + np.uint64(10_000_000 + 10 * (j * 2 + qf)), 0.0, 1.0)
                ang = 2 * math.pi * t[0]
                sh = 0.2 + 0.6 * t[1]
                fld += amp * 0.5 * np.tanh(((math.cos(ang) * X + math.sin(ang) * Y) - sh) / ell) * (1.0 if v != 1 else 0.5)
            prims.append(fld)
        if wl.dim == 2:
            rho, u, v_, p = prims
            rho = np.maximum(rho, 0.3)
            p = np.maximum(p, 0.3)
            out[j] = primitive_to_conservative(2, wl.gamma, rho, u, v_, p)
        else:
            rho, u, p = prims
            out[j] = primitive_to_conservative(1, wl.gamma, np.maximum(rho, 0.3), u, None, np.maximum(p, 0.3))
    return out
