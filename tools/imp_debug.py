"""Debug probe of the NEXT-4 GPU path against the oracle (prints, no asserts)."""
import dataclasses
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as orc  # noqa: E402
from paper_2301_01718_b200 import inputs  # noqa: E402
from paper_2301_01718_b200 import hrom as H  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def maxerr(a, b):
    scale = np.max(np.abs(b), axis=-1, keepdims=True)
    return float(np.max(np.abs(a - b) / np.maximum(scale, 1e-300)))


def filt(orders, sweeps, W=-1):
    wl = inputs.Workload(name="imp", dim=2, nx=44, ny=32, bc=2, recon=2, w=5, r=4, h=2, W=W, f=0.1, hdm="implicit",
                         flux=1, dt=4e-3, seed=11, filter_orders=orders, filter_max_sweeps=sweeps)
    q1 = inputs.initial_condition(wl, "random")
    q2 = inputs.initial_condition(dataclasses.replace(wl, seed=8), "random")
    rng = np.random.default_rng(6)
    v = q1 * (1.0 + 0.02 * np.where(rng.random(q1.shape) < 0.5, 1.0, -1.0))
    S = (rng.random(wl.N) < 0.1).astype(np.uint8)
    vo, kept_o, sw_o = orc.seam_filter_implicit(wl, v, q1, q2, S, wl.dt, order=2, flux=1)
    rom = H.ImplicitROM(wl)
    vg = dev(v).clone()
    kept_g, sw_g = rom.filter(vg, H.mask_from_cells(wl, S), dev(q1), dev(q2), order=2)
    kg = kept_g.cpu().numpy()
    vgn = vg.cpu().numpy()
    print(f"filter orders={orders} sweeps={sweeps} W={W}: sw {sw_g} vs {sw_o}; kept {kg.sum()} vs {kept_o.sum()}, "
          f"diff cells {(kg != kept_o).sum()}, S cells kept by gpu {(kg[S == 1]).sum()}, maxerr {maxerr(vgn, vo):.3e}")
    # the numpy candidate of the first sweep (orders[0])
    nx, ny, c = wl.nx, wl.ny, wl.c
    B = (S == 0) if W < 0 else (orc.dilate_square(wl, S, W).astype(bool) & (S == 0))
    Bm = B.reshape(ny, nx)
    wts = {2: ([1, 2, 1], 4.0), 4: ([-1, 4, 10, 4, -1], 16.0), 6: ([1, -6, 15, 44, 15, -6, 1], 64.0)}
    cf, den = wts[orders[0]]
    rad = len(cf) // 2
    V = v.reshape(c, ny, nx)
    X = sum(cf[m + rad] * V[:, :, np.clip(np.arange(nx) + m, 0, nx - 1)] for m in range(-rad, rad + 1)) / den
    vp = np.where(Bm[None], X, V)
    Y = sum(cf[m + rad] * vp[:, np.clip(np.arange(ny) + m, 0, ny - 1), :] for m in range(-rad, rad + 1)) / den
    vpp = np.where(Bm[None], Y, vp).reshape(c, -1)
    kk = kg.astype(bool)
    if sweeps == 1 and len(orders) == 1:
        if kk.any():
            print("   gpu-kept values vs numpy candidate:", np.max(np.abs(vgn[:, kk] - vpp[:, kk])))
        Rg_new = rom.residual(dev(vpp), dev(q1), dev(q2)).cpu().numpy()
        Rg_old = rom.residual(dev(v), dev(q1), dev(q2)).cpu().numpy()
        keep_formula = B & (np.abs(Rg_new).max(0) < np.abs(Rg_old).max(0))
        print("   keep by gpu residual kernel on numpy candidate:", keep_formula.sum(),
              "band size", B.sum(), "gpu band-count?", None)
    changed = np.nonzero(np.any(vgn != v, axis=0))[0]
    print("   gpu changed cells", changed.size, "oracle changed", np.nonzero(np.any(vo != v, axis=0))[0].size)


def lockstep(name, steps, **kw):
    wl = inputs.preset(name, newton_tol=1e-13, **kw)
    q0 = inputs.initial_condition(wl)
    R = orc.Run(wl, q0)
    rom = H.ImplicitROM(wl)
    rom.set_state(dev(q0))
    for k in range(steps):
        ko = R.step()
        rom.step()
        st = rom.stats()
        q = rom.get_state().cpu().numpy()
        e = maxerr(q, R.state())
        mg = H.cells_from_mask(wl, rom.mask())
        mo = R.mask()
        yo = R.y()
        print(f"{name} {kw} k={k + 1} kind o/g {ko}/{st[0]} J o/g {R.implicit_stats()[0]}/{st[1]} err {e:.3e} "
              f"mask diff {(mg != mo).sum()} |S| {mo.sum()} reff o/g {R.reff()}/{rom.effective_rank()}")
        if ko == 1:
            yg = rom.y().cpu().numpy()[:yo.size]
            print("    y o", np.array2string(yo, precision=6), " g", np.array2string(yg, precision=6))
            eo, eg = R.eps(), rom.indicator().cpu().numpy()
            print("    eps rel", np.linalg.norm(eo - eg) / max(np.linalg.norm(eo), 1e-300))


if __name__ == "__main__":
    filt((2,), 1)
    filt((2, 4, 6), 10)
    lockstep("sod", 12)

