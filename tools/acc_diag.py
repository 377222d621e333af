"""Diagnose one replay step (config-4 parameters on 512^2 by default): GPU-vs-oracle error split
by cell class (S-hat, seam band, filled complement), basis quantities (r_eff, sigma around the
cut, principal angles), gappy-LSQ conditioning kappa(Phi_S), y differences.

python tools/acc_diag.py [k_off] [nx]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as orc  # noqa: E402
from paper_2301_01718_b200 import inputs  # noqa: E402
from paper_2301_01718_b200 import hrom as H  # noqa: E402
import test_gpu_accuracy as T  # noqa: E402


def main():
    k_off = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    nx = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    wl, snaps = T.hdm_trajectory(orc, inputs, 4, inputs.config(4).w + k_off, nx=nx, ny=nx)
    k = wl.w + k_off
    S = (np.random.default_rng(44 + k_off).random(wl.N) < wl.f).astype(np.uint8)
    win = snaps[k - wl.w:k + 1]
    R = orc.Run(wl, win[0])
    R.set_window(k, win, S)
    rom = H.HybridROM(wl)
    rom.set_window(k, T.dev(win.reshape(wl.w + 1, -1)), H.mask_from_cells(wl, S))
    out = {"k": k, "reff_gpu": rom.effective_rank(), "reff_orc": R.reff()}
    sig = R.sigma()
    lam_g = rom.eigenvalues().cpu().numpy()
    re = R.reff()
    out["sigma_o"] = (sig[:min(re + 3, sig.size)] / sig[0]).tolist()
    out["lam_rel_err"] = (np.abs(lam_g[:re] - sig[:re] ** 2) / sig[:re] ** 2).tolist()
    phi_g, psi_g = rom.basis()
    P = phi_g.cpu().numpy().T
    Q = R.basis()
    out["max_principal_sine"] = float(np.linalg.svd(P - Q @ (Q.T @ P), compute_uv=False).max())
    out["col_dev"] = [float(min(np.linalg.norm(P[:, j] - Q[:, j]), np.linalg.norm(P[:, j] + Q[:, j]))) for j in range(re)]
    # gappy LSQ conditioning on the S-hat rows
    rows = np.concatenate([v * wl.N + np.nonzero(S)[0] for v in range(wl.c)])
    sv = np.linalg.svd(Q[rows], compute_uv=False)
    out["kappa_PhiS"] = float(sv[0] / sv[-1])
    dt = orc.dt(wl, win[-1])
    R.step(dt)
    rom.hybrid_step(dt=dt)
    rom.sync()
    g = rom.get_state().cpu().numpy()
    o = R.state()
    yg = rom.y().cpu().numpy()[:re]
    yo = R.y()[:re] if hasattr(R, "y") else None
    if yo is not None:
        out["y_rel_err"] = (np.abs(yg - yo) / np.maximum(np.abs(yo), 1e-300)).tolist()
    Sq = S.astype(bool).reshape(wl.ny, wl.nx)
    T2 = Sq.copy()
    for dy in range(-wl.W, wl.W + 1):
        for dx in range(-wl.W, wl.W + 1):
            T2 |= np.roll(np.roll(Sq, dy, 0), dx, 1)
    band = (T2 & ~Sq).reshape(-1)
    comp = ~T2.reshape(-1)
    err = np.abs(g - o) / np.max(np.abs(o), axis=1, keepdims=True)
    cell_err = err.max(axis=0)
    for name, m in (("S", S.astype(bool)), ("band", band), ("fill", comp)):
        out[f"maxerr_{name}"] = float(cell_err[m].max()) if m.any() else 0.0
        out[f"relL2_{name}"] = float(np.linalg.norm((g - o)[:, m]) / np.linalg.norm(o[:, m])) if m.any() else 0.0
    worst = np.argsort(cell_err)[::-1][:10]
    out["worst_cells"] = [(int(n), float(cell_err[n]), "S" if S[n] else ("band" if band[n] else "fill")) for n in worst]
    eg = rom.indicator().cpu().numpy()
    eo = R.eps()
    flip = (eg > 0) ^ (eo > 0)
    out["eps_flips"] = {name: int((flip & m).sum()) for name, m in (("S", S.astype(bool)), ("band", band), ("fill", comp))}
    fl = np.nonzero(flip)[0][:8]
    out["eps_flip_examples"] = [(int(n), float(eg[n]), float(eo[n]), float(cell_err[n])) for n in fl]
    out["eps_max"] = float(eo.max())
    out["bar"] = T.svd_bar(sig, re)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
