"""Oracle trajectories in worker processes (test infrastructure for the long trajectory tests).

run_oracle() runs Algorithm 1 of the oracle (oracle/, single-threaded) for `steps` steps from
the workload's seeded IC, optionally perturbed by 1e-15 (ensemble member `member` >= 0, the
method's own rounding sensitivity, G6), or the full-HDM trajectory (hdm=True), and
stores gamma_0..gamma_steps, the masks S-hat_{k+1} and the dt of every step in .npy files under
`outdir`.  Several runs execute concurrently in separate processes (one core each), so a
200-step config-2 ensemble costs one run's wall time.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def run_oracle(cfg, steps, member, outdir, hdm=False):
    import oracle
    from paper_2301_01718_b200 import inputs
    wl = inputs.config(cfg, steps=steps)
    q0 = inputs.initial_condition(wl)
    if member >= 0:
        rng = np.random.default_rng(member)
        q0 = q0 * (1.0 + 1e-15 * rng.standard_normal(q0.shape))
    tag = "hdm" if hdm else ("ref" if member < 0 else f"ens{member}")
    S = np.lib.format.open_memmap(os.path.join(outdir, f"{tag}_states.npy"), mode="w+", dtype=np.float64,
                                  shape=(steps + 1,) + q0.shape)
    M = np.lib.format.open_memmap(os.path.join(outdir, f"{tag}_masks.npy"), mode="w+", dtype=np.uint8,
                                  shape=(steps + 1, wl.N))
    dts = np.zeros(steps + 1)
    S[0] = q0
    if hdm:
        q = q0
        for k in range(1, steps + 1):
            dts[k] = oracle.dt(wl, q)
            q = oracle.full_step(wl, q, dts[k])
            S[k] = q
    else:
        R = oracle.Run(wl, q0)
        for k in range(1, steps + 1):
            R.step()
            S[k] = R.state()
            M[k] = R.mask()
            dts[k] = R.dt()
    S.flush()
    M.flush()
    np.save(os.path.join(outdir, f"{tag}_dts.npy"), dts)
    return tag
