"""Pins of the oracle's Algorithm-1 driver (explicit, z = inf).

The whole-trajectory values are "parity unpinned" against the paper (it prints
no explicit-path numbers); these tests pin the schedule and
the exact-reconstruction identities the north star names (BJ:5).
"""
import dataclasses

import numpy as np
import pytest


def _small(inputs, **kw):
    wl = inputs.Workload("small2d", dim=2, nx=24, ny=18, bc=0, recon=2, cfl=0.4,
                         w=6, r=3, f=0.2, h=2, W=2, seed=2)
    return dataclasses.replace(wl, **kw)


def test_schedule_and_reference_state(orc, inputs):
    wl = _small(inputs)
    q0 = inputs.initial_condition(wl, "quadrant")
    R = orc.Run(wl, q0)
    traj = [q0]
    kinds = []
    for _ in range(12):
        kinds.append(R.step())
        traj.append(R.state())
    # full for k+1 <= w, hybrid afterwards (z = inf)
    assert kinds[: wl.w - 1] == [0] * (wl.w - 1)
    assert all(k in (1, 2) for k in kinds[wl.w - 1:])
    # psi_{k+1} = mean(gamma_{k-w+1..k})
    k = len(traj) - 1
    psi_exp = np.mean(np.stack(traj[k - wl.w + 1:k + 1]), axis=0)
    np.testing.assert_allclose(R.psi(), psi_exp, rtol=1e-15, atol=1e-15)
    # basis orthonormal (BJ:5: 1e-12), rank <= r
    Phi = R.basis()
    assert R.reff() <= wl.r
    assert np.max(np.abs(Phi.T @ Phi - np.eye(Phi.shape[1]))) <= 1e-12
    # |S-hat| = min(ceil(fN), #eps>0)
    ng = orc.n_g(wl.f, wl.N)
    assert R.mask().sum() == min(ng, int((R.eps() > 0).sum()))


def test_lagged_centring_matches_eq9(orc, inputs):
    """Phi_{k+1} spans the POD of [gamma_{k-w+1..k}] - psi_k (A14)."""
    wl = _small(inputs)
    q0 = inputs.initial_condition(wl, "quadrant")
    R = orc.Run(wl, q0)
    traj = [q0]
    for _ in range(wl.w + 3):
        R.step()
        traj.append(R.state())
    k = len(traj) - 1
    psik = np.mean(np.stack(traj[k - wl.w:k]), axis=0)
    X = np.stack([(traj[j] - psik).reshape(-1) for j in range(k - wl.w + 1, k + 1)], axis=1)
    U, S, Vt = np.linalg.svd(X, full_matrices=False)
    Phi = R.basis()
    r = Phi.shape[1]
    # well-separated leading modes agree (LAPACK reference)
    Q = U[:, :r]
    sines = np.linalg.svd(Phi - Q @ (Q.T @ Phi), compute_uv=False)
    assert np.max(sines) < 1e-9 * S[0] / max(S[r - 1] - S[min(r, len(S) - 1)], 1e-300) + 1e-10
    np.testing.assert_allclose(R.sigma(), S, rtol=1e-10, atol=1e-14 * S[0])


def test_full_sample_set_reproduces_full_step(orc, inputs):
    """BJ:5 'exact reconstruction of the sampled cells when the sample set covers the
    grid': with S-hat = all cells the hybrid step equals the full HDM step bitwise."""
    wl = _small(inputs)
    snaps = inputs.smooth_window(wl, wl.w + 1, amp=0.02)
    R = orc.Run(wl, snaps[0])
    R.set_window(wl.w + 3, snaps, np.ones(wl.N, np.uint8))
    dt = orc.dt(wl, snaps[-1])
    assert R.step() == 1
    assert np.array_equal(R.state(), orc.full_step(wl, snaps[-1], dt))
    assert R.filter_stats()[0] == 0


def test_hybrid_step_structure(orc, inputs):
    """S-hat rows = exact HDM rows; S-breve rows = psi + Phi y except filtered band cells;
    y solves the gappy LSQ on the S-hat rows (Eq. 8)."""
    wl = _small(inputs, W=1)
    snaps = inputs.smooth_window(wl, wl.w + 1, amp=0.02)
    rng = np.random.default_rng(1)
    S = (rng.random(wl.N) < 0.15).astype(np.uint8)
    R = orc.Run(wl, snaps[0])
    R.set_window(wl.w + 3, snaps, S)
    Phi, psi = R.basis(), R.psi().reshape(-1)
    dt = orc.dt(wl, snaps[-1])
    R.step()
    g = R.state()
    full = orc.full_step(wl, snaps[-1], dt)
    assert np.array_equal(g[:, S == 1], full[:, S == 1])
    y = R.y()
    rows = np.concatenate([v * wl.N + np.nonzero(S)[0] for v in range(wl.c)])
    y_ref, *_ = np.linalg.lstsq(Phi[rows], (full.reshape(-1) - psi)[rows], rcond=None)
    np.testing.assert_allclose(y, y_ref, rtol=1e-9, atol=1e-12)
    rec = (psi + Phi @ y).reshape(wl.c, wl.N)
    band = orc.dilate_square(wl, S, wl.W) & (1 - S)
    untouched = (S == 0) & (band == 0)
    np.testing.assert_allclose(g[:, untouched], rec[:, untouched], rtol=1e-14, atol=1e-15)
    eps = R.eps()
    exp_eps = np.sum((g - rec) ** 2, axis=0)
    assert np.all(eps[untouched] == 0)
    np.testing.assert_allclose(eps[S == 1], exp_eps[S == 1], rtol=1e-12, atol=1e-30)


def test_config1_trajectory_runs_and_stays_positive(orc, inputs):
    wl = inputs.config(1, steps=60)
    q0 = inputs.initial_condition(wl)
    R = orc.Run(wl, q0)
    kinds = [R.step() for _ in range(wl.steps)]
    assert 2 not in kinds
    assert orc.positivity(wl, R.state()) == -1
    assert R.mask().sum() == orc.n_g(wl.f, wl.N)


# ---- finite full-HDM period z (NEXT-3, G8) ----

def test_z1_is_the_full_hdm_trajectory(orc, inputs):
    """S:448 / P:557: with z = 1 every step is a full HDM step (k mod 1 = 0) and no refresh
    runs ((k+1) mod 1 = 0), so the trajectory equals repeated full steps bitwise."""
    wl = _small(inputs, z=1)
    q0 = inputs.initial_condition(wl, "quadrant")
    R = orc.Run(wl, q0)
    q = q0.copy()
    for _ in range(wl.w + 4):
        assert R.step() == 0
        q = orc.full_step(wl, q, orc.dt(wl, q))
        assert np.array_equal(R.state(), q)


def test_finite_z_schedule_skip_and_projection_indicator(orc, inputs):
    """P:557 full iff k+1 <= w or k mod z = 0; P:578 refresh iff (k+1) mod z != 0; after a
    full step k >= w the indicator is the projection error of gamma_k - psi_{k+1} on
    Phi_{k+1} (G8), pinned against a LAPACK SVD of Eq. 9's X."""
    z = 4
    wl = _small(inputs, z=z)
    q0 = inputs.initial_condition(wl, "quadrant")
    R = orc.Run(wl, q0)
    traj = [q0]
    seen_full_refresh = False
    for k in range(1, 3 * wl.w + 1):
        mask_before, psi_before = R.mask(), R.psi()
        kind = R.step()
        traj.append(R.state())
        full = k + 1 <= wl.w or k % z == 0
        assert (kind == 0) == full, (k, kind)
        if k >= wl.w - 1 and (k + 1) % z == 0:
            # skipped refresh: S-hat_{k+1} and psi are left as they were
            assert np.array_equal(R.mask(), mask_before)
            assert np.array_equal(R.psi(), psi_before)
        if k >= wl.w and full and (k + 1) % z != 0:
            seen_full_refresh = True
            psik = np.mean(np.stack(traj[k - wl.w:k]), axis=0)
            psik1 = np.mean(np.stack(traj[k - wl.w + 1:k + 1]), axis=0)
            np.testing.assert_allclose(R.psi(), psik1, rtol=1e-14, atol=1e-15)
            X = np.stack([(traj[j] - psik).reshape(-1) for j in range(k - wl.w + 1, k + 1)], axis=1)
            U, S, _ = np.linalg.svd(X, full_matrices=False)
            r = R.reff()
            Q = U[:, :r]
            d = (traj[k] - psik1).reshape(-1)
            res = d - Q @ (Q.T @ d)
            eps_exp = (res.reshape(wl.c, wl.N) ** 2).sum(axis=0)
            np.testing.assert_allclose(R.eps(), eps_exp, rtol=1e-8, atol=1e-10 * eps_exp.max())
            # G8 algebra: d lies in range(X) (psi_{k+1} - psi_k = (gamma_k - gamma_{k-w}) / w)
            alpha = np.full(wl.w, -1.0 / wl.w)
            alpha[-1] += 1.0
            np.testing.assert_allclose(X @ alpha, d, rtol=0, atol=1e-13 * np.abs(d).max())
    assert seen_full_refresh


def test_rre_and_odeim_driver_sets(orc, inputs):
    """Algorithm 1 with the paper's own sampling (NEXT-1): RRE-delta selection of G (P:373-380,
    A35) and ODEIM points P of Phi_{k+1} (A36).  Each refresh: G is the oracle's own
    RRE rule on the step's indicator, P = ODEIM(Phi_{k+1}) recomputed from the driver's basis,
    S-hat = G u cells(P), and the hybrid step uses exactly those points (gappy rows = P)."""
    wl = _small(inputs, delta=0.9, n_p=2 * 3)
    q0 = inputs.initial_condition(wl, "quadrant")
    R = orc.Run(wl, q0)
    for k in range(1, wl.w + 6):
        R.step()
        if k < wl.w - 1:
            continue
        S = R.mask()
        G, _ = orc.select_rre(R.eps(), wl.delta)
        rows = R.points()
        phi = R.basis().T.copy()  # (reff, D)
        cells, rows_o = orc.odeim(phi, wl.N, min(wl.n_p, wl.N))
        assert np.array_equal(rows, rows_o)
        want = G.copy()
        want[cells] = 1
        assert np.array_equal(S, want), k
        if k == wl.w - 1:
            # Algorithm 1: G_w = {} at k = w-1, so S-hat_w = P_w exactly
            assert not np.any(R.eps()) and G.sum() == 0
            assert np.array_equal(np.nonzero(S)[0], np.unique(cells))
        assert len(set(cells.tolist())) == len(cells)
    assert np.all(np.isfinite(R.state()))
