"""Pins of the oracle's implicit HDM (NEXT-4, oracle/implicit.cpp; -m "not gpu").

Each test pins the oracle against something other than itself:
  * Roe flux against the textbook definition F = 1/2 (F_L + F_R) - 1/2 |A(U~)| dU with
    the ANALYTIC flux Jacobian of the Euler equations written here in numpy and its numerical
    eigen-decomposition; Roe's property A(U~) dU = dF; consistency; supersonic upwinding.
  * walls: quiescent free stream, mass and energy conservation, mirror symmetry.
  * Rusanov through the new residual == the pinned explicit oracle (orc_rhs).
  * BDF1/BDF2: steady fixed point, the residual's closed form, and the
    temporal order (Richardson ratio -> 4 for BDF2, -> 2 for BDF1).
  * Newton: ||R||_inf <= tol at the returned root; S-hat = all reproduces the full solve
    bitwise; a partial solve only reads S-hat u S-tilde (NaN elsewhere).
  * the implicit AROM on Sod against the exact Riemann solution; J within
    [1, j_max] and >= 2 when j_max > 1 (reading A41); z = 1 == the HDM bitwise.
"""
import dataclasses
import math

import numpy as np
import pytest

from exact_riemann import ExactRiemann


# ---------------- Roe flux ----------------
def _cons(dim, g, rho, u, p):
    u = np.atleast_1d(np.asarray(u, dtype=np.float64))
    return np.r_[rho, rho * u, p / (g - 1.0) + 0.5 * rho * (u @ u)]


def _flux(dim, axis, g, U):
    rho, m, E = U[0], U[1:1 + dim], U[-1]
    u = m / rho
    p = (g - 1.0) * (E - 0.5 * rho * (u @ u))
    F = np.empty(dim + 2)
    F[0] = m[axis]
    F[1:1 + dim] = m * u[axis]
    F[1 + axis] += p
    F[-1] = (E + p) * u[axis]
    return F


def _jacobian(dim, axis, g, U):
    """Analytic dF/dU of the Euler flux along `axis` (textbook, conservative variables)."""
    rho = U[0]
    u = U[1:1 + dim] / rho
    E = U[-1]
    q2 = u @ u
    H = g * E / rho - 0.5 * (g - 1.0) * q2
    un = u[axis]
    c = dim + 2
    A = np.zeros((c, c))
    A[0, 1 + axis] = 1.0
    for d in range(dim):
        row = 1 + d
        A[row, 0] = -u[d] * un + (0.5 * (g - 1.0) * q2 if d == axis else 0.0)
        for e in range(dim):
            A[row, 1 + e] = (u[d] if e == axis else 0.0) + (un if e == d else 0.0)
            if d == axis:
                A[row, 1 + e] -= (g - 1.0) * u[e]
        A[row, -1] = (g - 1.0) if d == axis else 0.0
    A[-1, 0] = un * (0.5 * (g - 1.0) * q2 - H)
    for e in range(dim):
        A[-1, 1 + e] = (H if e == axis else 0.0) - (g - 1.0) * u[e] * un
    A[-1, -1] = g * un
    return A


def _roe_state(dim, g, UL, UR):
    sL, sR = math.sqrt(UL[0]), math.sqrt(UR[0])
    uL, uR = UL[1:1 + dim] / UL[0], UR[1:1 + dim] / UR[0]
    pL = (g - 1.0) * (UL[-1] - 0.5 * UL[0] * (uL @ uL))
    pR = (g - 1.0) * (UR[-1] - 0.5 * UR[0] * (uR @ uR))
    HL, HR = (UL[-1] + pL) / UL[0], (UR[-1] + pR) / UR[0]
    u = (sL * uL + sR * uR) / (sL + sR)
    H = (sL * HL + sR * HR) / (sL + sR)
    rho = sL * sR
    p = (g - 1.0) / g * rho * (H - 0.5 * (u @ u))
    return _cons(dim, g, rho, u, p)


def _random_states(seed, dim, n):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        rl, rr = rng.uniform(0.1, 3.0, 2)
        pl, pr = rng.uniform(0.05, 3.0, 2)
        ul, ur = rng.uniform(-1.5, 1.5, (2, dim))
        out.append((_cons(dim, 1.4, rl, ul, pl), _cons(dim, 1.4, rr, ur, pr)))
    return out


def test_analytic_jacobian_is_the_flux_derivative():
    """The test's own Jacobian against central differences of the test's own flux."""
    for dim in (1, 2):
        for axis in range(dim):
            for UL, _ in _random_states(3, dim, 4):
                A = _jacobian(dim, axis, 1.4, UL)
                h = 1e-6
                for k in range(dim + 2):
                    e = np.zeros(dim + 2)
                    e[k] = h
                    fd = (_flux(dim, axis, 1.4, UL + e) - _flux(dim, axis, 1.4, UL - e)) / (2 * h)
                    assert np.allclose(A[:, k], fd, rtol=1e-7, atol=1e-7)


@pytest.mark.parametrize("dim", [1, 2])
def test_roe_equals_eigen_decomposition(orc, dim):
    """F = 1/2 (F_L + F_R) - 1/2 R |Lambda| R^-1 (U_R - U_L) at the Roe state (Roe 1981)."""
    g = 1.4
    worst = 0.0
    for axis in range(dim):
        for UL, UR in _random_states(11 + dim, dim, 20):
            A = _jacobian(dim, axis, g, _roe_state(dim, g, UL, UR))
            lam, R = np.linalg.eig(A)
            Aabs = (R @ np.diag(np.abs(lam)) @ np.linalg.inv(R)).real
            ref = 0.5 * (_flux(dim, axis, g, UL) + _flux(dim, axis, g, UR)) - 0.5 * Aabs @ (UR - UL)
            F = orc.roe(dim, axis, g, UL, UR)
            worst = max(worst, np.max(np.abs(F - ref)) / max(1.0, np.max(np.abs(ref))))
    assert worst <= 1e-12, worst


@pytest.mark.parametrize("dim", [1, 2])
def test_roe_property_and_consistency(orc, dim):
    g = 1.4
    for axis in range(dim):
        for UL, UR in _random_states(21 + dim, dim, 10):
            A = _jacobian(dim, axis, g, _roe_state(dim, g, UL, UR))
            dF = _flux(dim, axis, g, UR) - _flux(dim, axis, g, UL)
            assert np.allclose(A @ (UR - UL), dF, rtol=1e-12, atol=1e-12)  # Roe's property
            F = orc.roe(dim, axis, g, UL, UL)
            assert np.allclose(F, _flux(dim, axis, g, UL), rtol=1e-15, atol=1e-15)


def test_roe_supersonic_upwinding(orc):
    """u_n > a on both sides and at the Roe state: every |lambda| = lambda, so F = F(U_L)."""
    g = 1.4
    UL = _cons(2, g, 1.0, [3.0, 0.2], 1.0)
    UR = _cons(2, g, 0.8, [3.2, -0.1], 0.9)
    assert np.allclose(orc.roe(2, 0, g, UL, UR), _flux(2, 0, g, UL), rtol=1e-13, atol=1e-13)
    UL2 = _cons(2, g, 1.0, [0.1, -3.0], 1.0)
    UR2 = _cons(2, g, 0.9, [0.0, -3.1], 1.1)
    assert np.allclose(orc.roe(2, 1, g, UL2, UR2), _flux(2, 1, g, UR2), rtol=1e-13, atol=1e-13)


# ---------------- residual: walls, consistency with the explicit oracle ----------------
def _wl(inputs, **kw):
    base = dict(name="t", dim=2, nx=12, ny=10, bc=2, recon=2, hdm="implicit", flux=1, dt=1e-3)
    base.update(kw)
    return inputs.Workload(**base)


def test_walls_free_stream_and_conservation(orc, inputs):
    wl = _wl(inputs)
    q = inputs.primitive_to_conservative(2, 1.4, np.full(wl.N, 1.3), np.zeros(wl.N), np.zeros(wl.N),
                                         np.full(wl.N, 0.7))
    assert np.max(np.abs(orc.rhs2(wl, q))) == 0.0
    q = inputs.initial_condition(wl, "random")
    for flux in (0, 1):
        L = orc.rhs2(wl, q, flux)
        # no mass or energy crosses a wall: the flux differences telescope
        for v in (0, 3):
            assert abs(L[v].sum()) <= 1e-12 * np.abs(L[v]).sum()


def test_walls_mirror_symmetry(orc, inputs):
    """A state mirrored in x (u -> -u) has the mirrored residual."""
    wl = _wl(inputs, ny=1, dim=1, nx=30)
    q = inputs.initial_condition(wl, "random")
    L = orc.rhs2(wl, q)
    qm = q[:, ::-1].copy()
    qm[1] *= -1
    Lm = orc.rhs2(wl, qm)
    Lm = Lm[:, ::-1]
    Lm[1] *= -1
    assert np.allclose(L, Lm, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("bc", [0, 1])
def test_rusanov_residual_equals_explicit_oracle(orc, inputs, bc):
    wl = _wl(inputs, bc=bc)
    q = inputs.initial_condition(wl, "random")
    assert np.array_equal(orc.rhs2(wl, q, 0), orc.rhs(wl, q))


# ---------------- BDF ----------------
def test_bdf_residual_closed_form(orc, inputs):
    wl = _wl(inputs)
    q, q1, q2 = (inputs.initial_condition(dataclasses.replace(wl, seed=s), "random") for s in (1, 2, 3))
    L = orc.rhs2(wl, q)
    dt = 2e-3
    R2 = orc.bdf_residual(wl, q, q1, q2, dt, order=2)
    assert np.allclose(R2, q - (dt * (2.0 / 3.0) * L - (1.0 / 3.0) * q2 + (4.0 / 3.0) * q1), rtol=1e-14, atol=1e-14)
    R1 = orc.bdf_residual(wl, q, q1, None, dt, order=1)
    assert np.allclose(R1, q - (dt * L + q1), rtol=1e-14, atol=1e-14)


def test_bdf_steady_state_fixed_point(orc, inputs):
    wl = _wl(inputs)
    q = inputs.primitive_to_conservative(2, 1.4, np.full(wl.N, 0.9), np.zeros(wl.N), np.zeros(wl.N),
                                         np.full(wl.N, 1.1))
    out, its, st = orc.newton(wl, q, q, q, 0.01, order=2, tol=1e-14)
    assert its == 0 and np.array_equal(out, q)


@pytest.mark.parametrize("order,ratio", [(1, 2.0), (2, 4.0)])
def test_bdf_temporal_order(orc, inputs, order, ratio):
    """Same grid, dt / 2 / 4: (q_dt - q_dt/2) / (q_dt/2 - q_dt/4) -> 2^order (the spatial
    error cancels).  BDF2 started with one BDF1 step (reading A39) keeps order 2."""
    wl = inputs.Workload("ew", dim=1, nx=64, ny=1, bc=1, recon=2, hdm="implicit", flux=1)
    q0 = inputs.initial_condition(wl, "entropy_wave")
    T = 0.05

    def run(n):
        dt = T / n
        hist = [q0]
        for k in range(n):
            s = 1 if (order == 1 or k == 0) else 2
            qm2 = hist[-2] if s == 2 else None
            q, its, _ = orc.newton(wl, hist[-1], hist[-1], qm2, dt, order=s, tol=1e-14)
            assert its >= 0
            hist.append(q)
        return hist[-1]

    a, b, c = run(10), run(20), run(40)
    r = np.linalg.norm(a - b) / np.linalg.norm(b - c)
    assert abs(r - ratio) < 0.15 * ratio, r


# ---------------- Newton ----------------
def test_newton_root_and_partial_equals_full(orc, inputs):
    wl = _wl(inputs, nx=20, ny=16)
    q1 = inputs.initial_condition(wl, "random")
    q2 = inputs.initial_condition(dataclasses.replace(wl, seed=9), "random")
    dt = 4e-3
    full, its, st = orc.newton(wl, q1, q1, q2, dt, tol=1e-13)
    assert its > 0 and st[0] <= 1e-13
    assert np.max(np.abs(orc.bdf_residual(wl, full, q1, q2, dt))) <= 1e-13
    allm = np.ones(wl.N, dtype=np.uint8)
    part, its2, _ = orc.newton(wl, q1, q1, q2, dt, mask=allm, tol=1e-13)
    assert its2 == its and np.array_equal(part, full)


def test_newton_partial_reads_only_the_stencil(orc, inputs):
    """Partial HDM (Eq. 6b): unknowns on S-hat, frozen S-tilde = Neighbors(S-hat); every other
    entry NaN.  The solve converges and the S-hat rows satisfy R = 0 with the frozen data."""
    wl = _wl(inputs, nx=24, ny=20)
    q1 = inputs.initial_condition(wl, "random")
    S = np.zeros(wl.N, dtype=np.uint8)
    S[[30, 31, 55, 200, 201, 202, 470]] = 1
    T = orc.dilate_cross(wl, S, 2)
    q = np.where(T[None, :] > 0, q1, np.nan)
    dt = 4e-3
    out, its, st = orc.newton(wl, q, q1, q1, dt, mask=S, tol=1e-13)
    assert its > 0 and st[0] <= 1e-13
    Sb = S.astype(bool)
    assert np.all(np.isfinite(out[:, Sb]))
    # check the S-hat rows against a full residual evaluation (frozen values filled from q1)
    filled = np.where(np.isnan(out), q1, out)
    R = orc.bdf_residual(wl, filled, q1, q1, dt)
    assert np.max(np.abs(R[:, Sb])) <= 1e-13


# ---------------- the implicit AROM (Algorithm 1 with the paper's HDM) ----------------
def test_sod_implicit_hdm_vs_exact(orc, inputs):
    """z = 1: every step a full BDF2 + Roe HDM solve.  L1(rho) error at t = 0.2 against
    the exact Riemann solution is small; all steps converge."""
    wl = inputs.preset("sod", z=1, steps=999)
    q0 = inputs.initial_condition(wl)
    R = orc.Run(wl, q0)
    for _ in range(wl.steps):
        assert R.step() == 0
    q = R.state()
    X, _ = wl.cell_centres()
    rho_ex, _, _ = ExactRiemann((1.0, 0.0, 1.0), (0.125, 0.0, 0.1)).sample((X - 0.5) / 0.2)
    err = np.mean(np.abs(q[0] - rho_ex))
    assert err < 0.006, err


def test_sod_implicit_arom_runs(orc, inputs):
    """z = infinity, delta = 0.8, n_p = 8: J in [2, j_max] on every hybrid
    step, and the hybrid trajectory stays physical and close to the HDM at t = 0.02."""
    wl = inputs.preset("sod", steps=100)
    q0 = inputs.initial_condition(wl)
    R = orc.Run(wl, q0)
    H = orc.Run(dataclasses.replace(wl, z=1), q0)
    Js = []
    for _ in range(wl.steps):
        kind = R.step()
        H.step()
        assert kind in (0, 1, 2)
        if kind == 1:
            Js.append(R.implicit_stats()[0])
    assert Js and min(Js) >= 2 and max(Js) <= wl.j_max
    q, qh = R.state(), H.state()
    assert orc.positivity(wl, q) < 0
    e = np.abs(q - qh).sum() / np.abs(qh).sum()  # e_k
    assert e < 0.02, e


# ---------------- the filter gated by the implicit residual ----------------
def _np_implicit_filter(orc, wl, v, q1, q2, S):
    """Brute force of P:424-432 with the residual v - F_k(v) re-evaluated on the candidate
    (numpy; F_k from the pinned orc.bdf_residual): x-pass then y-pass on the band (every cell off
    S-hat for W = -1), keep where max_var |R| decreases, eps_f stop of reading A23'."""
    v = v.copy()
    nx, ny, c = wl.nx, wl.ny, wl.c
    band = (S == 0) if wl.W < 0 else (orc.dilate_square(wl, S, wl.W).astype(bool) & (S == 0))
    Bm = band.reshape(ny, nx)
    weights = {2: ([1, 2, 1], 4.0), 4: ([-1, 4, 10, 4, -1], 16.0), 6: ([1, -6, 15, 44, 15, -6, 1], 64.0)}
    kept_all = np.zeros(wl.N, np.uint8)
    sweeps = []
    for order in wl.filter_orders:
        cf, den = weights[order]
        rad = len(cf) // 2
        sw = 0
        for _ in range(wl.filter_max_sweeps):
            sw += 1
            V = v.reshape(c, ny, nx)
            X = sum(cf[m + rad] * V[:, :, np.clip(np.arange(nx) + m, 0, nx - 1)] for m in range(-rad, rad + 1)) / den
            vp = np.where(Bm[None], X, V)
            Y = sum(cf[m + rad] * vp[:, np.clip(np.arange(ny) + m, 0, ny - 1), :] for m in range(-rad, rad + 1)) / den
            vpp = np.where(Bm[None], Y, vp).reshape(c, -1)
            Ro = orc.bdf_residual(wl, v, q1, q2, wl.dt)
            Rn = orc.bdf_residual(wl, vpp, q1, q2, wl.dt)
            rold, rnew = np.abs(Ro).max(0), np.abs(Rn).max(0)
            fs = np.abs(v - Ro).max(0)
            keep = band & (rnew < rold)
            gate = keep & (rold > 2.0 ** -40 * fs)
            md = np.max((rold - rnew)[gate] / rold[gate]) if gate.any() else 0.0
            v[:, keep] = vpp[:, keep]
            kept_all[keep] = 1
            if not keep.any() or md < wl.filter_eps:
                break
        sweeps.append(sw)
    return v, kept_all, sweeps


@pytest.mark.parametrize("W", [-1, 2])
def test_implicit_filter_vs_numpy_brute_force(orc, inputs, W):
    wl = _wl(inputs, nx=30, ny=22, W=W)
    q1 = inputs.initial_condition(wl, "random")
    q2 = inputs.initial_condition(dataclasses.replace(wl, seed=8), "random")
    rng = np.random.default_rng(6)
    v = q1 * (1.0 + 0.02 * np.where(rng.random(q1.shape) < 0.5, 1.0, -1.0))
    S = (rng.random(wl.N) < 0.1).astype(np.uint8)
    vo, kept_o, sw_o = orc.seam_filter_implicit(wl, v, q1, q2, S, wl.dt, order=2, flux=1)
    vn, kept_n, sw_n = _np_implicit_filter(orc, wl, v, q1, q2, S)
    assert sw_o == sw_n and np.array_equal(kept_o, kept_n)
    assert np.max(np.abs(vo - vn)) <= 1e-14
    assert kept_o.sum() > 0
