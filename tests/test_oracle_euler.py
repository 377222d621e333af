"""Pins of the oracle's Euler finite-volume HDM and explicit step (-m "not gpu").

Each test pins oracle/euler.cpp against something other than itself: SPEC hand
examples (tests/golden/spec_examples.txt), closed forms, invariants (free
stream, conservation, symmetry, translation, dimensional reduction) and the
exact Sod solution that the paper plots in Fig. 8.
"""
import dataclasses
import math
import os

import numpy as np
import pytest

from exact_riemann import ExactRiemann

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    out = {}
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.split("#")[0].strip()
            if line:
                k, *v = line.split()
                out.setdefault(k, []).append(v)
    return out


def _wl(inputs, **kw):
    base = dict(name="t", dim=2, nx=24, ny=20, bc=1, recon=2, cfl=0.4, w=4, r=2, f=0.2, seed=7)
    base.update(kw)
    return inputs.Workload(**base)


# ---------------- pointwise pins ----------------
def test_eos_spec_examples(orc):
    for row in _golden("spec_examples.txt")["eos_1d"]:
        g, rho, m, E = map(float, row[:4])
        exp = list(map(float, row[5:8]))
        p = orc.pressure(1, g, [rho, m, E])
        assert abs(rho - exp[0]) == 0 and abs(m / rho - exp[1]) == 0
        assert abs(p - exp[2]) <= 1e-15 * max(1, abs(exp[2]))


def test_eos_round_trip(orc, inputs):
    wl = _wl(inputs)
    q = inputs.initial_condition(wl, "random")
    k = np.arange(wl.N, dtype=np.uint64) * np.uint64(4)
    p_in = inputs.uniform(wl.seed, inputs.STREAM_TEST, k + np.uint64(3), 0.5, 2.0)
    p = np.array([orc.pressure(2, wl.gamma, q[:, n]) for n in range(wl.N)])
    assert np.max(np.abs(p - p_in) / p_in) <= 1e-13


def test_minmod_and_muscl_examples(orc):
    gd = _golden("spec_examples.txt")
    for row in gd["minmod"]:
        a, b, _, e = row
        assert orc.minmod(float(a), float(b)) == float(e)
    for row in gd["muscl"]:
        um, u0, up, _, l, r = row
        assert orc.muscl_faces(float(um), float(u0), float(up)) == (float(l), float(r))


def test_physical_flux_closed_form_and_rotation(orc):
    g = 1.4
    U = np.array([1.3, 0.7, -0.4, 3.1])
    rho, mx, my, E = U
    p = (g - 1) * (E - 0.5 * (mx * mx + my * my) / rho)
    Fx = orc.physical_flux(2, 0, g, U)
    np.testing.assert_allclose(Fx, [mx, mx * mx / rho + p, my * mx / rho, (E + p) * mx / rho], rtol=1e-15)
    # rotation: y-flux of (rho, mx, my, E) = x-flux of (rho, my, mx, E) with momenta swapped
    Fy = orc.physical_flux(2, 1, g, U)
    Fr = orc.physical_flux(2, 0, g, np.array([rho, my, mx, E]))
    np.testing.assert_allclose(Fy, [Fr[0], Fr[2], Fr[1], Fr[3]], rtol=1e-15)


def test_rusanov_consistency_and_quiescent(orc):
    row = _golden("spec_examples.txt")["rusanov_quiescent"][0]
    g = float(row[0])
    U = np.array(list(map(float, row[1:4])))
    np.testing.assert_allclose(orc.rusanov(1, 0, g, U, U), list(map(float, row[5:8])), atol=1e-15)
    rng = np.random.default_rng(3)
    for _ in range(20):
        rho, u, v, p = rng.uniform(0.2, 2), rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(0.2, 2)
        U = np.array([rho, rho * u, rho * v, p / 0.4 + 0.5 * rho * (u * u + v * v)])
        for ax in (0, 1):
            np.testing.assert_allclose(orc.rusanov(2, ax, 1.4, U, U), orc.physical_flux(2, ax, 1.4, U), rtol=1e-14, atol=1e-15)
    # dissipation sign: Rusanov = central - a/2 jump with a = max(|u|+c)
    UL = np.array([1.0, 0.0, 2.5])
    UR = np.array([0.125, 0.0, 0.25])
    cL, cR = math.sqrt(1.4), math.sqrt(1.4 * 0.1 / 0.125)
    central = 0.5 * (orc.physical_flux(1, 0, 1.4, UL) + orc.physical_flux(1, 0, 1.4, UR))
    exp = central - 0.5 * max(cL, cR) * (UR - UL)
    np.testing.assert_allclose(orc.rusanov(1, 0, 1.4, UL, UR), exp, rtol=1e-15)


def test_dt_closed_form(orc, inputs):
    wl = _wl(inputs, bc=0)
    q = inputs.initial_condition(wl, "uniform")
    rho, u, v, p = 1.3, 0.4, -0.2, 2.1
    c = math.sqrt(1.4 * p / rho)
    exp = wl.cfl / ((abs(u) + c) / (1.0 / wl.nx) + (abs(v) + c) / (1.0 / wl.ny))
    assert abs(orc.dt(wl, q) - exp) <= 1e-14 * exp


def test_positivity_reports_lowest_cell(orc, inputs):
    wl = _wl(inputs)
    q = inputs.initial_condition(wl, "uniform")
    assert orc.positivity(wl, q) == -1
    q2 = q.copy()
    q2[3, 41] = 0.0  # E = 0 -> p < 0
    q2[0, 77] = -1.0
    assert orc.positivity(wl, q2) == 41


# ---------------- invariants of the full step ----------------
@pytest.mark.parametrize("dim,bc,recon", [(1, 0, 1), (1, 1, 2), (2, 0, 2), (2, 1, 1), (2, 1, 2)])
def test_free_stream_bitwise(orc, inputs, dim, bc, recon):
    wl = _wl(inputs, dim=dim, ny=1 if dim == 1 else 20, bc=bc, recon=recon)
    q = inputs.initial_condition(wl, "uniform")
    out = orc.full_step(wl, q, orc.dt(wl, q))
    assert np.array_equal(out, q)


@pytest.mark.parametrize("dim,recon,kind", [(1, 1, "random"), (1, 2, "random"), (2, 2, "random"), (2, 2, "blasts"), (2, 1, "blasts")])
def test_conservation_periodic(orc, inputs, dim, recon, kind):
    wl = _wl(inputs, dim=dim, ny=1 if dim == 1 else 20, bc=1, recon=recon)
    q = inputs.initial_condition(wl, kind)
    tot0 = q.sum(axis=1)
    for _ in range(5):
        q = orc.full_step(wl, q, orc.dt(wl, q))
    tot = q.sum(axis=1)
    scale = np.abs(q).sum(axis=1)
    assert np.all(np.abs(tot - tot0) <= 1e-13 * scale)


def test_mirror_symmetry_quadrant(orc, inputs):
    wl = _wl(inputs, nx=32, ny=32, bc=0)
    q = inputs.initial_condition(wl, "quadrant_clean")
    for _ in range(4):
        q = orc.full_step(wl, q, orc.dt(wl, q))
    Q = q.reshape(4, 32, 32)
    T = np.stack([Q[0].T, Q[2].T, Q[1].T, Q[3].T])  # x<->y with mx<->my
    assert np.max(np.abs(T - Q)) <= 1e-14 * np.max(np.abs(Q))


def test_translation_periodic_bitwise(orc, inputs):
    wl = _wl(inputs)
    q = inputs.initial_condition(wl, "blasts")
    Q = q.reshape(4, wl.ny, wl.nx)
    qs = np.roll(np.roll(Q, 5, axis=2), 3, axis=1).reshape(4, -1).copy()
    dt = 0.3 * orc.dt(wl, q)
    a = orc.full_step(wl, q, dt)
    b = orc.full_step(wl, qs, dt)
    A = np.roll(np.roll(a.reshape(4, wl.ny, wl.nx), 5, axis=2), 3, axis=1).reshape(4, -1)
    assert np.array_equal(A, b)


@pytest.mark.parametrize("recon", [1, 2])
def test_2d_y_uniform_reduces_to_1d(orc, inputs, recon):
    w1 = _wl(inputs, dim=1, nx=40, ny=1, bc=0, recon=recon)
    w2 = _wl(inputs, dim=2, nx=40, ny=4, bc=1, recon=recon)
    q1 = inputs.initial_condition(w1, "random")
    q2 = np.zeros((4, w2.N))
    for j in range(4):
        sl = slice(j * 40, (j + 1) * 40)
        q2[0, sl], q2[1, sl], q2[3, sl] = q1[0], q1[1], q1[2]
    w2b = dataclasses.replace(w2, bc=0)
    dt = 1e-3
    a = orc.full_step(w1, q1, dt)
    b = orc.full_step(w2b, q2, dt)
    for j in range(4):
        sl = slice(j * 40, (j + 1) * 40)
        assert np.array_equal(b[0, sl], a[0]) and np.array_equal(b[1, sl], a[1]) and np.array_equal(b[3, sl], a[2])
        assert np.all(b[2, sl] == 0.0)


# ---------------- accuracy against the exact solution ----------------
def test_exact_riemann_reproduces_golden_star_state():
    vals = {k: float(v[0][0]) for k, v in _golden("sod_star.txt").items()}
    ex = ExactRiemann((1.0, 0.0, 1.0), (0.125, 0.0, 0.1))
    assert abs(ex.p_star - vals["p_star"]) < 1e-10
    assert abs(ex.u_star - vals["u_star"]) < 1e-10
    assert abs(ex.star_density("L") - vals["rho_star_left"]) < 1e-10
    assert abs(ex.star_density("R") - vals["rho_star_right"]) < 1e-10
    assert abs(ex.shock_speed_right() - vals["shock_speed"]) < 1e-10
    h, t = ex.rarefaction_left()
    assert abs(h - vals["rarefaction_head"]) < 1e-10 and abs(t - vals["rarefaction_tail"]) < 1e-10


def _sod_l1(orc, inputs, N, recon, T=0.2):
    wl = inputs.Workload("sod", dim=1, nx=N, ny=1, bc=0, recon=recon, cfl=0.5)
    q = inputs.initial_condition(wl, "sod_clean")
    t = 0.0
    while t < T - 1e-15:
        dt = min(orc.dt(wl, q), T - t)
        q = orc.full_step(wl, q, dt)
        t += dt
    X, _ = wl.cell_centres()
    rho_ex, _, _ = ExactRiemann((1.0, 0.0, 1.0), (0.125, 0.0, 0.1)).sample((X - 0.5) / T)
    return np.mean(np.abs(q[0] - rho_ex))


@pytest.mark.parametrize("recon", [1, 2])
def test_sod_l1_error_decreases_under_refinement(orc, inputs, recon):
    errs = [_sod_l1(orc, inputs, N, recon) for N in (250, 500, 1000, 2000)]
    assert all(b < a for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < (0.02 if recon == 1 else 0.008), errs


def test_entropy_wave_order(orc, inputs):
    """rho = 1 + 0.2 sin(2 pi (x - t)), u = 1, p = 1 is an exact periodic Euler solution."""
    errs = []
    T = 0.25
    for N in (64, 128, 256):
        wl = inputs.Workload("ew", dim=1, nx=N, ny=1, bc=1, recon=2, cfl=0.4)
        q = inputs.initial_condition(wl, "entropy_wave")
        nsteps = int(math.ceil(T / (0.2 / N)))
        dt = T / nsteps
        for _ in range(nsteps):
            q = orc.full_step(wl, q, dt)
        X, _ = wl.cell_centres()
        # exact cell average of rho at T
        dx = 1.0 / N
        ex = 1.0 + 0.2 * (np.cos(2 * np.pi * (X - dx / 2 - T)) - np.cos(2 * np.pi * (X + dx / 2 - T))) / (2 * np.pi * dx)
        errs.append(np.mean(np.abs(q[0] - ex)))
    orders = [math.log2(a / b) for a, b in zip(errs, errs[1:])]
    assert min(orders) > 1.5, (errs, orders)


# ---------------- exact restriction of the masked step (Eq. 7) ----------------
@pytest.mark.parametrize("dim,bc,recon", [(1, 0, 1), (2, 0, 2), (2, 1, 2)])
def test_masked_step_exact_restriction(orc, inputs, dim, bc, recon):
    wl = _wl(inputs, dim=dim, nx=30, ny=1 if dim == 1 else 22, bc=bc, recon=recon, h=2)
    q = inputs.initial_condition(wl, "random")
    dt = 0.5 * orc.dt(wl, q)
    full = orc.full_step(wl, q, dt)
    rng = np.random.default_rng(11)
    T = (rng.random(wl.N) < 0.08).astype(np.uint8)
    out = orc.masked_step(wl, q, dt, T)
    sel = np.nonzero(T)[0]
    assert np.array_equal(out[:, sel], full[:, sel])
    assert np.all(np.isnan(out[:, T == 0]))
    # perturbing a cell outside A0 = T (+) C_h three times leaves the T rows unchanged
    A0 = orc.dilate_cross(wl, orc.dilate_cross(wl, orc.dilate_cross(wl, T, 2), 2), 2)
    outside = np.nonzero(A0 == 0)[0]
    q2 = q.copy()
    q2[:, outside] *= 1.01
    out2 = orc.masked_step(wl, q2, dt, T)
    assert np.array_equal(out2[:, sel], out[:, sel])
    # T = all -> the full step
    allm = np.ones(wl.N, np.uint8)
    assert np.array_equal(orc.masked_step(wl, q, dt, allm), full)
