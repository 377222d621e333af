"""Pins of the oracle's sampling sets, indicator selection and seam
filter.  Brute-force set algebra, SPEC hand examples and the closed-form
Shapiro response 1 - sin^{2n}(theta/2)."""
import dataclasses
import math
import os

import numpy as np
import pytest

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
    base = dict(name="t", dim=2, nx=10, ny=10, bc=0, recon=2, w=4, r=2, f=0.2, seed=3, h=2, W=3)
    base.update(kw)
    return inputs.Workload(**base)


# ---------------- dilation / sets ----------------
def test_dilation_spec_examples(orc, inputs):
    for row in _golden("spec_examples.txt")["dilate1d"]:
        N, g, h = int(row[1]), int(row[3]), int(row[5])
        exp = sorted(int(x) for x in row[7:])
        wl = _wl(inputs, dim=1, nx=N, ny=1)
        m = np.zeros(N, np.uint8)
        m[g] = 1
        out = orc.dilate_cross(wl, m, h)
        assert sorted(np.nonzero(out)[0].tolist()) == exp


def _brute_dilate(wl, m, offsets):
    out = np.zeros(wl.N, np.uint8)
    for n in range(wl.N):
        i, j = n % wl.nx, n // wl.nx
        for a, b in offsets:
            ii, jj = i + a, j + b
            if wl.bc == 1:
                ii %= wl.nx
                jj %= wl.ny
            elif not (0 <= ii < wl.nx and 0 <= jj < wl.ny):
                continue
            if m[jj * wl.nx + ii]:
                out[n] = 1
    return out


@pytest.mark.parametrize("bc", [0, 1])
def test_dilation_brute_force_and_set_identities(orc, inputs, bc):
    wl = _wl(inputs, bc=bc)
    rng = np.random.default_rng(5 + bc)
    for trial in range(5):
        S = (rng.random(wl.N) < 0.07).astype(np.uint8)
        for h in (1, 2, 3):
            cross = [(a, 0) for a in range(-h, h + 1)] + [(0, b) for b in range(-h, h + 1)]
            assert np.array_equal(orc.dilate_cross(wl, S, h), _brute_dilate(wl, S, cross))
        sq = [(a, b) for a in range(-3, 4) for b in range(-3, 4)]
        assert np.array_equal(orc.dilate_square(wl, S, 3), _brute_dilate(wl, S, sq))
        # S-hat u S-breve = all, S-hat n S-breve = 0, S-tilde subset of S-breve
        A = orc.dilate_cross(wl, S, 2)
        Sb = 1 - S
        St = A & Sb
        assert np.all((S | Sb) == 1) and np.all((S & Sb) == 0) and np.all(St <= Sb)


# ---------------- selection ----------------
def test_n_g(orc):
    assert orc.n_g(0.10, 1000) == 100
    assert orc.n_g(0.15, 65536) == 9831
    assert orc.n_g(0.10, 2048 * 2048) == 419431
    assert orc.n_g(0.05, 2048 * 2048) == 209716


def _brute_select(eps, ng):
    order = sorted(range(len(eps)), key=lambda i: (-eps[i], i))
    chosen = [i for i in order if eps[i] > 0][:ng]
    m = np.zeros(len(eps), np.uint8)
    m[chosen] = 1
    return m


def test_select_vs_brute_force_with_ties(orc):
    rng = np.random.default_rng(9)
    for trial in range(40):
        N = int(rng.integers(1, 300))
        eps = np.round(rng.random(N) * 5) / 5.0 * (rng.random(N) < 0.7)  # many ties and zeros
        ng = int(rng.integers(0, N + 3))
        m, k = orc.select(eps, ng)
        assert np.array_equal(m, _brute_select(eps, ng))
        assert k == min(ng, int((eps > 0).sum()))
    m, k = orc.select(np.zeros(50), 10)
    assert k == 0 and m.sum() == 0


def test_select_rre_examples_and_minimality(orc):
    gd = _golden("spec_examples.txt")["rre"]
    for row in gd:
        eps = np.array([float(x) for x in row[:4]])
        delta = float(row[5])
        m, k = orc.select_rre(eps, delta)
        assert k == int(row[7])
    rng = np.random.default_rng(4)
    for _ in range(200):
        eps = rng.random(int(rng.integers(1, 60))) ** 3
        delta = float(rng.uniform(0.05, 1.0))
        m, k = orc.select_rre(eps, delta)
        srt = np.sort(eps)[::-1]
        frac = np.cumsum(srt) / srt.sum()
        assert frac[k - 1] >= delta - 1e-12
        assert k == 1 or frac[k - 2] < delta + 1e-12


def _rre_exact(eps, delta):
    """Brute force with exact rationals: descending order, ties by ascending index, smallest
    n_g with sum_{j<=n_g} eps / sum eps >= delta (reading A35)."""
    from fractions import Fraction
    order = sorted(range(len(eps)), key=lambda i: (-eps[i], i))
    pos = [i for i in order if eps[i] > 0]
    T = sum(Fraction(float(eps[i])) for i in pos)
    sel = np.zeros(len(eps), np.uint8)
    if T == 0:
        return sel, 0
    target = Fraction(delta) * T
    S = Fraction(0)
    for n, i in enumerate(pos, 1):
        S += Fraction(float(eps[i]))
        sel[i] = 1
        if S >= target:
            return sel, n
    raise AssertionError("unreachable for delta <= 1")


def test_select_rre_exact_sums(orc):
    """The RRE decision is exact: wide exponent ranges (incl. subnormals and huge values), ties,
    zeros, delta = 1 (every positive cell), and deltas placed exactly on a prefix ratio."""
    rng = np.random.default_rng(7)
    cases = []
    for _ in range(120):
        n = int(rng.integers(1, 80))
        e = rng.random(n) * 2.0 ** rng.integers(-1074, 1000, n).astype(float)
        e[rng.random(n) < 0.2] = 0.0
        if n > 3:
            e[1] = e[2] = e[3]  # ties
        cases.append((e, float(rng.choice([1e-300, 0.3, 0.5, 0.9, 0.999999, 1.0]))))
    # a delta exactly equal to a prefix ratio: eps = (3, 1) -> RRE(1) = 3/4
    cases.append((np.array([1.0, 3.0]), 0.75))
    cases.append((np.array([5e-324, 5e-324, 1.0]), 1.0))     # delta = 1 needs the subnormals too
    cases.append((np.array([1e308, 1e308, 1e-308]), 1.0))
    cases.append((np.array([2.0 ** -1074] * 5), 0.5))          # all tied subnormals: ceil(2.5) = 3
    for eps, delta in cases:
        m, k = orc.select_rre(eps, delta)
        me, ke = _rre_exact(eps, delta)
        assert k == ke, (eps, delta, k, ke)
        assert np.array_equal(m, me)
    m, k = orc.select_rre(np.zeros(9), 0.5)
    assert k == 0 and m.sum() == 0


# ---------------- Shapiro filter (A24) ----------------
@pytest.mark.parametrize("order", [2, 4, 6])
def test_shapiro_dc_nyquist_response(orc, order):
    n = order // 2
    const = np.full(17, 3.25)
    np.testing.assert_array_equal(orc.shapiro_1d(const, order), const)
    nyq = np.array([(-1.0) ** i for i in range(32)])
    out = orc.shapiro_1d(nyq, order, periodic=True)
    assert np.max(np.abs(out)) <= 1e-15
    # response at theta = pi/2: 1 - sin^{2n}(pi/4) = 1 - 2^{-n}
    L = 40
    wave = np.cos(np.pi * np.arange(L) / 2)
    out = orc.shapiro_1d(wave, order, periodic=True)
    np.testing.assert_allclose(out, (1 - 2.0 ** (-n)) * wave, atol=1e-15)
    # general theta: 1 - sin^{2n}(theta/2)
    th = 2 * np.pi * 5 / L
    wave = np.cos(th * np.arange(L))
    out = orc.shapiro_1d(wave, order, periodic=True)
    np.testing.assert_allclose(out, (1 - math.sin(th / 2) ** (2 * n)) * wave, atol=1e-14)


def test_shapiro_spike_readback(orc):
    exp = [float(x) for x in _golden("spec_examples.txt")["shapiro2_spike"][0][1:]]
    line = np.zeros(11)
    line[5] = 1.0
    out = orc.shapiro_1d(line, 2)
    np.testing.assert_array_equal(out[4:7], exp)
    out6 = orc.shapiro_1d(line, 6)
    np.testing.assert_allclose(out6[2:9], np.array([1, -6, 15, 44, 15, -6, 1]) / 64.0, rtol=0, atol=0)
    # zeroth-order extrapolation at the ends: a step at the boundary stays flat
    step = np.array([2.0] * 4 + [0.0] * 4)
    np.testing.assert_array_equal(orc.shapiro_1d(step, 2)[:3], [2.0, 2.0, 2.0])


# ---------------- seam filter ----------------
def _filter_case(orc, inputs, bc, seed):
    wl = _wl(inputs, nx=28, ny=20, bc=bc, seed=seed)
    rng = np.random.default_rng(seed)
    F = inputs.initial_condition(wl, "random")
    v = F * (1.0 + 0.05 * rng.standard_normal(F.shape))
    S = np.zeros(wl.N, np.uint8)
    S[rng.choice(wl.N, 12, replace=False)] = 1
    v[:, S == 1] = F[:, S == 1]  # S-hat rows are exact HDM rows (residual 0)
    return wl, v, F, S


@pytest.mark.parametrize("bc,seed", [(0, 1), (1, 2), (0, 3)])
def test_seam_filter_invariants(orc, inputs, bc, seed):
    wl, v, F, S = _filter_case(orc, inputs, bc, seed)
    out, kept, sweeps = orc.seam_filter(wl, v, F, S)
    B = orc.dilate_square(wl, S, wl.W) & (1 - S)
    assert np.all(kept <= B)                       # only band cells change
    assert np.array_equal(out[:, B == 0], v[:, B == 0])
    assert np.array_equal(out[:, S == 1], v[:, S == 1])
    r_in = np.max(np.abs(v - F), axis=0)
    r_out = np.max(np.abs(out - F), axis=0)
    assert np.all(r_out <= r_in + 1e-14)           # gate: per-cell residual never increases
    assert np.all(r_out[kept == 1] < r_in[kept == 1])
    assert all(1 <= s <= wl.filter_max_sweeps for s in sweeps)
    assert kept.sum() > 0


def test_seam_filter_degenerate_bands(orc, inputs):
    wl, v, F, S = _filter_case(orc, inputs, 0, 4)
    for Sd in (np.zeros(wl.N, np.uint8), np.ones(wl.N, np.uint8)):
        out, kept, _ = orc.seam_filter(wl, v, F, Sd)
        if Sd.sum() == 0:
            assert np.array_equal(out, v) and kept.sum() == 0
        else:
            assert np.array_equal(out, v) and kept.sum() == 0
    # residual already zero everywhere: nothing can strictly decrease
    out, kept, _ = orc.seam_filter(wl, F, F, S)
    assert np.array_equal(out, F) and kept.sum() == 0


@pytest.mark.parametrize("bc,seed", [(0, 5), (1, 6)])
def test_whole_domain_filter(orc, inputs, bc, seed):
    """W = -1: the filter runs on every cell off S-hat (the paper's whole hybrid state,
    P:424-432).  Same result as a square band wide enough to cover the grid;
    S-hat untouched; the per-cell residual gate holds."""
    wl, v, F, S = _filter_case(orc, inputs, bc, seed)
    whole = dataclasses.replace(wl, W=-1)
    out, kept, sweeps = orc.seam_filter(whole, v, F, S)
    out2, kept2, sweeps2 = orc.seam_filter(dataclasses.replace(wl, W=max(wl.nx, wl.ny)), v, F, S)
    assert np.array_equal(out, out2) and np.array_equal(kept, kept2) and sweeps == sweeps2
    assert np.array_equal(out[:, S == 1], v[:, S == 1]) and kept[S == 1].sum() == 0
    r_in = np.max(np.abs(v - F), axis=0)
    r_out = np.max(np.abs(out - F), axis=0)
    assert np.all(r_out <= r_in + 1e-14)
    assert kept.sum() > 0


def test_whole_domain_filter_nyquist(orc, inputs):
    """Closed form: a constant state plus a checkerboard a(-1)^(i+j) on a periodic grid with
    S-hat empty.  The order-2 x-pass annihilates the Nyquist mode ((1, 2, 1)/4 of (-1, 1, -1) is
    0), so the first sweep returns the constant exactly on every cell (residual 0 < a: all kept),
    the second keeps nothing (no strict decrease of a zero residual): output = F bit for bit."""
    wl = _wl(inputs, nx=24, ny=16, bc=1, seed=1)
    wl = dataclasses.replace(wl, W=-1)
    F = np.empty((wl.c, wl.N))
    F[:] = np.array([1.0, 0.25, -0.5, 2.5])[:, None]
    i, j = np.meshgrid(np.arange(wl.nx), np.arange(wl.ny))
    cb = ((-1.0) ** (i + j)).reshape(-1)
    v = F + np.array([2.0 ** -10, 2.0 ** -9, 2.0 ** -8, 2.0 ** -7])[:, None] * cb[None, :]  # exact sums
    out, kept, sweeps = orc.seam_filter(wl, v, F, np.zeros(wl.N, np.uint8))
    assert np.array_equal(out, F)
    assert kept.sum() == wl.N
    assert sweeps[0] == 2


# ---------------- ODEIM points (Eq. 10; reading A36) ----------------
def test_odeim_spec_examples(orc):
    """S:295-296 worked examples: a single canonical mode e_7 -> cell 7; two canonical modes
    e_3, e_9 -> cells {3, 9} (here D = N: one variable per cell)."""
    e = np.zeros((1, 20))
    e[0, 7] = 1.0
    cells, rows = orc.odeim(e, 20, 1)
    assert list(cells) == [7] and list(rows) == [7]
    e = np.zeros((2, 20))
    e[0, 3] = 1.0
    e[1, 9] = 1.0
    cells, rows = orc.odeim(e, 20, 2)
    assert list(cells) == [3, 9]
    with pytest.raises(ValueError):
        orc.odeim(e, 20, 21)


def _odeim_brute(phi, N, n_p):
    """Independent re-statement of reading A36 with numpy's least squares (no shared code)."""
    m, D = phi.shape
    P, chosen = [], set()
    for j in range(n_p):
        l = j % m
        r = phi[l].copy()
        if l > 0:
            A = phi[:l][:, P].T
            c = np.linalg.lstsq(A, phi[l][P], rcond=None)[0]
            r = phi[l] - phi[:l].T @ c
        a = np.abs(r)
        for e in range(D):
            if e % N in chosen:
                a[e] = -1.0
        e = int(np.argmax(a))  # first maximum: lowest index
        P.append(e)
        chosen.add(e % N)
    return np.array([e % N for e in P]), np.array(P)


@pytest.mark.parametrize("m,c,N,n_p,seed", [(3, 1, 20, 3, 1), (4, 3, 30, 8, 2), (6, 4, 50, 12, 3),
                                            (5, 4, 40, 13, 4)])
def test_odeim_vs_brute_force_and_deim_property(orc, m, c, N, n_p, seed):
    """Random orthonormal Phi: the same points as an independent greedy; the first m points
    interpolate (P^T Phi nonsingular, the DEIM projector reproduces every mode), points are
    distinct cells, oversampled points reduce the LSQ conditioning."""
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((c * N, m)))
    phi = Q.T.copy()
    cells, rows = orc.odeim(phi, N, n_p)
    cb, rb = _odeim_brute(phi, N, n_p)
    assert np.array_equal(rows, rb) and np.array_equal(cells, cb)
    assert len(set(cells.tolist())) == n_p
    PtP = phi[:, rows[:m]].T  # P^T Phi, m x m
    assert np.linalg.matrix_rank(PtP) == m    # DEIM interpolation is well posed
    # each point carries a nonzero greedy residual, so no column of P^T Phi is dependent
    assert np.all(np.abs(np.diag(np.linalg.qr(PtP)[1])) > 1e-12)
    if n_p > m:
        s_int = np.linalg.svd(phi[:, rows[:m]], compute_uv=False)[-1]
        s_ovs = np.linalg.svd(phi[:, rows], compute_uv=False)[-1]
        assert s_ovs >= s_int - 1e-15  # adding rows never lowers sigma_min (Cauchy interlacing)


# ---------------- seam filter vs an independent brute force ----------------
def _brute_seam_filter(orc, wl, v, F, S, eps_rule="relative"):
    """Independent statement of the residual-gated filter cascade of P:424-438 (readings
    A21-A24): band B = (S-hat (+) Q_W) \\ S-hat; per order of the cascade 2 -> 4 -> 6, sweeps
    j = 1..j_max of  v' = S^x(v) on B  (whole grid lines through orc.shapiro_1d, pinned by the
    closed-form responses above), then  v'' = S^y(v')  on B, residual r = max_var |. - F| per
    cell, keep v'' where r strictly decreases; stop the order when nothing is kept or the largest
    decrease is below eps_f ("relative": (r_old - r_new) / r_old, reading A23; "absolute":
    r_old - r_new, the literal alternative -- used only to show the pins can tell them apart);
    only cells whose old residual exceeds 2^-40 max_var |F| enter the stop test (reading A23')."""
    nx, ny, N, c = wl.nx, (wl.ny if wl.dim == 2 else 1), wl.N, wl.c
    per = wl.bc == 1
    if wl.W < 0:
        B = (S == 0).astype(np.uint8)
    else:
        offs = [(a, b) for a in range(-wl.W, wl.W + 1) for b in (range(-wl.W, wl.W + 1) if wl.dim == 2 else [0])]
        B = _brute_dilate(wl, S, offs) & (1 - S)
    band = np.nonzero(B)[0]
    v = v.copy()
    kept = np.zeros(N, np.uint8)
    sweeps = []
    for order in wl.filter_orders:
        nsw = 0
        for _ in range(wl.filter_max_sweeps):
            nsw += 1
            vp = v.copy()
            for var in range(c):
                g = v[var].reshape(ny, nx)
                xs = np.stack([orc.shapiro_1d(g[j], order, per) for j in range(ny)])
                vp[var, band] = xs.reshape(-1)[band]
            vpp = vp.copy()
            if wl.dim == 2:
                for var in range(c):
                    g = vp[var].reshape(ny, nx)
                    ys = np.stack([orc.shapiro_1d(g[:, i], order, per) for i in range(nx)], axis=1)
                    vpp[var, band] = ys.reshape(-1)[band]
            r_old = np.max(np.abs(v[:, band] - F[:, band]), axis=0)
            r_new = np.max(np.abs(vpp[:, band] - F[:, band]), axis=0)
            fscale = np.max(np.abs(F[:, band]), axis=0)
            keep = r_new < r_old
            if not keep.any():
                break
            cells = band[keep]
            kept[cells] = 1
            v[:, cells] = vpp[:, cells]
            dec = r_old[keep] - r_new[keep]
            if eps_rule == "relative":
                dec = dec / r_old[keep]
            # reading A23': only residuals above the rounding level of the state enter the stop test
            dec = dec[r_old[keep] > 2.0 ** -40 * fscale[keep]]
            if (dec.max() if dec.size else 0.0) < wl.filter_eps:
                break
        sweeps.append(nsw)
    return v, kept, sweeps


@pytest.mark.parametrize("dim,nx,ny,bc,W,nS,seed", [(2, 28, 20, 0, 3, 12, 1), (2, 28, 20, 1, 3, 12, 2),
                                                    (2, 17, 23, 0, 2, 30, 3), (2, 20, 16, 1, -1, 8, 4),
                                                    (1, 90, 1, 0, 3, 6, 5), (1, 64, 1, 1, 3, 5, 6)])
def test_seam_filter_vs_brute_force(orc, inputs, dim, nx, ny, bc, W, nS, seed):
    """orc_seam_filter equals the numpy brute force above on random hybrid states: same output
    bit for bit (the same stencil sums in the same order), kept set and sweep counts."""
    wl = _wl(inputs, dim=dim, nx=nx, ny=ny, bc=bc, seed=seed, W=W)
    rng = np.random.default_rng(seed)
    F = inputs.initial_condition(wl, "random")
    v = F * (1.0 + 0.05 * rng.standard_normal(F.shape))
    S = np.zeros(wl.N, np.uint8)
    S[rng.choice(wl.N, nS, replace=False)] = 1
    v[:, S == 1] = F[:, S == 1]
    out, kept, sweeps = orc.seam_filter(wl, v, F, S)
    bo, bk, bs = _brute_seam_filter(orc, wl, v, F, S)
    assert list(sweeps[:len(bs)]) == bs
    assert np.array_equal(kept, bk)
    np.testing.assert_allclose(out, bo, rtol=2e-16, atol=0)


def test_seam_filter_x_only_checkerboard(orc, inputs):
    """Closed form that separates the x- and y-passes: F constant plus a(-1)^i (varying in x only)
    on a periodic grid, whole-domain band (S-hat empty).  The order-2 x-pass annihilates the x
    Nyquist mode, so v' = F and v'' = S^y(v') = F on every cell: all cells kept in sweep 1, nothing
    in sweep 2, output = F bit for bit.  A y-pass reading v instead of v' would return v (constant
    along y) and keep nothing."""
    wl = dataclasses.replace(_wl(inputs, nx=24, ny=18, bc=1, seed=1), W=-1)
    F = np.empty((wl.c, wl.N))
    F[:] = np.array([1.0, 0.25, -0.5, 2.5])[:, None]
    i = np.tile(np.arange(wl.nx), wl.ny)
    v = F + np.array([2.0 ** -10, 2.0 ** -9, 2.0 ** -8, 2.0 ** -7])[:, None] * ((-1.0) ** i)[None, :]
    out, kept, sweeps = orc.seam_filter(wl, v, F, np.zeros(wl.N, np.uint8))
    assert np.array_equal(out, F)
    assert kept.sum() == wl.N and sweeps[0] == 2
    bo, bk, bs = _brute_seam_filter(orc, wl, v, F, np.zeros(wl.N, np.uint8))
    assert np.array_equal(bo, F) and bs == list(sweeps[:len(bs)])


def test_seam_filter_relative_not_absolute_eps(orc, inputs):
    """The eps_f stop is relative (reading A23): with residuals of order 1e-6 every absolute
    decrease is far below eps_f = 1e-2, so an absolute stop would end each order after its first
    sweep; the relative rule keeps sweeping while some cell's residual drops by >= 1 %.  The oracle
    follows the relative brute force, and the two rules give different sweep counts here."""
    wl = _wl(inputs, nx=28, ny=20, bc=1, seed=7)
    rng = np.random.default_rng(7)
    F = np.empty((wl.c, wl.N))
    F[:] = np.array([1.0, 0.25, -0.5, 2.5])[:, None]  # smooth reference: the filter removes the noise
    v = F + 1e-6 * rng.standard_normal(F.shape)
    S = np.zeros(wl.N, np.uint8)
    S[rng.choice(wl.N, 10, replace=False)] = 1
    v[:, S == 1] = F[:, S == 1]
    out, kept, sweeps = orc.seam_filter(wl, v, F, S)
    _, _, rel_sw = _brute_seam_filter(orc, wl, v, F, S, "relative")
    _, _, abs_sw = _brute_seam_filter(orc, wl, v, F, S, "absolute")
    assert list(sweeps[:len(rel_sw)]) == rel_sw
    assert rel_sw != abs_sw and max(rel_sw) > 1 and abs_sw == [1] * len(abs_sw)


def test_seam_filter_stop_ignores_rounding_level_residuals(orc, inputs):
    """Reading A23': a band cell whose residual is at the rounding level of the state (here
    exactly 2^-52 |F|, one ulp) does not keep the cascade sweeping, however large its relative
    decrease.  A constant state with one-ulp perturbations on a periodic grid: the order-2 sweep
    removes them (relative decrease 1 on every perturbed cell), yet the first sweep already stops
    each order (sweeps == [1, 1, 1]); without the floor the relative rule would sweep again."""
    wl = dataclasses.replace(_wl(inputs, nx=24, ny=20, bc=1, seed=3), W=-1)
    F = np.empty((wl.c, wl.N))
    F[:] = np.array([1.0, 0.5, 0.25, 2.0])[:, None]
    rng = np.random.default_rng(3)
    v = F * (1.0 + 2.0 ** -52 * rng.integers(-1, 2, size=F.shape))
    out, kept, sweeps = orc.seam_filter(wl, v, F, np.zeros(wl.N, np.uint8))
    assert kept.sum() > 0
    assert list(sweeps) == [1, 1, 1]
    _, _, bs = _brute_seam_filter(orc, wl, v, F, np.zeros(wl.N, np.uint8))
    assert bs == [1, 1, 1]
