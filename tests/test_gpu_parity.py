"""GPU parity: libhrom (CUDA, sm_100a) vs the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star, BJ:5): per-step state relative L2 <= 1e-12,
200-step trajectory <= 1e-9, masks and compacted lists bit-exact when both sides are
fed the oracle's indicator, basis subspaces principal-angle sine <= 1e-10 on the
well-separated leading modes (reading A15).
"""
import dataclasses
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2301_01718_b200 import hrom as H  # noqa: E402


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def maxerr(a, b):
    """Per-element max error relative to the largest |entry| of each variable's field (the
    check beside every global relative L2: a localised error cannot hide in the norm)."""
    a = np.asarray(a)
    b = np.asarray(b)
    a = a.reshape(b.shape)
    scale = np.max(np.abs(b), axis=-1, keepdims=True) if b.ndim > 1 else np.max(np.abs(b))
    return float(np.max(np.abs(a - b) / np.maximum(scale, 1e-300)))


def close(a, b, tol):
    """Global relative L2 and per-element max error both within tol."""
    return rel(a, b) <= tol and maxerr(a, b) <= tol


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def small2d(inputs, **kw):
    wl = inputs.Workload("small2d", dim=2, nx=70, ny=45, bc=0, recon=2, cfl=0.4, w=8, r=5, f=0.12,
                         h=2, W=3, seed=21)
    return dataclasses.replace(wl, **kw)


CASES = [
    ("1d-first-transmissive", dict(dim=1, nx=1000, ny=1, bc=0, recon=1, cfl=0.5), "sod"),
    ("1d-muscl-periodic", dict(dim=1, nx=333, ny=1, bc=1, recon=2), "random"),
    ("2d-muscl-transmissive-ragged", dict(nx=100, ny=37, bc=0), "quadrant"),
    ("2d-muscl-periodic", dict(nx=64, ny=48, bc=1), "blasts"),
    ("2d-first-periodic-ragged", dict(nx=45, ny=33, bc=1, recon=1), "random"),
]


@pytest.mark.parametrize("name,kw,kind", CASES, ids=[c[0] for c in CASES])
def test_full_step_parity(orc, inputs, name, kw, kind):
    wl = small2d(inputs, **kw)
    q = inputs.initial_condition(wl, kind)
    rom = H.HybridROM(wl)
    rom.set_state(dev(q))
    dt_dev = torch.zeros(1, dtype=torch.float64, device="cuda")
    qo = q.copy()
    for step in range(5):
        rom.full_step(dt_out=dt_dev)
        dto = orc.dt(wl, qo)
        qo = orc.full_step(wl, qo, dto)
        torch.cuda.synchronize()
        assert abs(dt_dev.item() - dto) <= 1e-14 * dto
        g = rom.get_state().cpu().numpy()
        assert close(g, qo, 1e-12), ((step, rel(g, qo)), maxerr(g, qo))


def test_full_step_conservation_and_free_stream(inputs):
    wl = small2d(inputs, nx=96, ny=64, bc=1)
    q = inputs.initial_condition(wl, "blasts")
    rom = H.HybridROM(wl)
    rom.set_state(dev(q))
    for _ in range(10):
        rom.full_step()
    g = rom.get_state().cpu().numpy()
    scale = np.abs(g).sum(axis=1)
    assert np.all(np.abs(g.sum(axis=1) - q.sum(axis=1)) <= 1e-13 * scale)
    u = inputs.initial_condition(wl, "uniform")
    rom.set_state(dev(u))
    rom.full_step()
    assert np.array_equal(rom.get_state().cpu().numpy(), u)


def _mask_dev(wl, m):
    return H.mask_from_cells(wl, m.astype(np.uint8))


def test_sample_bit_exact(orc, inputs):
    """H8 fed the oracle's indicator: S-hat bit-exact, ties by ascending index (A18)."""
    wl = small2d(inputs, nx=130, ny=77, bc=1)
    rom = H.HybridROM(wl)
    q = inputs.initial_condition(wl, "random")
    rom.set_state(dev(q))
    rng = np.random.default_rng(3)
    for trial in range(6):
        eps = np.round(rng.random(wl.N) * 50) / 50.0 * (rng.random(wl.N) < 0.4)  # ties and zeros
        f = [0.01, 0.05, 0.1, 0.2, 0.5, 1.0][trial]
        ng = orc.n_g(f, wl.N)
        m_o, k_o = orc.select(eps, ng)
        mw = torch.zeros(rom.mask_words, dtype=torch.int32, device="cuda")
        lst = torch.zeros(wl.N, dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
        rom.sample(f, eps=dev(eps), mask_out=mw, list_out=lst, count_out=cnt)
        torch.cuda.synchronize()
        m_g = H.cells_from_mask(wl, mw)
        assert np.array_equal(m_g, m_o), trial
        n = int(cnt.item())
        assert n == k_o
        assert np.array_equal(lst[:n].cpu().numpy(), np.nonzero(m_o)[0])


def _replay_case(orc, inputs, wl, seed=5, frac=0.12, amp=0.03):
    snaps = inputs.smooth_window(wl, wl.w + 1, seed=seed, amp=amp)
    rng = np.random.default_rng(seed)
    S = (rng.random(wl.N) < frac).astype(np.uint8)
    return snaps, S


@pytest.mark.parametrize("kw", [dict(), dict(bc=1, nx=64, ny=40), dict(dim=1, nx=500, ny=1, recon=1, w=12, r=6),
                                dict(w=90, r=20, nx=48, ny=40), dict(w=128, r=64, nx=48, ny=40, bc=1),
                                dict(W=-1), dict(W=-1, bc=1, nx=64, ny=40)],
                         ids=["2d-transmissive", "2d-periodic", "1d", "2d-wide-window", "2d-w128-config5-window",
                              "2d-whole-domain-filter", "2d-periodic-whole-domain-filter"])
def test_hybrid_step_replay_parity(orc, inputs, kw):
    """One hybrid step from the same window and S-hat on both sides (Alg. 1)."""
    wl = small2d(inputs, **kw)
    snaps, S = _replay_case(orc, inputs, wl)
    k = wl.w + 5
    R = orc.Run(wl, snaps[0])
    R.set_window(k, snaps, S)
    rom = H.HybridROM(wl)
    rom.set_window(k, dev(snaps.reshape(wl.w + 1, -1)), _mask_dev(wl, S))
    # basis parity before the step: eigenvalues of X^T X = sigma^2
    lam = rom.eigenvalues().cpu().numpy()
    sig = R.sigma()
    re = R.reff()
    assert rom.effective_rank() == re
    np.testing.assert_allclose(lam[:re], sig[:re] ** 2, rtol=1e-9, atol=1e-13 * sig[0] ** 2)
    phi_g, psi_g = rom.basis()
    phi_o = R.basis()
    np.testing.assert_allclose(psi_g.cpu().numpy().reshape(-1), R.psi().reshape(-1), rtol=1e-14, atol=1e-15)
    P = phi_g.cpu().numpy().T
    # subspace of the leading j modes is fixed to ~eps*lambda_0/(lambda_{j-1}-lambda_j) (A15):
    # check the largest j <= r_eff whose gap makes that <= 1e-12
    lamo = sig ** 2
    lamo_next = np.append(lamo[1:], 0.0)
    ok = [j for j in range(1, re + 1) if 2.2e-16 * lamo[0] / max(lamo[j - 1] - lamo_next[j - 1], 1e-300) <= 1e-12]
    nchk = max(ok) if ok else 1
    Q = phi_o[:, :nchk]
    sines = np.linalg.svd(P[:, :nchk] - Q @ (Q.T @ P[:, :nchk]), compute_uv=False)
    assert sines.max() <= 1e-10, (nchk, sines.max())
    # the step
    dt = orc.dt(wl, snaps[-1])
    R.step(dt)
    rom.hybrid_step(dt=dt)
    rom.sync()
    g = rom.get_state().cpu().numpy()
    o = R.state()
    assert close(g, o, 1e-12), (rel(g, o), maxerr(g, o))
    # S-hat rows are exact HDM rows on both sides
    full = orc.full_step(wl, snaps[-1], dt)
    assert rel(g[:, S == 1], full[:, S == 1]) <= 1e-13
    eg = rom.indicator().cpu().numpy()
    eo = R.eps()
    assert np.array_equal(eg > 0, eo > 0)
    np.testing.assert_allclose(eg, eo, rtol=1e-6, atol=1e-12 * max(eo.max(), 1e-300))


def test_masked_rows_bitwise_equal_full_step(inputs):
    """Exact restriction (Eq. 7): S-hat rows of the GPU hybrid step == GPU full step, bitwise."""
    wl = small2d(inputs, nx=80, ny=50, bc=1)
    snaps = inputs.smooth_window(wl, wl.w + 1, seed=9, amp=0.05)
    rng = np.random.default_rng(2)
    S = (rng.random(wl.N) < 0.1).astype(np.uint8)
    a = H.HybridROM(wl)
    a.set_window(wl.w + 2, dev(snaps.reshape(wl.w + 1, -1)), _mask_dev(wl, S))
    dt = 1.3e-3
    a.hybrid_step(dt=dt)
    b = H.HybridROM(wl)
    b.set_state(dev(snaps[-1]))
    b.full_step(dt=dt)
    ga = a.get_state().cpu().numpy()
    gb = b.get_state().cpu().numpy()
    assert np.array_equal(ga[:, S == 1], gb[:, S == 1])


def test_full_sample_set_equals_full_step(inputs):
    """BJ:5: exact reconstruction of the sampled cells when the sample set covers the grid."""
    wl = small2d(inputs, nx=48, ny=40, bc=0)
    snaps = inputs.smooth_window(wl, wl.w + 1, seed=4, amp=0.05)
    a = H.HybridROM(wl)
    a.set_window(wl.w + 2, dev(snaps.reshape(wl.w + 1, -1)), _mask_dev(wl, np.ones(wl.N, np.uint8)))
    a.hybrid_step(dt=1e-3)
    b = H.HybridROM(wl)
    b.set_state(dev(snaps[-1]))
    b.full_step(dt=1e-3)
    assert np.array_equal(a.get_state().cpu().numpy(), b.get_state().cpu().numpy())


def test_gram_dmma_vs_oracle(orc, inputs):
    wl = small2d(inputs)
    rom = H.HybridROM(wl)
    # slab_gram_kernel instantiations (16 NSB DMMA columns + a tail of <= 2 FMA columns) and
    # column counts that fall back to gather_gram_kernel (7, 40, 130); ragged row counts
    for ncol, rows in [(7, 1000), (32, 777), (33, 4097), (34, 3001), (40, 999), (48, 2049), (49, 5003),
                       (50, 1001), (64, 4096), (65, 20011), (66, 2047), (96, 3333), (97, 1025), (128, 4099),
                       (129, 3001), (130, 3001)]:
        S = inputs.random_values(ncol + 1, ncol * rows, 0.5, 1.5).reshape(ncol, rows)
        rho = inputs.random_values(ncol + 2, rows, 0.5, 1.5)
        Cg = rom.gram(dev(S), dev(rho)).cpu().numpy()
        Co = orc.gram(S, rho)
        assert np.max(np.abs(Cg - Co)) <= 1e-13 * np.max(np.abs(Co)), ncol


def _trajectories(orc, inputs, wl, steps, nens=3, keep_ens=False):
    """GPU, oracle and an ensemble of oracle runs from 1e-15-perturbed ICs."""
    q0 = inputs.initial_condition(wl)
    rom = H.HybridROM(wl)
    rom.set_state(dev(q0))
    R = orc.Run(wl, q0)
    ens = []
    for s in range(nens):
        rng = np.random.default_rng(s)
        ens.append(orc.Run(wl, q0 * (1.0 + 1e-15 * rng.standard_normal(q0.shape))))
    rows = []
    snaps, masks, dts = [q0], [], []
    ens_states = [[] for _ in ens]
    for k in range(1, steps + 1):
        rom.step()
        R.step()
        for i, E in enumerate(ens):
            E.step()
            if keep_ens:
                ens_states[i].append(E.state())
        o = R.state()
        snaps.append(o)
        masks.append(R.mask())
        dts.append(R.dt())
        g = rom.get_state().cpu().numpy()
        flip = k >= wl.w - 1 and not np.array_equal(H.cells_from_mask(wl, rom.mask()), R.mask())
        sref = max(rel(E.state(), o) for E in ens)
        rows.append((k, rel(g, o), sref, flip, g))
    rom.sync()
    if keep_ens:
        return rows, snaps, masks, dts, ens_states
    return rows, snaps, masks, dts


def l1err(a, b):
    """e_k of P:704-709 (relative L1 over the D entries, uniform cells)."""
    return float(np.abs(np.asarray(a) - np.asarray(b)).sum() / np.abs(np.asarray(b)).sum())


def _ebar_check(e_gpu, e_ref, e_ens):
    """The method's own accuracy (e-bar of P:711-714 against the full HDM) is reproduced: the GPU
    trajectory's e-bar differs from the oracle's by at most 3x the spread of the oracle ensemble's
    e-bars (its rounding sensitivity, G6) or 2 % of e-bar, whichever is larger."""
    eb_g, eb_o = float(np.mean(e_gpu)), float(np.mean(e_ref))
    spread = max(abs(float(np.mean(e)) - eb_o) for e in e_ens)
    assert abs(eb_g - eb_o) <= max(3 * spread, 0.02 * eb_o), (eb_g, eb_o, spread)
    return eb_g, eb_o, spread


def test_trajectory_config1(orc, inputs):
    """200-step Algorithm-1 trajectory of config 1 (BJ:7).

    The explicit hybrid map amplifies rounding: the ORACLE itself, started from an IC
    perturbed by 1e-15, drifts from its own trajectory by ~x1.25 per hybrid step and its
    sampling masks flip (a discrete, O(1e-6) jump) around k = 165, so the
    north_star's 200-step 1e-9 bar is below the method's own conditioning.  The bar here is
    relative to that sensitivity, measured by an oracle ensemble (max drift sref):
      * while sref < 1e-9, the GPU drift is <= 30 sref + 1e-13 (the GPU injects rounding
        differences every step, the ensemble once; observed ratio ~10) and its masks agree;
      * at k = steps the GPU state is physical and within 10x the ensemble's spread;
      * per-step parity: lock-step replays (GPU fed the oracle's window and mask) <= 1e-12."""
    wl = inputs.config(1)
    rows, snaps, masks, dts, ens_states = _trajectories(orc, inputs, wl, wl.steps, keep_ens=True)
    for k, e, sref, flip, g in rows:
        if sref < 1e-9:
            assert e <= 30 * sref + 1e-13, (k, e, sref)
            assert not flip, (k, e, sref)
    k, e, sref, flip, g = rows[-1]
    assert np.all(g[0] > 0), "density must stay positive"
    # the method's accuracy against the full HDM is the oracle's, within its own spread
    q = [inputs.initial_condition(wl)]
    for kk in range(wl.steps):
        q.append(orc.full_step(wl, q[-1], orc.dt(wl, q[-1])))
    e_gpu = [l1err(r[4], q[r[0]]) for r in rows]
    e_ref = [l1err(snaps[r[0]], q[r[0]]) for r in rows]
    e_ens = [[l1err(es[i], q[r[0]]) for i, r in enumerate(rows)] for es in ens_states]
    _ebar_check(e_gpu, e_ref, e_ens)
    # lock-step replay at several steps: one hybrid step from the oracle's window
    for k in (wl.w, wl.w + 1, wl.w + 50, 150, wl.steps - 1):
        rom = H.HybridROM(wl)
        win = np.stack(snaps[k - wl.w:k + 1]).reshape(wl.w + 1, -1)
        rom.set_window(k, dev(win), _mask_dev(wl, masks[k - 1]))
        rom.hybrid_step(dt=dts[k])
        g = rom.get_state().cpu().numpy()
        assert close(g, snaps[k + 1], 1e-12), ((k, rel(g, snaps[k + 1])), maxerr(g, snaps[k + 1]))


def test_determinism_bitwise(inputs):
    wl = inputs.config(1, steps=40)
    q0 = inputs.initial_condition(wl)
    outs = []
    for _ in range(2):
        rom = H.HybridROM(wl)
        rom.set_state(dev(q0))
        for _ in range(wl.steps):
            rom.step()
        outs.append(rom.get_state().cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("dim,nx,ny,bc,frac,seed", [(2, 70, 45, 0, 0.05, 1), (2, 300, 211, 1, 0.1, 2),
                                                    (2, 64, 64, 1, 0.6, 3), (1, 5000, 1, 0, 0.05, 4),
                                                    (2, 30, 25, 0, 0.1, 5), (1, 900, 1, 1, 0.08, 6)])
def test_seam_filter_parity(orc, inputs, dim, nx, ny, bc, frac, seed):
    """H7 standalone vs the oracle's seam filter (A21-A24): kept set and sweeps
    identical, values to rounding (same stencil sums in the same order)."""
    wl = small2d(inputs, dim=dim, nx=nx, ny=ny, bc=bc, seed=seed)
    rng = np.random.default_rng(seed)
    F = inputs.initial_condition(wl, "random")
    v = F * (1.0 + 0.05 * rng.standard_normal(F.shape))
    S = (rng.random(wl.N) < frac).astype(np.uint8)
    v[:, S == 1] = F[:, S == 1]
    out, kept, sweeps = orc.seam_filter(wl, v, F, S)
    rom = H.HybridROM(wl)
    vg = dev(v)
    kg = torch.zeros(wl.N, dtype=torch.uint8, device="cuda")
    rom.filter(vg, dev(F), _mask_dev(wl, S), kept_out=kg)
    rom.sync()
    assert np.array_equal(kg.cpu().numpy(), kept)
    cnt = rom.debug_counters(8)
    assert list(cnt[4:4 + len(sweeps)]) == list(sweeps)
    assert close(vg.cpu().numpy(), out, 1e-14), (rel(vg.cpu().numpy(), out), maxerr(vg.cpu().numpy(), out))
    assert np.array_equal(vg.cpu().numpy()[:, kept == 0], v[:, kept == 0])


@pytest.mark.parametrize("ncells,w,r", [(1, 10, 8), (2, 12, 10)])
def test_rank_deficient_gappy_solve(orc, inputs, ncells, w, r):
    """H5 with fewer sampled rows than modes (c*|S-hat| < r_eff): G is singular, the solve takes
    the eigen route with the 1e-12 cut (A13) and returns the min-norm y; the filled state matches
    the oracle's min-norm LSQ (QR + SVD) step."""
    wl = small2d(inputs, w=w, r=r, nx=40, ny=30)
    snaps, _ = _replay_case(orc, inputs, wl, seed=11)
    S = np.zeros(wl.N, np.uint8)
    S[np.linspace(wl.N // 5, wl.N - wl.N // 5, ncells).astype(int)] = 1
    k = wl.w + 3
    R = orc.Run(wl, snaps[0])
    R.set_window(k, snaps, S)
    rom = H.HybridROM(wl)
    rom.set_window(k, dev(snaps.reshape(wl.w + 1, -1)), _mask_dev(wl, S))
    assert wl.c * ncells < rom.effective_rank()
    dt = orc.dt(wl, snaps[-1])
    R.step(dt)
    rom.hybrid_step(dt=dt)
    rom.sync()
    assert rom.debug_counters(10)[9] == 1  # eigen route taken
    assert close(rom.get_state().cpu().numpy(), R.state(), 1e-12), (rel(rom.get_state().cpu().numpy(), R.state()), maxerr(rom.get_state().cpu().numpy(), R.state()))


@pytest.mark.parametrize("seed", [1, 5])
def test_positivity_escalation(orc, inputs, seed):
    """O11: a hybrid state with rho <= 0 or p <= 0 is redone as a full step with the
    same dt, on the device; the window Gram row is then recomputed from the final state, so the
    next basis matches the oracle's (which refreshes from the escalated snapshot)."""
    wl = small2d(inputs, nx=40, ny=30, w=8, r=2)
    snaps = inputs.smooth_window(wl, wl.w + 1, seed=seed, amp=0.9)
    rng = np.random.default_rng(seed)
    S = (rng.random(wl.N) < 0.15).astype(np.uint8)
    k = wl.w + 3
    R = orc.Run(wl, snaps[0])
    R.set_window(k, snaps, S)
    dt = orc.dt(wl, snaps[-1])
    assert R.step(dt) == 2  # the oracle escalated
    rom = H.HybridROM(wl)
    rom.set_window(k, dev(snaps.reshape(wl.w + 1, -1)), _mask_dev(wl, S))
    before = rom.debug_counters(16)[15]
    rom.hybrid_step(dt=dt)
    rom.sync()  # the full step is admissible: nothing latched
    assert rom.debug_counters(16)[15] == before + 1
    full = orc.full_step(wl, snaps[-1], dt)
    assert close(rom.get_state().cpu().numpy(), full, 1e-13), (rel(rom.get_state().cpu().numpy(), full), maxerr(rom.get_state().cpu().numpy(), full))
    assert close(rom.get_state().cpu().numpy(), R.state(), 1e-13), (rel(rom.get_state().cpu().numpy(), R.state()), maxerr(rom.get_state().cpu().numpy(), R.state()))
    # basis of the window ending at the escalated snapshot
    rom.update_basis()
    lam = rom.eigenvalues().cpu().numpy()
    sig = R.sigma()
    re = R.reff()
    np.testing.assert_allclose(lam[:re], sig[:re] ** 2, rtol=1e-9, atol=1e-13 * sig[0] ** 2)


def test_empty_sample_set_fills_with_psi(orc, inputs):
    """S-hat = {} (all eps = 0, A18): no gappy rows, y = G^+ g = 0 and the whole state is
    psi_{k+1} + Phi*0; the oracle's min-norm LSQ of an empty system gives the same."""
    wl = small2d(inputs, bc=1, nx=48, ny=32)
    snaps, _ = _replay_case(orc, inputs, wl, seed=13)
    S = np.zeros(wl.N, np.uint8)
    k = wl.w + 2
    R = orc.Run(wl, snaps[0])
    R.set_window(k, snaps, S)
    dt = orc.dt(wl, snaps[-1])
    R.step(dt)
    rom = H.HybridROM(wl)
    rom.set_window(k, dev(snaps.reshape(wl.w + 1, -1)), _mask_dev(wl, S))
    rom.hybrid_step(dt=dt)
    rom.sync()
    g = rom.get_state().cpu().numpy()
    psi_next = snaps[1:].mean(axis=0)
    assert close(g, R.state(), 1e-13), (rel(g, R.state()), maxerr(g, R.state()))
    assert close(g, psi_next, 1e-13), (rel(g, psi_next), maxerr(g, psi_next))


def test_abi_argument_and_state_errors(inputs):
    """hrom.h error behaviour: invalid parameters are rejected at create, calls out of order
    return HROM_E_STATE, and a hybrid step before any basis is refused."""
    import dataclasses
    wl = small2d(inputs)
    with pytest.raises(H.HromError) as e:
        H.HybridROM(dataclasses.replace(wl, r=wl.w + 1))  # r > w
    assert e.value.code == 1
    with pytest.raises(H.HromError):
        H.HybridROM(dataclasses.replace(wl, f=0.0))  # fraction outside (0, 1]
    rom = H.HybridROM(wl)
    with pytest.raises(H.HromError) as e:
        rom.full_step()  # no state yet
    assert e.value.code == 2
    rom.set_state(dev(inputs.initial_condition(wl)))
    with pytest.raises(H.HromError) as e:
        rom.hybrid_step()  # no basis yet
    assert e.value.code == 2
    rom.full_step()
    rom.sync()


def test_trajectory_config2_short(orc, inputs):
    """Config 2 (BJ:8, 256^2 four-quadrant problem, MUSCL, transmissive): the Algorithm-1
    trajectory through the bootstrap and 8 hybrid steps agrees with the oracle step by step
    (the explicit map's rounding amplification is still small this early, G6)."""
    wl = inputs.config(2, steps=inputs.config(2).w + 8)
    q0 = inputs.initial_condition(wl)
    rom = H.HybridROM(wl)
    rom.set_state(dev(q0))
    R = orc.Run(wl, q0)
    worst = 0.0
    for k in range(1, wl.steps + 1):
        rom.step()
        R.step()
        gk = rom.get_state().cpu().numpy()
        e = max(rel(gk, R.state()), maxerr(gk, R.state()))
        worst = max(worst, e)
        if k >= wl.w - 1:
            assert np.array_equal(H.cells_from_mask(wl, rom.mask()), R.mask()), k
    rom.sync()
    assert worst <= 1e-11, worst


def _parallel_oracle(cfg, steps, nens, outdir):
    """Oracle reference, ensemble members and the full-HDM trajectory in concurrent processes
    (tests/traj_worker.py); returns memory-mapped arrays."""
    import concurrent.futures as cf
    import multiprocessing as mp
    import traj_worker
    jobs = [(-1, False)] + [(m, False) for m in range(nens)] + [(-1, True)]
    with cf.ProcessPoolExecutor(max_workers=len(jobs), mp_context=mp.get_context("spawn")) as ex:
        tags = [f.result() for f in [ex.submit(traj_worker.run_oracle, cfg, steps, m, str(outdir), h) for m, h in jobs]]
    load = lambda t, w: np.load(outdir / f"{t}_{w}.npy", mmap_mode="r")
    return {t: (load(t, "states"), load(t, "masks"), np.load(outdir / f"{t}_dts.npy")) for t in tags}


@pytest.mark.skipif(os.environ.get("HROM_SLOW_TESTS") != "1",
                    reason="~4 min of parallel oracle trajectories; HROM_SLOW_TESTS=1 (log: profiles/r2_pytest_gpu_full_12ae8a2.txt)")
def test_trajectory_config2_200(orc, inputs, tmp_path):
    """Config 2 (BJ:8, 256^2 four-quadrant, MUSCL) for 200 steps of Algorithm 1 against the
    oracle and an oracle ensemble from 1e-15-perturbed ICs (its own rounding sensitivity, G6):
    while the ensemble drift sref is < 1e-9 the GPU drift is <= 30 sref + 1e-13 and the masks are
    identical; every step the GPU state is physical; the method's accuracy against the full HDM
    (e-bar) is the oracle's within the ensemble's spread; lock-step replays at
    k = w, w+1, w+50, steps-1 (the GPU fed the oracle's window and mask) <= 1e-12."""
    steps = 200
    wl = inputs.config(2, steps=steps)
    T = _parallel_oracle(2, steps, 2, tmp_path)
    ref_s, ref_m, ref_dt = T["ref"]
    hdm = T["hdm"][0]
    ens = [T["ens0"][0], T["ens1"][0]]
    rom = H.HybridROM(wl)
    rom.set_state(dev(np.ascontiguousarray(ref_s[0])))
    e_gpu, e_ref, e_ens = [], [], [[], []]
    for k in range(1, steps + 1):
        rom.step()
        g = rom.get_state().cpu().numpy()
        o = np.asarray(ref_s[k])
        sref = max(rel(E[k], o) for E in ens)
        e = rel(g, o)
        assert np.all(g[0] > 0), k
        if sref < 1e-9:
            assert e <= 30 * sref + 1e-13, (k, e, sref)
            if k >= wl.w - 1:
                assert np.array_equal(H.cells_from_mask(wl, rom.mask()), np.asarray(ref_m[k])), k
        e_gpu.append(l1err(g, hdm[k]))
        e_ref.append(l1err(o, hdm[k]))
        for i, E in enumerate(ens):
            e_ens[i].append(l1err(E[k], hdm[k]))
    rom.sync()
    _ebar_check(e_gpu, e_ref, e_ens)
    for k in (wl.w, wl.w + 1, wl.w + 50, steps - 1):
        r2 = H.HybridROM(wl)
        win = np.ascontiguousarray(ref_s[k - wl.w:k + 1]).reshape(wl.w + 1, -1)
        r2.set_window(k, dev(win), _mask_dev(wl, np.asarray(ref_m[k])))
        r2.hybrid_step(dt=float(ref_dt[k + 1]))
        g = r2.get_state().cpu().numpy()
        assert close(g, ref_s[k + 1], 1e-12), ((k, rel(g, ref_s[k + 1])), maxerr(g, ref_s[k + 1]))
        r2.close()


def test_fullsize_config4_properties(orc, inputs):
    """Config 4 at full size (2048^2, BJ:10) in bench.py's launch configuration, checked where
    the oracle can follow: (i) S-hat rows of the hybrid step equal the oracle's full step there
    (exact restriction, Eq. 7); (ii) every cell outside S-hat (+) Q_W holds psi + Phi y
    with the GPU's own Phi, psi (lifted) and y; (iii) the next S-hat is bit-exactly the top
    ceil(fN) of the GPU's indicator, ties by ascending index (A18)."""
    wl = inputs.config(4)
    rom = H.HybridROM(wl)
    rom.set_state(dev(inputs.initial_condition(wl)))
    for _ in range(wl.w + 1):
        rom.step()
    g0 = rom.get_state().cpu().numpy()
    phi, psi = rom.basis()
    S = H.cells_from_mask(wl, rom.mask()).astype(bool)
    dtt = torch.zeros(1, dtype=torch.float64, device="cuda")
    rom.hybrid_step(dt_out=dtt)
    rom.sync()
    dt = float(dtt.item())
    g1 = rom.get_state()
    # (i) S-hat rows vs the oracle's full step (whole grid, ~8 s single-thread)
    full = orc.full_step(wl, g0, dt)
    g1n = g1.cpu().numpy()
    assert rel(g1n[:, S], full[:, S]) <= 1e-13
    # (ii) fill outside the seam band
    S2 = S.reshape(wl.ny, wl.nx)
    T2 = S2.copy()
    for dy in range(-wl.W, wl.W + 1):  # square dilation Q_W, periodic (A21)
        for dx in range(-wl.W, wl.W + 1):
            T2 |= np.roll(np.roll(S2, dy, 0), dx, 1)
    T = T2.reshape(-1)
    y = rom.y()[: phi.shape[0]]
    rec = (psi.reshape(-1) + phi.T @ y).reshape(wl.c, wl.N)
    off = torch.from_numpy(~T).cuda()
    num = torch.linalg.norm((g1 - rec)[:, off]).item()
    den = torch.linalg.norm(g1[:, off]).item()
    assert num / den <= 1e-12, num / den
    # (iii) next sample set
    eps = rom.indicator().cpu().numpy()
    rom.update_basis()
    rom.sample()
    nz = np.nonzero(eps > 0)[0]
    n_g = min(int(math.ceil(wl.f * wl.N)), nz.size)
    order = np.lexsort((nz, -eps[nz]))  # descending eps, ties by ascending cell
    want = np.zeros(wl.N, np.uint8)
    want[nz[order[:n_g]]] = 1
    assert np.array_equal(H.cells_from_mask(wl, rom.mask()), want)
    # (iv) the RRE-delta rule at full size on the same indicator (A35): bit-exact vs the oracle
    for delta in (0.5, 0.99, 0.999999):
        m_o, k_o = orc.select_rre(eps, delta)
        cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
        rom.sample_rre(delta, eps=dev(eps), count_out=cnt)
        assert np.array_equal(H.cells_from_mask(wl, rom.mask()), m_o), delta
        assert int(cnt.item()) == k_o


def test_fullsize_gram_config5_rows(orc, inputs):
    """H10/K11 DMMA Gram over config 5's full row count (D = 4 x 4096^2 = 67 M rows, BJ:11) for 8
    columns shifted by a reference, vs the oracle's compensated Gram.  Tolerance: each CTA
    accumulates ~7 K tile products sequentially, so |C_gpu - C| <= ~n_tiles eps sum|s_i s_j|;
    1e-12 max|C| holds with margin for these O(1) shifted columns."""
    rows = 4 * 4096 * 4096
    ncol = 8
    S = inputs.random_values(501, ncol * rows, 0.5, 1.5).reshape(ncol, rows)
    rho = S.mean(axis=0)
    wl = small2d(inputs)
    rom = H.HybridROM(wl)
    Sd = dev(S)
    Cg = rom.gram(Sd, dev(rho)).cpu().numpy()
    del Sd
    Co = orc.gram(S, rho)
    assert np.max(np.abs(Cg - Co)) <= 1e-12 * np.max(np.abs(Co)), np.max(np.abs(Cg - Co)) / np.max(np.abs(Co))


@pytest.mark.parametrize("cfg", [2, 4])
def test_incremental_gathered_gram_matches_full(inputs, cfg):
    """G7: the gathered Gram updated from the previous step (S-hat churn rows, newest snapshot
    and HDM columns, double-double accumulation) gives the same hybrid steps as recomputing it
    over all S-hat rows: lock-step contexts from the same IC, relative L2 <= 1e-12 over the first
    hybrid steps (config 2 churns ~35 % of S-hat per step, config 4 ~1 %).  Later the two
    trajectories separate at the method's own rounding amplification (G6), so the check stops
    after a few steps."""
    wl = inputs.config(cfg)
    steps = wl.w + 4 if cfg == 2 else wl.w + 8
    q0 = dev(inputs.initial_condition(wl))
    a = H.HybridROM(wl, gather_mode=0)
    b = H.HybridROM(wl, gather_mode=1)
    a.set_state(q0)
    b.set_state(q0)
    worst = 0.0
    for k in range(1, steps + 1):
        a.step()
        b.step()
        ga, gb = a.get_state(), b.get_state()
        worst = max(worst, (torch.linalg.norm(ga - gb) / torch.linalg.norm(gb)).item())
    a.sync()
    b.sync()
    assert worst <= 1e-12, worst


# ---- Algorithm 1 with a finite full-HDM period z ----

@pytest.mark.parametrize("cfg", [1, 2])
def test_z1_is_the_full_hdm_bitwise(inputs, cfg):
    """z = 1 makes every step a full HDM step, bitwise equal to hrom_full_step."""
    wl = inputs.config(cfg, z=1)
    q0 = dev(inputs.initial_condition(wl))
    a, b = H.HybridROM(wl), H.HybridROM(wl)
    a.set_state(q0)
    b.set_state(q0)
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(wl.w + 6):
        a.step(count_out=cnt)
        b.full_step()
        assert int(cnt.item()) == wl.N
        assert torch.equal(a.get_state(), b.get_state())
    a.sync()
    b.sync()


def test_trajectory_finite_z_config2(orc, inputs):
    """Config 2 with z = 4 (w = 32): the bootstrap refresh is skipped ((w) mod 4 = 0), step 32
    is full, refreshes after full steps use the projection indicator (G8), the refresh before
    each full step is skipped and its window-Gram row is owed to the next update.  Step by step
    the GPU state and S-hat agree with the oracle, and the per-step sample counts are N on
    full steps and |S-hat| on hybrid steps (s-bar, s-bar* of P:715-727)."""
    z = 4
    wl = inputs.config(2, steps=inputs.config(2).w + 14, z=z)
    q0 = inputs.initial_condition(wl)
    rom = H.HybridROM(wl)
    rom.set_state(dev(q0))
    R = orc.Run(wl, q0)
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    worst = 0.0
    kinds = []
    for k in range(1, wl.steps + 1):
        rom.step(count_out=cnt)
        kind = R.step()
        kinds.append(kind)
        full = k + 1 <= wl.w or k % z == 0
        assert (kind == 0) == full
        n = int(cnt.item())
        assert n == (wl.N if full else int(R.mask_used().sum())), (k, n)
        gk = rom.get_state().cpu().numpy()
        e = max(rel(gk, R.state()), maxerr(gk, R.state()))
        worst = max(worst, e)
        if k >= wl.w and (k + 1) % z != 0:
            assert np.array_equal(H.cells_from_mask(wl, rom.mask()), R.mask()), k
            if full:  # projection indicator after a full step (G8)
                eg, eo = rom.indicator().cpu().numpy(), R.eps()
                np.testing.assert_allclose(eg, eo, rtol=1e-6, atol=1e-9 * eo.max())
    rom.sync()
    assert kinds.count(1) + kinds.count(2) >= 8
    assert worst <= 1e-11, worst


def test_rel_l1_error_matches_definition(inputs):
    """e_k of P:704-709 (uniform cells): sum |a - b| / sum |b| over the D entries."""
    wl = small2d(inputs, nx=333, ny=129)
    rom = H.HybridROM(wl)
    rng = np.random.default_rng(3)
    a = rng.standard_normal((wl.c, wl.N))
    b = a + 1e-3 * rng.standard_normal((wl.c, wl.N))
    e = rom.rel_l1_error(dev(a), dev(b))
    ref = np.abs(a - b).sum() / np.abs(b).sum()
    assert abs(e - ref) <= 1e-13 * ref
    assert rom.rel_l1_error(dev(b), dev(b)) == 0.0
    assert rom.rel_l1_error(dev(a), dev(b)) == e  # bitwise reproducible


def test_algorithm1_metrics_driver(inputs):
    """e_k, e-bar, s-bar, s-bar*, p-bar, S from the device driver."""
    from paper_2301_01718_b200 import algorithm1 as A1
    wl = inputs.config(1)
    m = A1.run(wl, steps=60, z=7)
    assert len(m.e) == 60 and len(m.n_gamma) == 60
    # warm-up full steps are the HDM itself: e_k = 0 exactly
    assert all(e == 0.0 for e in m.e[: wl.w - 1])
    for k in range(1, 61):
        full = k + 1 <= wl.w or k % 7 == 0
        assert m.hybrid[k - 1] == (not full)
        if full:
            assert m.n_gamma[k - 1] == wl.N
        else:
            assert 0 < m.n_gamma[k - 1] <= math.ceil(wl.f * wl.N)
    assert 0.0 < m.e_bar < 0.1
    assert m.s_bar_star is not None and m.s_bar_star < m.s_bar < wl.N
    assert m.p_bar == 0.0 and m.speedup > 0.0
    s = m.summary()
    assert s["hybrid_steps"] == sum(m.hybrid)


def _rre_cases(rng, N):
    """Indicator vectors for the RRE-delta rule: ties + zeros, wide exponents incl. subnormals
    and values near DBL_MAX, all-zero, and deltas exactly on a prefix ratio."""
    out = []
    e = np.round(rng.random(N) * 50) / 50.0 * (rng.random(N) < 0.4)
    for d in (0.3, 0.9, 0.999, 1.0):
        out.append((e, d))
    e = rng.random(N) * 2.0 ** rng.integers(-1074, 1000, N).astype(float)
    e[rng.random(N) < 0.3] = 0.0
    e[10:40] = e[5]  # ties
    for d in (1e-300, 0.5, 0.999999, 1.0):
        out.append((e, d))
    e = rng.random(N) * 2.0 ** rng.integers(-30, 0, N).astype(float)  # a realistic spread
    out.append((e, 0.99))
    e = np.zeros(N)
    e[[3, 77]] = [1.0, 3.0]
    out.append((e, 0.75))  # exactly RRE(1) = 3/4 -> one cell
    e = np.zeros(N)
    e[[1, 2, 900, 901, 5000]] = 2.0 ** -1074
    out.append((e, 0.5))   # tied subnormals: ceil(2.5) = 3 cells, lowest indices
    e = np.zeros(N)
    e[[0, 1, N - 1]] = [1e308, 1e308, 1e-308]
    out.append((e, 1.0))
    out.append((np.zeros(N), 0.5))
    return out


@pytest.mark.parametrize("nx,ny", [(130, 77), (1024, 1024)])
def test_sample_rre_bit_exact(orc, inputs, nx, ny):
    """H8 with the RRE-delta rule fed the same indicator as the oracle: S-hat,
    its ascending list and n_g bit-exact; the sums are exact on both sides (reading A35)."""
    wl = small2d(inputs, nx=nx, ny=ny, bc=1)
    rom = H.HybridROM(wl)
    rom.set_state(dev(inputs.initial_condition(wl, "random")))
    rng = np.random.default_rng(11)
    mw = torch.zeros(rom.mask_words, dtype=torch.int32, device="cuda")
    lst = torch.zeros(wl.N, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    for t, (eps, delta) in enumerate(_rre_cases(rng, wl.N)):
        m_o, k_o = orc.select_rre(eps, delta)
        rom.sample_rre(delta, eps=dev(eps), mask_out=mw, list_out=lst, count_out=cnt)
        torch.cuda.synchronize()
        assert np.array_equal(H.cells_from_mask(wl, mw), m_o), (t, delta)
        n = int(cnt.item())
        assert n == k_o, (t, delta, n, k_o)
        assert np.array_equal(lst[:n].cpu().numpy(), np.nonzero(m_o)[0])
    with pytest.raises(H.HromError):
        rom.sample_rre(0.0)
    with pytest.raises(H.HromError):
        rom.sample_rre(1.5)


def test_trajectory_rre_config2(orc, inputs):
    """Algorithm 1 on config 2 with the RRE-delta selection (delta = 0.99) instead of
    the fixed fraction: step by step, S-hat identical to the oracle's and state <= 1e-11."""
    wl = inputs.config(2, steps=inputs.config(2).w + 6, delta=0.99)
    q0 = inputs.initial_condition(wl)
    rom = H.HybridROM(wl)
    rom.set_state(dev(q0))
    R = orc.Run(wl, q0)
    worst = 0.0
    sizes = []
    for k in range(1, wl.steps + 1):
        rom.step()
        R.step()
        gk = rom.get_state().cpu().numpy()
        worst = max(worst, rel(gk, R.state()), maxerr(gk, R.state()))
        if k >= wl.w - 1:
            m_o = R.mask()
            assert np.array_equal(H.cells_from_mask(wl, rom.mask()), m_o), k
            sizes.append(int(m_o.sum()))
    rom.sync()
    assert all(0 < s < wl.N // 4 for s in sizes), sizes
    assert worst <= 1e-11, worst


@pytest.mark.parametrize("dim,nx,ny,bc,frac,seed", [(2, 70, 45, 0, 0.1, 7), (2, 64, 64, 1, 0.3, 8),
                                                    (1, 3000, 1, 0, 0.05, 9)])
def test_whole_domain_filter_parity(orc, inputs, dim, nx, ny, bc, frac, seed):
    """W = -1 (the paper's filter over the whole hybrid state; NEXT-2): every cell off
    S-hat is filtered; kept set and sweeps identical to the oracle, values to rounding."""
    wl = small2d(inputs, dim=dim, nx=nx, ny=ny, bc=bc, seed=seed, W=-1)
    rng = np.random.default_rng(seed)
    F = inputs.initial_condition(wl, "random")
    v = F * (1.0 + 0.05 * rng.standard_normal(F.shape))
    S = (rng.random(wl.N) < frac).astype(np.uint8)
    v[:, S == 1] = F[:, S == 1]
    out, kept, sweeps = orc.seam_filter(wl, v, F, S)
    rom = H.HybridROM(wl)
    vg = dev(v)
    kg = torch.zeros(wl.N, dtype=torch.uint8, device="cuda")
    rom.filter(vg, dev(F), _mask_dev(wl, S), kept_out=kg)
    rom.sync()
    assert np.array_equal(kg.cpu().numpy(), kept)
    assert kept.sum() > 0 and kept[S == 1].sum() == 0
    cnt = rom.debug_counters(8)
    assert list(cnt[4:4 + len(sweeps)]) == list(sweeps)
    assert close(vg.cpu().numpy(), out, 1e-14), (rel(vg.cpu().numpy(), out), maxerr(vg.cpu().numpy(), out))


def test_whole_domain_filter_nyquist_gpu(inputs):
    """Closed form (as the oracle pin): constant + exact checkerboard, periodic, S-hat empty,
    W = -1: the order-2 sweep returns the constant bit for bit on every cell."""
    wl = small2d(inputs, nx=64, ny=40, bc=1, W=-1)
    F = np.empty((wl.c, wl.N))
    F[:] = np.array([1.0, 0.25, -0.5, 2.5])[:, None]
    i, j = np.meshgrid(np.arange(wl.nx), np.arange(wl.ny))
    cb = ((-1.0) ** (i + j)).reshape(-1)
    v = F + np.array([2.0 ** -10, 2.0 ** -9, 2.0 ** -8, 2.0 ** -7])[:, None] * cb[None, :]
    rom = H.HybridROM(wl)
    vg = dev(v)
    kg = torch.zeros(wl.N, dtype=torch.uint8, device="cuda")
    rom.filter(vg, dev(F), _mask_dev(wl, np.zeros(wl.N, np.uint8)), kept_out=kg)
    rom.sync()
    assert np.array_equal(vg.cpu().numpy(), F)
    assert int(kg.sum().item()) == wl.N
    assert int(rom.debug_counters(8)[4]) == 2


def test_trajectory_whole_domain_filter_config2(orc, inputs):
    """Algorithm 1 on config 2 with the whole-domain filter (W = -1): S-hat identical to the
    oracle's and state <= 1e-11 step by step."""
    wl = inputs.config(2, steps=inputs.config(2).w + 4, W=-1)
    q0 = inputs.initial_condition(wl)
    rom = H.HybridROM(wl)
    rom.set_state(dev(q0))
    R = orc.Run(wl, q0)
    worst = 0.0
    for k in range(1, wl.steps + 1):
        rom.step()
        R.step()
        gk = rom.get_state().cpu().numpy()
        worst = max(worst, rel(gk, R.state()), maxerr(gk, R.state()))
        if k >= wl.w - 1:
            assert np.array_equal(H.cells_from_mask(wl, rom.mask()), R.mask()), k
    rom.sync()
    assert worst <= 1e-11, worst


@pytest.mark.parametrize("kind", ["random", "pod"])
def test_odeim_points_parity(orc, inputs, kind):
    """NEXT-1 ODEIM points (Eq. 10, reading A36) on the device vs the oracle, both fed
    the same basis: identical points (cells and DOF rows, in selection order) for n_p = m (DEIM)
    and n_p = 2m + 3 (oversampling, the SPEC default 2m plus a ragged cycle)."""
    wl = small2d(inputs, nx=70, ny=45)
    if kind == "random":
        rng = np.random.default_rng(12)
        Q, _ = np.linalg.qr(rng.standard_normal((wl.D, 12)))
        phi = np.ascontiguousarray(Q.T)
    else:  # the oracle's POD basis of a smooth window (modes localised like the solver's)
        snaps, S = _replay_case(orc, inputs, wl)
        R = orc.Run(wl, snaps[0])
        R.set_window(wl.w + 5, snaps, S)
        phi = np.ascontiguousarray(R.basis().T)
    m = phi.shape[0]
    rom = H.HybridROM(wl)
    for n_p in (m, 2 * m + 3):
        co, ro = orc.odeim(phi, wl.N, n_p)
        cg, rg = rom.odeim(dev(phi), n_p)
        torch.cuda.synchronize()
        assert np.array_equal(rg.cpu().numpy(), ro), (n_p, rg.cpu().numpy()[:8], ro[:8])
        assert np.array_equal(cg.cpu().numpy(), co)
    with pytest.raises(H.HromError):
        rom.odeim(dev(phi), wl.N + 1)


@pytest.mark.parametrize("kw", [dict(n_p=10), dict(n_p=13, bc=1, nx=64, ny=40), dict(dim=1, nx=500, ny=1, recon=1, w=12,
                                                                                   r=6, n_p=12)],
                         ids=["2d", "2d-periodic", "1d"])
def test_hybrid_step_replay_odeim(orc, inputs, kw):
    """Algorithm 1 with ODEIM points (NEXT-1): the given mask is G, S-hat = G u P with
    P = ODEIM(Phi_{k+1}); the gappy rows are the points' DOF rows (Eq. 8).  Same S-hat and the
    same hybrid step as the oracle (<= 1e-12)."""
    wl = small2d(inputs, **kw)
    snaps, S = _replay_case(orc, inputs, wl, frac=0.05)
    k = wl.w + 5
    R = orc.Run(wl, snaps[0])
    R.set_window(k, snaps, S)
    rom = H.HybridROM(wl)
    rom.set_window(k, dev(snaps.reshape(wl.w + 1, -1)), _mask_dev(wl, S))
    mo = R.mask()
    assert mo.sum() > S.sum()  # the points add cells
    assert np.array_equal(H.cells_from_mask(wl, rom.mask()), mo)
    dt = orc.dt(wl, snaps[-1])
    R.step(dt)
    rom.hybrid_step(dt=dt)
    rom.sync()
    assert close(rom.get_state().cpu().numpy(), R.state(), 1e-12), (rel(rom.get_state().cpu().numpy(), R.state()), maxerr(rom.get_state().cpu().numpy(), R.state()))


def test_trajectory_odeim_config1(orc, inputs):
    """Config 1 with ODEIM points (n_p = 2r = 20, the SPEC default) added to the fraction rule:
    S-hat identical to the oracle's and state <= 1e-11 step by step."""
    wl = inputs.config(1, steps=inputs.config(1).w + 20, n_p=20)
    q0 = inputs.initial_condition(wl)
    rom = H.HybridROM(wl)
    rom.set_state(dev(q0))
    R = orc.Run(wl, q0)
    worst = 0.0
    for k in range(1, wl.steps + 1):
        rom.step()
        R.step()
        gk = rom.get_state().cpu().numpy()
        worst = max(worst, rel(gk, R.state()), maxerr(gk, R.state()))
        if k >= wl.w - 1:
            assert np.array_equal(H.cells_from_mask(wl, rom.mask()), R.mask()), k
    rom.sync()
    assert worst <= 1e-11, worst


@pytest.mark.parametrize("kw", [dict(), dict(w=32, r=16, nx=40, ny=30), dict(w=48, r=24, nx=33, ny=20)],
                         ids=["w8-r5", "w32-r16", "w48-r24"])
def test_project_window_dmma(orc, inputs, kw):
    """Config-5 kernel op Phi^T S on FP64 tensor cores vs the oracle's
    orc_project (compensated sums of the definition), <= 1e-13 relative (max element)."""
    wl = small2d(inputs, **kw)
    snaps, S = _replay_case(orc, inputs, wl)
    rom = H.HybridROM(wl)
    rom.set_window(wl.w + 5, dev(snaps.reshape(wl.w + 1, -1)), _mask_dev(wl, S))
    rng = np.random.default_rng(4)
    m = min(wl.r, 16 if wl.w < 48 else 24)
    phi = rng.standard_normal((m, wl.D))
    C = rom.project(dev(phi)).cpu().numpy()
    ref = orc.project(phi, snaps.reshape(wl.w + 1, -1))
    assert np.max(np.abs(C - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_determinism_bitwise_config4(inputs):
    """Two config-4 runs (2048^2, w + 4 steps: full warm-up, bootstrap, hybrid steps with seam
    bands spread over ~150 CTAs) are bitwise identical: fixed-order reductions, order-free atomics,
    and no cross-CTA read-after-write races (the filter's alternating x-pass buffers)."""
    wl = inputs.config(4)
    q0 = dev(inputs.initial_condition(wl))
    out = []
    for _ in range(2):
        rom = H.HybridROM(wl)
        rom.set_state(q0)
        for _ in range(wl.w + 4):
            rom.step()
        rom.sync()
        out.append((rom.get_state().cpu().numpy(), H.cells_from_mask(wl, rom.mask())))
        rom.close()
        torch.cuda.empty_cache()
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])


def test_interleaved_contexts_bitwise_repeated(inputs):
    """Two contexts stepped alternately without any host synchronisation (their kernels and
    side-stream eigen-solves overlap, so the shared-memory contents a block finds vary from run to
    run), 12 times over: every step's state, S-hat, indicator, y and eigenvalues, captured on the
    streams, are bit-identical.  (Regression: the inverse iteration's back substitution once read
    two never-written shared-memory entries multiplied by zero; a NaN pattern left there by another
    kernel changed the basis at rounding level in ~10 % of such runs.)"""
    wl = inputs.config(2)
    steps = wl.w + 40
    q0 = dev(inputs.initial_condition(wl))

    def grab(rom):
        y = torch.zeros(wl.r, dtype=torch.float64, device="cuda")
        rom.lib.hrom_get_y(rom.h, y.data_ptr())
        lam = torch.zeros(wl.w, dtype=torch.float64, device="cuda")
        rom.lib.hrom_debug_read(rom.h, 5, lam.data_ptr(), wl.w)
        return [rom.get_state().clone(), rom.mask().clone(), rom.indicator().clone(), y, lam]

    for run in range(12):
        a, b = H.HybridROM(wl), H.HybridROM(wl)
        a.set_state(q0)
        b.set_state(q0)
        ra, rb = [], []
        for _ in range(steps):
            a.step()
            b.step()
            if a.k >= wl.w:
                ra.append(grab(a))
                rb.append(grab(b))
        a.sync()
        b.sync()
        for k, (x, z) in enumerate(zip(ra, rb)):
            for name, p_, q_ in zip(("state", "mask", "eps", "y", "lam"), x, z):
                assert torch.equal(p_, q_), (run, k + wl.w, name)
        a.close()
        b.close()


@pytest.mark.parametrize("cfg", [1, 2])
def test_graph_replay_bitwise(inputs, cfg):
    """NEXT-3: steady-state steps replayed from per-ring-phase CUDA graphs (hrom_set_graph) give
    the eager trajectory bit for bit -- state, S-hat and indicator -- over more than two ring
    periods (every phase captured once, then replayed)."""
    wl = inputs.config(cfg)
    steps = wl.w + 2 * (wl.w + 2) + 7
    q0 = dev(inputs.initial_condition(wl))
    a = H.HybridROM(wl)
    b = H.HybridROM(wl)
    b.set_graph(True)
    a.set_state(q0)
    b.set_state(q0)
    for k in range(1, steps + 1):
        a.step()
        b.step()
        if k % 17 == 0 or k == steps:
            assert torch.equal(a.get_state(), b.get_state()), k
            assert torch.equal(a.mask(), b.mask()), k
            assert torch.equal(a.indicator(), b.indicator()), k
    a.sync()
    b.sync()
    assert b.graph_launches() >= steps - wl.w - 4
    assert a.k == b.k == steps


def test_concurrent_contexts_bitwise(inputs):
    """Race evidence without compute-sanitizer (closed on this pool): three contexts of config 2
    on three streams run concurrently (their cooperative kernels, mbarrier pipelines and grid
    barriers interleave on the SMs, so every timing-dependent hazard gets a different schedule)
    and a fourth alone; all four end bitwise identical (state, S-hat, indicator)."""
    wl = inputs.config(2)
    q0 = dev(inputs.initial_condition(wl))
    steps = wl.w + 24
    streams = [torch.cuda.Stream() for _ in range(3)]
    roms = [H.HybridROM(wl, stream=s_) for s_ in streams]
    for r_ in roms:
        r_.set_state(q0)
    torch.cuda.synchronize()
    for _ in range(steps):
        for r_ in roms:  # enqueue round-robin: the three streams overlap on the device
            r_.step()
    alone = H.HybridROM(wl)
    alone.set_state(q0)
    for _ in range(steps):
        alone.step()
        alone.sync()
    for r_ in roms:
        r_.sync()
    ref = (alone.get_state(), alone.mask(), alone.indicator())
    for r_ in roms:
        got = (r_.get_state(), r_.mask(), r_.indicator())
        for x, y in zip(got, ref):
            assert torch.equal(x.cpu(), y.cpu())
