"""GPU parity at the oracle's own accuracy (G11): full-size config-3 replays and
config-4-parameter replays (w = 64, r = 32: fill_kernel<34> with its double-double Gram row)
against the oracle, element by element.

Bars (BASELINE.json north_star, BJ:5): per-step state <= max(1e-12, 10 eps sigma_1 / gap_sigma),
where eps sigma_1 / gap_sigma (gap_sigma = sigma_reff - sigma_reff+1) is the conditioning of the
SVD's POD_m itself (A15), i.e. what the oracle's own QR + Jacobi SVD guarantees; per-element
max error on the same bar; indicator eps to <= 1e-9 relative; masks bit-exact when both sides are
fed the oracle's indicator, and the GPU's own selection equal to the oracle's except for cells
whose indicator lies within 1e-12 (relative) of the selection threshold.
"""
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2301_01718_b200 import hrom as H  # noqa: E402

EPS = 2.220446049250313e-16
# the full replay set (k in {w, w+1, w+50} at configs 3 and 4, and the 2048^2 config-4 step whose
# single-threaded oracle POD takes ~18 min) runs with HROM_SLOW_TESTS=1; the default GPU suite
# keeps one replay per config (k = w + 1).  Full-set log: profiles/r2_pytest_gpu_full_12ae8a2.txt
SLOW = os.environ.get("HROM_SLOW_TESTS") == "1"
K_OFFS = [0, 1, 50] if SLOW else [1]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def maxerr(a, b):
    """Per-element max error relative to the largest entry of each variable's field."""
    a = np.asarray(a).reshape(b.shape)
    scale = np.max(np.abs(b), axis=-1, keepdims=True)
    return float(np.max(np.abs(a - b) / np.maximum(scale, 1e-300)))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def svd_bar(sig, reff):
    """max(1e-12, 10 eps sigma_1 / gap_sigma) for the POD of this window (A15)."""
    s_next = sig[reff] if reff < sig.size else 0.0
    gap = sig[reff - 1] - s_next
    return max(1e-12, 10 * EPS * sig[0] / max(gap, 1e-300))


def near_threshold(eps, n_g, tol=1e-12):
    """Cells whose indicator lies within tol (relative) of the top-n_g threshold."""
    pos = eps[eps > 0]
    if n_g <= 0 or pos.size <= n_g:
        return np.zeros(eps.size, bool)
    thr = np.sort(pos)[::-1][n_g - 1]
    return np.abs(eps - thr) <= tol * thr


_TRAJ = {}


def hdm_trajectory(orc, inputs, cfg, steps, **kw):
    """Oracle full-HDM snapshots gamma_0..gamma_steps (the replay windows), cached per module."""
    key = (cfg, steps, tuple(sorted(kw.items())))
    if key not in _TRAJ:
        wl = inputs.config(cfg, **kw)
        q = inputs.initial_condition(wl)
        snaps = [q]
        for _ in range(steps):
            snaps.append(orc.full_step(wl, snaps[-1], orc.dt(wl, snaps[-1])))
        _TRAJ[key] = (wl, np.stack(snaps))
    return _TRAJ[key]


def replay(orc, inputs, wl, snaps, k, S, steps=1):
    """Window gamma_{k-w}..gamma_k and S-hat_{k+1} = S on both sides, then `steps` hybrid steps
    (the GPU fed the oracle's next mask from the second step on).  Returns per-step records."""
    win = snaps[k - wl.w:k + 1]
    R = orc.Run(wl, win[0])
    R.set_window(k, win, S)
    rom = H.HybridROM(wl)
    rom.set_window(k, dev(win.reshape(wl.w + 1, -1)), H.mask_from_cells(wl, S))
    assert rom.effective_rank() == R.reff()
    out = []
    for st in range(steps):
        sig = R.sigma()
        bar = svd_bar(sig, R.reff())
        dt = orc.dt(wl, R.state())  # the oracle's current state (gamma_k at st = 0)
        mask_o = R.mask()
        R.step(dt)
        rom.hybrid_step(None if st == 0 else H.mask_from_cells(wl, mask_o), dt=dt)
        rom.sync()
        g = rom.get_state().cpu().numpy()
        o = R.state()
        out.append(dict(g=g, o=o, bar=bar, eg=rom.indicator().cpu().numpy(), eo=R.eps(), mask_o_next=R.mask(),
                        rom=rom, R=R))
        if st + 1 < steps:
            rom.update_basis()
            assert rom.effective_rank() == R.reff()
    return out


def check_step(rec, wl, orc, S_used):
    g, o, bar = rec["g"], rec["o"], rec["bar"]
    e_rel, e_max = rel(g, o), maxerr(g, o)
    assert e_rel <= bar, (e_rel, bar)
    assert e_max <= bar, (e_max, bar)
    eg, eo = rec["eg"], rec["eo"]
    # indicator: globally and per element to 1e-9; a cell may be zero on one side only
    # where its value is at the rounding level (kept-or-not filter decisions of cells whose
    # residual is rounding noise, A23')
    assert rel(eg, eo) <= 1e-9, rel(eg, eo)
    assert np.max(np.abs(eg - eo)) <= 1e-9 * np.max(eo), np.max(np.abs(eg - eo)) / np.max(eo)
    flip = (eg > 0) ^ (eo > 0)
    assert np.all(np.maximum(eg, eo)[flip] <= 1e-20 * np.max(eo)), np.max(np.maximum(eg, eo)[flip])
    return e_rel, e_max


@pytest.mark.parametrize("k_off", K_OFFS)
def test_replay_config3_fullsize(orc, inputs, k_off):
    """Config 3 at full size (1024^2, w = 48, r = 24, BJ:9): the window gamma_{k-w}..gamma_k from
    the oracle's full steps, S-hat = a seeded 10 % of the cells, one hybrid step on both sides
    (Alg. 1) at k = w + k_off.  State within the SVD-class bar, per-element and global;
    indicator to 1e-9; next S-hat: bit-exact when the GPU is fed the oracle's indicator, and from
    its own indicator equal to the oracle's mask off the threshold's 1e-12 neighbourhood."""
    wl0 = inputs.config(3)
    wl, snaps = hdm_trajectory(orc, inputs, 3, wl0.w + max(K_OFFS))
    k = wl.w + k_off
    S = (np.random.default_rng(33 + k_off).random(wl.N) < wl.f).astype(np.uint8)
    rec = replay(orc, inputs, wl, snaps, k, S)[0]
    check_step(rec, wl, orc, S)
    full = orc.full_step(wl, snaps[k], orc.dt(wl, snaps[k]))
    assert rel(rec["g"][:, S == 1], full[:, S == 1]) <= 1e-13
    rom = rec["rom"]
    n_g = orc.n_g(wl.f, wl.N)
    rom.update_basis()
    rom.sample(eps=dev(rec["eo"]))
    m_o, _ = orc.select(rec["eo"], n_g)
    assert np.array_equal(H.cells_from_mask(wl, rom.mask()), m_o)
    rom.sample(eps=dev(rec["eg"]))
    mg = H.cells_from_mask(wl, rom.mask())
    diff = mg != m_o
    assert not np.any(diff & ~near_threshold(rec["eo"], n_g)), int((diff & ~near_threshold(rec["eo"], n_g)).sum())


@pytest.mark.parametrize("k_off", K_OFFS)
def test_replay_config4_params_512(orc, inputs, k_off):
    """Config-4 parameters (periodic blasts, w = 64, r = 32, f = 10 %, BJ:10) on a 512^2 grid:
    the headline instantiation fill_kernel<34> (w + 2 = 66 ring slots) with its fused
    double-double Gram row.  Two hybrid steps from the oracle's window at k = w + k_off: the
    second step's basis is built from the first step's fused row, so the row is checked
    against the oracle too (the GPU is fed the oracle's next mask)."""
    wl, snaps = hdm_trajectory(orc, inputs, 4, inputs.config(4).w + max(K_OFFS) + 1, nx=512, ny=512)
    k = wl.w + k_off
    S = (np.random.default_rng(44 + k_off).random(wl.N) < wl.f).astype(np.uint8)
    recs = replay(orc, inputs, wl, snaps, k, S, steps=2)
    for rec in recs:
        check_step(rec, wl, orc, S)


@pytest.mark.skipif(not SLOW, reason="~18 min of single-threaded oracle POD; HROM_SLOW_TESTS=1")
def test_fullsize_config4_replay_step(orc, inputs):
    """One config-4 hybrid step at full size (2048^2, w = 64, r = 32, f = 10 %) in bench.py's
    launch configuration against the oracle: window = the shared generator's smooth blast-like
    columns (a full-HDM oracle window would cost ~9 min of single-thread full steps), seeded
    10 % S-hat.  State per element and globally within the SVD-class bar."""
    wl = inputs.config(4)
    snaps = inputs.smooth_window(wl, wl.w + 1, seed=404, amp=0.03)
    S = (np.random.default_rng(404).random(wl.N) < wl.f).astype(np.uint8)
    rec = replay(orc, inputs, wl, snaps, wl.w, S)[0]
    g, o, bar = rec["g"], rec["o"], rec["bar"]
    assert rel(g, o) <= bar, (rel(g, o), bar)
    assert maxerr(g, o) <= bar, (maxerr(g, o), bar)
