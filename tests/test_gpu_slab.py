"""Row-slab sharding of one problem (include/hrom.h hrom_slab_*), on ONE GPU: the
slabs are separate contexts of this process that exchange messages by plain device copies
(LocalComm), no kernel of one context ever waits on another.  Compared with the unsharded
context on the same seeded input:

* full steps (H1, H2 + halo exchange): bitwise;
* Algorithm 1 with hybrid steps (H3-H12): the state within the double-double reduction-order
  difference (1e-13 relative, per element), S-hat bit for bit, y and the eigenvalues to 1e-10;
* the replicated quantities (y, eigenvalues) bitwise identical on every rank;
* the distributed top-n_g selection against the unsharded hrom_sample on the same indicator;
* against the ORACLE: the sharded trajectory within the unsharded path's own tolerance.
"""
import dataclasses

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _mk(inputs, cfg, nranks, filt=False, **over):
    from paper_2301_01718_b200.hrom import HybridROM
    from paper_2301_01718_b200 import slab
    wl = inputs.config(cfg, **over)
    if not filt:
        wl = dataclasses.replace(wl, filter_orders=())
    q0 = torch.from_numpy(inputs.initial_condition(wl)).cuda()
    ref = HybridROM(wl, gather_mode=1)
    ref.set_state(q0)
    roms = [slab.SlabROM(wl, r, nranks) for r in range(nranks)]
    for r in roms:
        r.set_state(q0)
    return wl, q0, ref, roms, slab.LocalComm(nranks)


@pytest.mark.parametrize("cfg,nx,ny,nranks", [(2, 96, 80, 2), (4, 128, 96, 2), (4, 128, 120, 3), (2, 70, 50, 1),
                                              (4, 70, 100, 3), (2, 45, 101, 4)])
def test_slab_full_steps_bitwise(inputs, cfg, nx, ny, nranks):
    """Warm-up HDM steps: dt from the all-reduced CFL maximum, local RK3 on [halo | own | halo], halo
    exchange -> every own row equals the unsharded step bit for bit (transmissive and periodic)."""
    from paper_2301_01718_b200 import slab
    wl, q0, ref, roms, comm = _mk(inputs, cfg, nranks, nx=nx, ny=ny, w=12, r=6)
    assert sum(int(r.info.rows_own) for r in roms) == ny
    for _ in range(wl.w - 2):
        ref.step()
        slab.step_all(roms, comm)
    ref.sync()
    for r in roms:
        r.sync()
    a = ref.get_state().cpu().numpy()
    b = slab.assemble(roms, "state").cpu().numpy()
    assert np.array_equal(a, b)


@pytest.mark.parametrize("filt", [False, True])
@pytest.mark.parametrize("cfg,nx,ny,nranks,w,r", [(2, 96, 96, 2, 8, 4), (4, 128, 128, 2, 12, 6), (4, 128, 144, 3, 8, 4),
                                                   (4, 64, 64, 1, 8, 4), (4, 70, 100, 3, 8, 4), (2, 45, 101, 4, 10, 5)])
def test_slab_algorithm1_matches_unsharded(inputs, cfg, nx, ny, nranks, w, r, filt):
    from paper_2301_01718_b200 import slab
    from paper_2301_01718_b200.hrom import cells_from_mask
    wl, q0, ref, roms, comm = _mk(inputs, cfg, nranks, filt=filt, nx=nx, ny=ny, w=w, r=r)
    nsteps = w + 6
    for k in range(1, nsteps + 1):
        ref.step()
        slab.step_all(roms, comm)
        if k < w - 1:
            continue
        ref.sync()
        a = ref.get_state().cpu().numpy()
        b = slab.assemble(roms, "state").cpu().numpy()
        scale = np.abs(a).max(axis=1, keepdims=True)
        err = float((np.abs(a - b) / scale).max())
        assert err <= 1e-12, (k, err)
        if k >= w:  # replicated solves: every rank holds the same bits
            ys = [x.get_y().cpu().numpy() for x in roms]
            ls = [x.get_eigen().cpu().numpy() for x in roms]
            for y in ys[1:]:
                assert np.array_equal(y, ys[0])
            for l in ls[1:]:
                assert np.array_equal(l, ls[0])
        # S-hat_{k+1}: bit for bit (the indicator agrees to rounding; a cell exactly at the
        # threshold may differ, north_star's 1e-12 rule)
        ma = torch.empty(ref.mask_words, dtype=torch.int32, device="cuda")
        ref.lib.hrom_get_mask(ref.h, ma.data_ptr())
        sa = cells_from_mask(wl, ma)
        mb = slab.assemble(roms, "mask")
        sb = cells_from_mask(wl, mb)
        ng = int(np.ceil(wl.f * wl.N))
        assert sa.sum() == sb.sum() and sa.sum() <= ng
        diff = np.nonzero(sa != sb)[0]
        if diff.size:
            ea = torch.empty(wl.N, dtype=torch.float64, device="cuda")
            ref.lib.hrom_get_indicator(ref.h, ea.data_ptr())
            ea = ea.cpu().numpy()
            tau = np.sort(ea)[::-1][ng - 1]
            assert np.all(np.abs(ea[diff] - tau) <= 1e-12 * max(tau, 1e-300)), (k, diff[:8])
    for x in roms:
        x.sync()
    assert all(x.effective_rank() == ref.effective_rank() for x in roms)
    if filt:  # sweeps of the last step's cascade (ireg[4..6]) as the unsharded filter counted them
        import ctypes as C
        def sweeps(rom):
            out = (C.c_int32 * 8)()
            rom.lib.hrom_debug_counters(rom.h, C.cast(out, C.c_void_p), 8)
            return list(out)[4:7]
        assert all(sweeps(x) == sweeps(ref) for x in roms), (sweeps(ref), [sweeps(x) for x in roms])


def test_slab_selection_matches_unsharded_sample(inputs):
    """The distributed radix select (histogram all-reduce per pass, tie quota by rank order, then by
    cell) against hrom_sample on the same indicator: a trajectory's own indicator, equal values
    straddling the threshold on every rank (ordered-tie path), and fewer positive cells than n_g."""
    from paper_2301_01718_b200 import slab
    from paper_2301_01718_b200.hrom import cells_from_mask
    wl, q0, ref, roms, comm = _mk(inputs, 4, 3, filt=True, nx=96, ny=96, w=8, r=4)
    for _ in range(wl.w + 2):
        ref.step()
        slab.step_all(roms, comm)
    m = torch.empty(ref.mask_words, dtype=torch.int32, device="cuda")

    def check(eps):
        ref.sample(eps=eps, mask_out=m)
        ref.sync()
        slab.resample_all(roms, comm, eps)
        a, b = cells_from_mask(wl, m), cells_from_mask(wl, slab.assemble(roms, "mask"))
        assert np.array_equal(a, b), (int(a.sum()), int(b.sum()))
        return int(a.sum())

    ng = int(np.ceil(wl.f * wl.N))
    assert check(slab.assemble(roms, "indicator")) == ng
    rng = np.random.RandomState(3)
    e = rng.rand(wl.N) ** 3
    e[rng.rand(wl.N) < 0.5] = 0.0
    assert check(torch.from_numpy(e).cuda()) == ng
    t = e.copy()
    thr = np.sort(t)[::-1][ng - 1]
    t[5:wl.N:11] = thr  # ~840 equal values at the threshold on every rank: only some are taken
    assert check(torch.from_numpy(t).cuda()) == ng
    few = np.zeros(wl.N)
    few[rng.choice(wl.N, ng // 2, replace=False)] = 1.0 + rng.rand(ng // 2)
    assert check(torch.from_numpy(few).cuda()) == ng // 2
    allsame = np.full(wl.N, 0.5)  # every cell ties: the first n_g cells by index
    assert check(torch.from_numpy(allsame).cuda()) == ng


def test_slab_against_oracle(inputs, orc):
    """The sharded path against the CPU oracle (same bar as the unsharded trajectory tests while
    the trajectory is not yet sensitive): per-step relative error <= 1e-11 over w + 5 steps."""
    from paper_2301_01718_b200 import slab
    wl, q0, ref, roms, comm = _mk(inputs, 4, 2, filt=True, nx=64, ny=64, w=8, r=4)
    R = orc.Run(wl, q0.cpu().numpy())
    for k in range(1, wl.w + 6):
        R.step()
        slab.step_all(roms, comm)
        o = R.state()
        b = slab.assemble(roms, "state").cpu().numpy().reshape(o.shape)
        err = np.linalg.norm(b - o) / np.linalg.norm(o)
        assert err <= 1e-11, (k, err)


def test_slab_refuses_unsupported(inputs):
    from paper_2301_01718_b200 import slab
    from paper_2301_01718_b200.hrom import HromError
    wl = dataclasses.replace(inputs.config(4, nx=64, ny=64, w=8, r=4), filter_orders=())
    with pytest.raises(HromError):  # fewer own rows than halo rows
        slab.SlabROM(wl, 0, 16)
    with pytest.raises(HromError):  # 1-D grids have no rows to split
        slab.SlabROM(inputs.config(1), 0, 2)


def test_slab_nccl_transport_one_rank(inputs):
    """The DistComm transport (torch.distributed all_gather_into_tensor over NCCL) with the one GPU
    this box has: a one-rank group drives SlabROM.step through every phase of the protocol; the
    result equals the LocalComm run bit for bit."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2301_01718_b200 import slab
    wl, q0, ref, roms, comm = _mk(inputs, 4, 1, filt=True, nx=64, ny=64, w=8, r=4)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        d = slab.SlabROM(wl, 0, 1)
        d.set_state(q0)
        dc = slab.DistComm()
        for _ in range(wl.w + 5):
            d.step(dc)
            slab.step_all(roms, comm)
        d.sync()
        assert torch.equal(d.get_state(), roms[0].get_state())
        assert torch.equal(d.get_mask(), roms[0].get_mask())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed,nranks,ny", [(1, 2, 30), (5, 3, 45)])
def test_slab_replay_and_positivity_escalation(orc, inputs, seed, nranks, ny):
    """hrom_slab_set_window (replay) + S:478 on slabs: a violent window makes the hybrid state
    non-physical on some rank; every rank then redoes the step as a full step with the same dt, and
    the sharded state equals the oracle's escalated step and the unsharded context's; the next basis
    (window-Gram row recomputed over the own rows, summed over the ranks) matches too."""
    from paper_2301_01718_b200 import slab
    from paper_2301_01718_b200.hrom import HybridROM, mask_from_cells
    wl = inputs.Workload("small2d", dim=2, nx=40, ny=ny, bc=0, recon=2, cfl=0.4, w=8, r=2, f=0.12, h=2, W=3, seed=21)
    snaps = inputs.smooth_window(wl, wl.w + 1, seed=seed, amp=0.9)
    rng = np.random.default_rng(seed)
    S = (rng.random(wl.N) < 0.15).astype(np.uint8)
    k = wl.w + 3
    R = orc.Run(wl, snaps[0])
    R.set_window(k, snaps, S)
    dt = orc.dt(wl, snaps[-1])
    assert R.step(dt) == 2  # the oracle escalated
    sn = torch.from_numpy(snaps.reshape(wl.w + 1, -1)).cuda().contiguous()
    mk = mask_from_cells(wl, S)
    ref = HybridROM(wl)
    ref.set_window(k, sn, mk)
    ref.step()
    ref.sync()
    roms = [slab.SlabROM(wl, r, nranks) for r in range(nranks)]
    comm = slab.LocalComm(nranks)
    slab.set_window_all(roms, comm, k, sn, mk)
    slab.step_all(roms, comm)
    for x in roms:
        x.sync()  # the full step is admissible: nothing latched
    assert all(x.escalations() == 1 for x in roms)
    b = slab.assemble(roms, "state").cpu().numpy()
    o = R.state().reshape(b.shape)
    a = ref.get_state().cpu().numpy()
    assert np.abs(b - o).max() <= 1e-13 * np.abs(o).max()
    assert np.array_equal(a, b)  # a full step: bitwise the unsharded one
    # the basis of the window ending at the escalated snapshot
    lam = roms[0].get_eigen().cpu().numpy()
    sig = R.sigma()
    re = R.reff()
    np.testing.assert_allclose(lam[:re], sig[:re] ** 2, rtol=1e-9, atol=1e-13 * sig[0] ** 2)
    for x in roms[1:]:
        assert np.array_equal(x.get_eigen().cpu().numpy(), lam)


def test_slab_replay_hybrid_step_matches_oracle(orc, inputs):
    """Lock-step replay on slabs: one hybrid step from the oracle's window and S-hat (filter on)."""
    from paper_2301_01718_b200 import slab
    from paper_2301_01718_b200.hrom import mask_from_cells
    wl = inputs.Workload("small2d", dim=2, nx=64, ny=60, bc=1, recon=2, cfl=0.4, w=8, r=5, f=0.12, h=2, W=3, seed=21)
    snaps = inputs.smooth_window(wl, wl.w + 1, seed=3, amp=0.05)
    rng = np.random.default_rng(3)
    S = (rng.random(wl.N) < 0.12).astype(np.uint8)
    k = wl.w + 2
    R = orc.Run(wl, snaps[0])
    R.set_window(k, snaps, S)
    assert R.step(orc.dt(wl, snaps[-1])) != 2
    roms = [slab.SlabROM(wl, r, 3) for r in range(3)]
    comm = slab.LocalComm(3)
    slab.set_window_all(roms, comm, k, torch.from_numpy(snaps.reshape(wl.w + 1, -1)).cuda().contiguous(),
                        mask_from_cells(wl, S))
    slab.step_all(roms, comm)
    for x in roms:
        x.sync()
    assert all(x.escalations() == 0 for x in roms)
    b = slab.assemble(roms, "state").cpu().numpy()
    o = R.state().reshape(b.shape)
    scale = np.abs(o).max(axis=1, keepdims=True)
    assert float((np.abs(b - o) / scale).max()) <= 1e-12
