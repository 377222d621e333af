"""Host logic of the row-slab sharding on CPU: the partition (C ABI, no GPU), and
the transport layer over torch.distributed with the gloo backend, world size 2 -- rank-ordered
all-gather, neighbour halo assembly (periodic and open ends), and the all-reduce protocol of the
distributed top-n_g selection (2048-bin histograms per radix pass, ties by ascending cell across
ranks) emulated in numpy against a sort of the whole array."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_covers_the_grid_once():
    from paper_2301_01718_b200 import slab
    for ny, P, per in [(2048, 8, True), (130, 3, False), (96, 2, True), (50, 1, False), (1024, 5, False)]:
        infos = [slab.partition(ny, P, r, per, 8) for r in range(P)]
        assert infos[0].row0 == 0 and sum(i.rows_own for i in infos) == ny
        for a, b in zip(infos, infos[1:]):
            assert b.row0 == a.row0 + a.rows_own
            assert abs(a.rows_own - b.rows_own) <= 1
        for i in infos:
            inner_lo = per or i.rank > 0
            inner_hi = per or i.rank < P - 1
            assert i.halo_lo == (8 if (P > 1 and inner_lo) else 0)
            assert i.halo_hi == (8 if (P > 1 and inner_hi) else 0)


def test_partition_refuses_slabs_thinner_than_the_halo():
    from paper_2301_01718_b200 import slab
    from paper_2301_01718_b200.hrom import HromError
    with pytest.raises(HromError):
        slab.partition(64, 16, 0, True, 8)


def _select_protocol(eps_own, comm, rank, n_g):
    """The message protocol of csrc/slab.cu's selection (6 radix passes over the IEEE patterns of
    eps > 0, one 2048-bin histogram all-gather per pass, tie quota by rank order) in numpy."""
    bits = eps_own.view(np.uint64)
    prefix, rem, allpos = np.uint64(0), n_g, False
    digit = 0
    gath = None
    for p in range(6):
        shift = 53 - 11 * p if p < 5 else 0
        width = 9 if shift == 0 else 11
        hm = np.uint64(0) if p == 0 else np.uint64((~0 << (shift + width)) & 0xFFFFFFFFFFFFFFFF)
        cand = (bits != 0) & ((bits & hm) == prefix)
        hist = np.bincount(((bits[cand] >> np.uint64(shift)) & np.uint64(2047)).astype(np.int64), minlength=2048)
        gath = comm.all_gather(torch.from_numpy(hist.astype(np.int32))).numpy().reshape(comm.nranks, 2048)
        tot = gath.astype(np.int64).sum(axis=0)
        if p == 0 and n_g >= tot.sum():
            allpos = True
        if allpos:
            continue
        above = 0
        for b in range(2047, -1, -1):
            if above < rem <= above + tot[b]:
                digit = b
                break
            above += tot[b]
        prefix |= np.uint64(digit) << np.uint64(shift)
        rem -= above
    if allpos:
        return bits != 0
    before = int(gath[:rank, digit].sum())
    mine = int(gath[rank, digit])
    quota = min(max(rem - before, 0), mine)
    sel = bits > prefix
    ties = np.nonzero(bits == prefix)[0]
    sel[ties[:quota]] = True
    return sel


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2301_01718_b200 import slab
        comm = slab.DistComm()
        res = {}
        # (1) rank-ordered all-gather
        g = comm.all_gather(torch.full((3,), float(rank), dtype=torch.float64))
        res["gather"] = g.tolist()
        # (2) halo assembly: every rank sends [first H own rows | last H own rows]; the lower halo is
        # the previous rank's LAST rows, the upper halo the next rank's FIRST rows
        ny, nx, H = 40, 6, 4
        field = np.arange(ny * nx, dtype=np.float64).reshape(ny, nx)
        for per in (True, False):
            info = slab.partition(ny, world, rank, per, H)
            own = field[info.row0:info.row0 + info.rows_own]
            msg = torch.from_numpy(np.concatenate([own[:H].ravel(), own[-H:].ravel()]))
            gath = comm.all_gather(msg).numpy().reshape(world, 2, H, nx)
            lo = gath[(rank - 1) % world, 1] if info.halo_lo else np.zeros((0, nx))
            hi = gath[(rank + 1) % world, 0] if info.halo_hi else np.zeros((0, nx))
            local = np.concatenate([lo, own, hi])
            rows = [(info.row0 - info.halo_lo + j) % ny for j in range(local.shape[0])]
            res[f"halo{int(per)}"] = bool(np.array_equal(local, field[rows]))
        # (3) the selection protocol: union of the ranks' masks = top n_g of the whole array with
        # ties by ascending cell; cases: plain, ties at the threshold across ranks, few positives
        rng = np.random.RandomState(7)
        N = 4000
        cases = {}
        e = rng.rand(N) ** 4
        e[rng.rand(N) < 0.6] = 0.0
        cases["plain"] = (e, 300)
        t = e.copy()
        t[100:N:7] = 0.25  # many equal values straddling both ranks
        cases["ties"] = (t, 450)
        cases["fewpos"] = (e, 3000)
        for name, (arr, n_g) in cases.items():
            lo = rank * (N // world)
            hi = N if rank == world - 1 else lo + N // world
            sel = _select_protocol(arr[lo:hi].copy(), comm, rank, n_g)
            allsel = comm.all_gather(torch.from_numpy(np.pad(sel, (0, N - sel.size)).astype(np.uint8)))
            parts = allsel.numpy().reshape(world, N)
            whole = np.concatenate([parts[r][: (N if r == world - 1 else (r + 1) * (N // world)) - r * (N // world)]
                                    for r in range(world)]).astype(bool)
            pos = np.nonzero(arr > 0)[0]
            order = pos[np.lexsort((pos, -arr[pos]))][:n_g]  # descending value, ties by ascending cell
            want = np.zeros(N, dtype=bool)
            want[order] = True
            res[f"sel_{name}"] = bool(np.array_equal(whole, want))
        out[rank] = res
    finally:
        dist.destroy_process_group()


def test_transport_and_selection_protocol_two_ranks_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        assert res[r]["gather"] == [0.0, 0.0, 0.0, 1.0, 1.0, 1.0]
        for key in ("halo0", "halo1", "sel_plain", "sel_ties", "sel_fewpos"):
            assert res[r][key], (r, key)
