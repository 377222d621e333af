"""Row-slab sharding of ONE problem across ranks (include/hrom.h, hrom_slab_*).

Plumbing only: every reduction, halo pack / unpack, selection pass and solve runs in the CUDA
kernels of libhrom (csrc/slab.cu).  This module owns the transport: `hrom_slab_step` leaves one
message per phase in a device buffer, a communicator all-gathers the ranks' messages in rank order,
and the gathered buffer goes into the next call.

* ``DistComm``   -- one process per GPU, ``torch.distributed.all_gather_into_tensor`` (NCCL over
                    NVLink / NVSwitch on GPUs; gloo on CPU for the host-logic tests).
* ``LocalComm``  -- several slab contexts inside ONE process (one GPU): the gathered buffer is the
                    concatenation of their messages.  Used by the single-GPU parity test and by
                    ``step_all``; no kernel of one context waits on another.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import torch

from . import hrom as H


def partition(ny: int, nranks: int, rank: int, periodic: bool, halo_rows: int) -> H.SlabInfo:
    """Host-only: the rows rank `rank` of `nranks` owns (no GPU needed)."""
    info = H.SlabInfo()
    H._ck(H.load_library().hrom_slab_partition(ny, nranks, rank, int(periodic), halo_rows, C.byref(info)),
          "hrom_slab_partition")
    return info


def halo_rows(wl) -> int:
    """max(3 h, 2 h + W): reach of a three-stage step and of the set dilations (hrom.h)."""
    return max(3 * wl.h, 2 * wl.h + max(wl.W, 0))


class DistComm:
    """All-gather over torch.distributed (rank order = process-group rank order)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.nranks = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_gather(self, msg: torch.Tensor) -> torch.Tensor:
        out = torch.empty(self.nranks * msg.numel(), dtype=msg.dtype, device=msg.device)
        self.dist.all_gather_into_tensor(out, msg.contiguous(), group=self.group)
        return out


class LocalComm:
    """All ranks live in this process: gather = concatenate (rank order = list order)."""

    def __init__(self, nranks: int):
        self.nranks = nranks

    def all_gather_many(self, msgs: Sequence[torch.Tensor]) -> torch.Tensor:
        assert len(msgs) == self.nranks and len({m.numel() for m in msgs}) == 1
        return torch.cat([m.reshape(-1) for m in msgs])


class SlabROM:
    """One rank's row slab of a sharded explicit hybrid-snapshot AROM (one hrom_ctx)."""

    def __init__(self, wl, rank: int, nranks: int, stream: Optional[torch.cuda.Stream] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("libhrom needs a CUDA device (B200, sm_100a); no CPU fallback exists")
        self.lib = H.load_library()
        self.wl = wl
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        g = H.Grid(wl.dim, wl.nx, wl.ny if wl.dim == 2 else 1, wl.x0, wl.x1, wl.y0, wl.y1, wl.bc, wl.recon)
        fo = (C.c_int32 * 3)(*(list(wl.filter_orders) + [0, 0, 0])[:3])
        # a slab runs Algorithm 1 with z = infinity and the fixed sampling fraction (P = S-hat)
        p = H.Params(wl.w, wl.r, wl.h, wl.W, fo, len(wl.filter_orders), wl.filter_max_sweeps, wl.filter_eps,
                     wl.eig_rel_cutoff, wl.lsq_rel_cutoff, wl.f, 0, 0, 1, 0, 0, 0.0, 0)
        h = C.c_void_p()
        H._ck(self.lib.hrom_slab_create(C.byref(g), wl.gamma, wl.cfl, C.byref(p), C.c_void_p(self.stream.cuda_stream),
                                        rank, nranks, C.byref(h)), "hrom_slab_create")
        self.h = h
        self.info = H.SlabInfo()
        H._ck(self.lib.hrom_slab_get_info(self.h, C.byref(self.info)), "hrom_slab_get_info")
        self.rank, self.nranks = rank, nranks
        self.send = torch.zeros(int(self.info.max_message_bytes), dtype=torch.uint8, device="cuda")
        self.wpr = (wl.nx + 31) // 32

    def close(self):
        if getattr(self, "h", None):
            self.lib.hrom_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- state I/O (own rows) ----
    def set_state(self, q_global: torch.Tensor):
        """q_global: the WHOLE initial state (c, N_global); the slab copies its rows and halos."""
        assert q_global.dtype == torch.float64 and q_global.is_contiguous() and q_global.numel() == self.wl.D
        H._ck(self.lib.hrom_slab_set_state(self.h, H._ptr(q_global)), "hrom_slab_set_state")

    def get_state(self) -> torch.Tensor:
        out = torch.empty((self.wl.c, int(self.info.cells_own)), dtype=torch.float64, device="cuda")
        H._ck(self.lib.hrom_slab_get_state(self.h, H._ptr(out)), "hrom_slab_get_state")
        return out

    def get_mask(self) -> torch.Tensor:
        out = torch.empty(int(self.info.rows_own) * self.wpr, dtype=torch.int32, device="cuda")
        H._ck(self.lib.hrom_slab_get_mask(self.h, H._ptr(out)), "hrom_slab_get_mask")
        return out

    def get_indicator(self) -> torch.Tensor:
        out = torch.empty(int(self.info.cells_own), dtype=torch.float64, device="cuda")
        H._ck(self.lib.hrom_slab_get_indicator(self.h, H._ptr(out)), "hrom_slab_get_indicator")
        return out

    def get_y(self) -> torch.Tensor:
        out = torch.zeros(self.wl.r, dtype=torch.float64, device="cuda")
        H._ck(self.lib.hrom_get_y(self.h, H._ptr(out)), "hrom_get_y")
        return out

    def get_eigen(self) -> torch.Tensor:
        out = torch.zeros(self.wl.w, dtype=torch.float64, device="cuda")
        H._ck(self.lib.hrom_get_eigen(self.h, H._ptr(out)), "hrom_get_eigen")
        return out

    @property
    def k(self) -> int:
        return int(self.lib.hrom_step_index(self.h))

    def effective_rank(self) -> int:
        return int(self.lib.hrom_effective_rank(self.h))

    def sync(self):
        code = self.lib.hrom_sync(self.h)
        if code == 3:
            raise H.HromError(code, f"hrom_sync (slab rank {self.rank}, local cell {self.lib.hrom_error_cell(self.h)})")
        H._ck(code, "hrom_sync")

    # ---- the phase protocol ----
    def phase(self, gathered: Optional[torch.Tensor]) -> Optional[torch.Tensor]:
        """Run the local work up to the next exchange; returns this rank's message (a view of the
        send buffer) or None when the step is complete."""
        n = C.c_int64(0)
        H._ck(self.lib.hrom_slab_step(self.h, H._ptr(gathered), H._ptr(self.send), C.byref(n)), "hrom_slab_step")
        return self.send[: n.value] if n.value > 0 else None

    def resample_begin(self, eps_own: torch.Tensor) -> torch.Tensor:
        """Start H8 alone on an explicit indicator of the own cells (hrom_slab_resample)."""
        assert eps_own.dtype == torch.float64 and eps_own.is_contiguous() and eps_own.numel() == int(self.info.cells_own)
        n = C.c_int64(0)
        H._ck(self.lib.hrom_slab_resample(self.h, H._ptr(eps_own), H._ptr(self.send), C.byref(n)), "hrom_slab_resample")
        return self.send[: n.value]

    def resample(self, eps_own: torch.Tensor, comm: DistComm):
        msg = self.resample_begin(eps_own)
        while msg is not None:
            msg = self.phase(comm.all_gather(msg))

    def set_window_begin(self, k: int, snaps_global: torch.Tensor, mask_global: torch.Tensor) -> torch.Tensor:
        """Replay hook: whole-grid window (w+1, c, N) and whole-grid S-hat bitmap (hrom_slab_set_window)."""
        assert snaps_global.dtype == torch.float64 and snaps_global.is_contiguous()
        n = C.c_int64(0)
        H._ck(self.lib.hrom_slab_set_window(self.h, k, H._ptr(snaps_global), snaps_global.shape[0], H._ptr(mask_global),
                                            H._ptr(self.send), C.byref(n)), "hrom_slab_set_window")
        return self.send[: n.value]

    def escalations(self) -> int:
        return int(self.lib.hrom_slab_escalations(self.h))

    def step(self, comm: DistComm):
        """One step of Algorithm 1 on this rank's slab; collective over `comm`."""
        msg = self.phase(None)
        while msg is not None:
            msg = self.phase(comm.all_gather(msg))


def step_all(roms: List[SlabROM], comm: LocalComm):
    """One step of Algorithm 1 on all slabs of one process, in lock step."""
    msgs = [r.phase(None) for r in roms]
    while msgs[0] is not None:
        assert all(m is not None for m in msgs)
        gathered = comm.all_gather_many(msgs)
        msgs = [r.phase(gathered) for r in roms]
    assert all(m is None for m in msgs)


def resample_all(roms: List[SlabROM], comm: LocalComm, eps_global: torch.Tensor):
    """H8 alone on all slabs of one process from a whole-grid indicator."""
    msgs = []
    for r in roms:
        lo = int(r.info.row0) * r.wl.nx
        msgs.append(r.resample_begin(eps_global[lo: lo + int(r.info.cells_own)].contiguous()))
    while msgs[0] is not None:
        gathered = comm.all_gather_many(msgs)
        msgs = [r.phase(gathered) for r in roms]


def set_window_all(roms: List[SlabROM], comm: LocalComm, k: int, snaps_global: torch.Tensor, mask_global: torch.Tensor):
    """Replay hook on all slabs of one process."""
    msgs = [r.set_window_begin(k, snaps_global, mask_global) for r in roms]
    while msgs[0] is not None:
        gathered = comm.all_gather_many(msgs)
        msgs = [r.phase(gathered) for r in roms]


def assemble(roms: List[SlabROM], what: str = "state") -> torch.Tensor:
    """Concatenate the own rows of all slabs (rank order) into the whole-grid array."""
    wl = roms[0].wl
    if what == "state":
        parts = [r.get_state().reshape(wl.c, int(r.info.rows_own), wl.nx) for r in roms]
        return torch.cat(parts, dim=1).reshape(wl.c, wl.N)
    if what == "mask":
        return torch.cat([r.get_mask() for r in roms])
    if what == "indicator":
        return torch.cat([r.get_indicator() for r in roms])
    raise ValueError(what)
