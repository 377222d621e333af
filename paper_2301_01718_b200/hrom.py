"""Thin ctypes binding of libhrom (include/hrom.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels of
libhrom.so.  PyTorch provides device memory and the stream.  There is no CPU
fallback: if libhrom.so cannot be loaded, or no CUDA device is present, every
constructor raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhrom.so")

HROM_STATUS = {0: "ok", 1: "invalid argument", 2: "call out of order", 3: "non-positive density or pressure",
               4: "zero least-squares matrix", 5: "CUDA error", 6: "out of device memory"}


class HromError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {HROM_STATUS.get(code, code)} (status {code})")
        self.code = code


class Grid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32),
                ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
                ("bc", C.c_int32), ("recon", C.c_int32)]


class Params(C.Structure):
    _fields_ = [("window", C.c_int32), ("rank", C.c_int32), ("halo", C.c_int32), ("band", C.c_int32),
                ("filter_orders", C.c_int32 * 3), ("n_filter_orders", C.c_int32),
                ("filter_max_sweeps", C.c_int32), ("filter_eps", C.c_double),
                ("eig_rel_cutoff", C.c_double), ("lsq_rel_cutoff", C.c_double),
                ("sample_fraction", C.c_double), ("gram_mode", C.c_int32), ("rebase_period", C.c_int32),
                ("gather_mode", C.c_int32), ("full_period", C.c_int32),
                ("sample_mode", C.c_int32), ("rre_delta", C.c_double), ("odeim_points", C.c_int32)]


class SlabInfo(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("ny_global", C.c_int32), ("row0", C.c_int32),
                ("rows_own", C.c_int32), ("halo_lo", C.c_int32), ("halo_hi", C.c_int32), ("halo", C.c_int32),
                ("cells_own", C.c_int64), ("cells_local", C.c_int64), ("cells_global", C.c_int64),
                ("max_message_bytes", C.c_int64)]


class ImpParams(C.Structure):
    _fields_ = [("flux", C.c_int32), ("dt", C.c_double), ("eps_y", C.c_double), ("j_max", C.c_int32),
                ("newton_tol", C.c_double), ("newton_maxit", C.c_int32)]


# every entry point of include/hrom.h with its ctypes signature
_VP = C.c_void_p
_SIGS = {
    "hrom_create": (C.c_int, [C.POINTER(Grid), C.c_double, C.c_double, C.POINTER(Params), _VP, C.POINTER(_VP)]),
    "hrom_destroy": (None, [_VP]),
    "hrom_set_state": (C.c_int, [_VP, _VP]),
    "hrom_get_state": (C.c_int, [_VP, _VP]),
    "hrom_full_step": (C.c_int, [_VP, C.c_double, _VP]),
    "hrom_hybrid_step": (C.c_int, [_VP, _VP, C.c_double, _VP]),
    "hrom_update_basis": (C.c_int, [_VP]),
    "hrom_sample": (C.c_int, [_VP, C.c_double, _VP, _VP, _VP, _VP]),
    "hrom_sample_rre": (C.c_int, [_VP, C.c_double, _VP, _VP, _VP, _VP]),
    "hrom_odeim": (C.c_int, [_VP, _VP, C.c_int32, C.c_int32, _VP, _VP]),
    "hrom_project": (C.c_int, [_VP, _VP, C.c_int32, _VP]),
    "hrom_reconstruct": (C.c_int, [_VP, _VP, _VP, _VP, _VP]),
    "hrom_filter": (C.c_int, [_VP, _VP, _VP, _VP, _VP]),
    "hrom_step": (C.c_int, [_VP, C.c_double]),
    "hrom_step_ex": (C.c_int, [_VP, C.c_double, _VP]),
    "hrom_rel_l1_error": (C.c_int, [_VP, _VP, _VP, C.POINTER(C.c_double)]),
    "hrom_sync": (C.c_int, [_VP]),
    "hrom_join": (C.c_int, [_VP]),
    "hrom_set_graph": (C.c_int, [_VP, C.c_int32]),
    "hrom_graph_launches": (C.c_int64, [_VP]),
    "hrom_points_used": (C.c_int32, [_VP]),
    "hrom_error_cell": (C.c_int64, [_VP]),
    "hrom_step_index": (C.c_int64, [_VP]),
    "hrom_effective_rank": (C.c_int32, [_VP]),
    "hrom_status_string": (C.c_char_p, [C.c_int]),
    "hrom_set_window": (C.c_int, [_VP, C.c_int64, _VP, C.c_int32, _VP]),
    "hrom_put_snapshot": (C.c_int, [_VP, C.c_int64, _VP]),
    "hrom_rebuild_basis": (C.c_int, [_VP, C.c_int64, _VP]),
    "hrom_get_basis": (C.c_int, [_VP, _VP, _VP]),
    "hrom_get_indicator": (C.c_int, [_VP, _VP]),
    "hrom_get_mask": (C.c_int, [_VP, _VP]),
    "hrom_get_y": (C.c_int, [_VP, _VP]),
    "hrom_get_eigen": (C.c_int, [_VP, _VP]),
    "hrom_mask_words": (C.c_int64, [_VP]),
    "hrom_gram": (C.c_int, [_VP, _VP, C.c_int32, C.c_int64, _VP, _VP]),
    "hrom_put_state": (C.c_int, [_VP, _VP]),
    "hrom_profile": (C.c_int, [_VP, C.c_int32]),
    "hrom_profile_read": (C.c_int, [_VP, _VP, _VP, C.c_int32]),
    "hrom_launch_count": (C.c_int64, [_VP]),
    "hrom_debug_counters": (C.c_int, [_VP, _VP, C.c_int32]),
    "hrom_debug_timers": (C.c_int, [_VP, _VP, C.c_int32]),
    "hrom_debug_read": (C.c_int, [_VP, C.c_int32, _VP, C.c_int64]),
    "hrom_imp_create": (C.c_int, [C.POINTER(Grid), C.c_double, C.POINTER(Params), C.POINTER(ImpParams), _VP,
                                  C.POINTER(_VP)]),
    "hrom_imp_destroy": (None, [_VP]),
    "hrom_imp_set_state": (C.c_int, [_VP, _VP]),
    "hrom_imp_get_state": (C.c_int, [_VP, _VP]),
    "hrom_imp_step": (C.c_int, [_VP, _VP]),
    "hrom_imp_stats": (C.c_int, [_VP, _VP]),
    "hrom_imp_get_mask": (C.c_int, [_VP, _VP]),
    "hrom_imp_get_indicator": (C.c_int, [_VP, _VP]),
    "hrom_imp_get_y": (C.c_int, [_VP, _VP]),
    "hrom_imp_mask_words": (C.c_int64, [_VP]),
    "hrom_imp_effective_rank": (C.c_int32, [_VP]),
    "hrom_imp_sync": (C.c_int, [_VP]),
    "hrom_imp_residual": (C.c_int, [_VP, C.c_int32, _VP, _VP, _VP, _VP]),
    "hrom_imp_newton": (C.c_int, [_VP, C.c_int32, _VP, _VP, _VP, _VP, C.POINTER(C.c_int32)]),
    "hrom_imp_filter": (C.c_int, [_VP, C.c_int32, _VP, _VP, _VP, _VP, _VP, C.POINTER(C.c_int32)]),
    "hrom_imp_set_window": (C.c_int, [_VP, C.c_int64, _VP, C.c_int32, _VP]),
    "hrom_imp_get_band": (C.c_int, [_VP, _VP, _VP]),
    "hrom_imp_debug_timers": (C.c_int, [_VP, _VP]),
    "hrom_slab_partition": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(SlabInfo)]),
    "hrom_slab_create": (C.c_int, [C.POINTER(Grid), C.c_double, C.c_double, C.POINTER(Params), _VP, C.c_int32,
                                   C.c_int32, C.POINTER(_VP)]),
    "hrom_slab_get_info": (C.c_int, [_VP, C.POINTER(SlabInfo)]),
    "hrom_slab_set_state": (C.c_int, [_VP, _VP]),
    "hrom_slab_get_state": (C.c_int, [_VP, _VP]),
    "hrom_slab_get_mask": (C.c_int, [_VP, _VP]),
    "hrom_slab_get_indicator": (C.c_int, [_VP, _VP]),
    "hrom_slab_step": (C.c_int, [_VP, _VP, _VP, C.POINTER(C.c_int64)]),
    "hrom_slab_resample": (C.c_int, [_VP, _VP, _VP, C.POINTER(C.c_int64)]),
    "hrom_slab_set_window": (C.c_int, [_VP, C.c_int64, _VP, C.c_int32, _VP, _VP, C.POINTER(C.c_int64)]),
    "hrom_slab_escalations": (C.c_int64, [_VP]),
}

SECTIONS = ["dt", "masked_rk3", "gathered_gram", "pinv_solve", "fill_pass", "indicator", "seam_filter",
            "band_gram", "positivity", "basis_update", "sampling", "full_step", "rebase_gram", "basis_eigen_side_stream"]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libhrom.so and bind every symbol; raises if the library or a symbol is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libhrom.so not built at {path}; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)  # AttributeError if the ABI lost a symbol
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def _ck(code: int, where: str):
    if code != 0:
        raise HromError(code, where)


def mask_from_cells(wl, cells, device="cuda") -> torch.Tensor:
    """Row-padded N-bit bitmap (hrom.h convention) of a cell list or a 0/1 array of length N."""
    import numpy as np
    arr = np.asarray(cells)
    if arr.dtype == np.uint8 or arr.dtype == bool:
        if arr.size != wl.N:
            raise ValueError("0/1 mask must have N entries")
        idx = np.nonzero(arr)[0]
    else:
        idx = arr.astype(np.int64)
    wpr = (wl.nx + 31) // 32
    ny = wl.ny if wl.dim == 2 else 1
    nwords = max(ny * wpr, (wl.N + 31) // 32)
    words = np.zeros(nwords, dtype=np.uint32)
    i = idx % wl.nx
    j = idx // wl.nx
    np.bitwise_or.at(words, j * wpr + i // 32, (np.uint32(1) << (i % 32).astype(np.uint32)))
    return torch.from_numpy(words.view(np.int32).copy()).to(device)


def cells_from_mask(wl, words: torch.Tensor):
    import numpy as np
    w = words.cpu().numpy().view(np.uint32)
    wpr = (wl.nx + 31) // 32
    ny = wl.ny if wl.dim == 2 else 1
    out = np.zeros(wl.N, dtype=np.uint8)
    for j in range(ny):
        row = w[j * wpr:(j + 1) * wpr]
        bits = ((row[:, None] >> np.arange(32, dtype=np.uint32)[None, :]) & 1).reshape(-1)[: wl.nx]
        out[j * wl.nx:(j + 1) * wl.nx] = bits
    return out


class HybridROM:
    """One hrom_ctx: an explicit hybrid-snapshot AROM on one grid, on the current CUDA device."""

    def __init__(self, wl, stream: Optional[torch.cuda.Stream] = None, gram_mode: int = 0,
                 rebase_period: int = 0, gather_mode: int = 0, full_period: Optional[int] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("libhrom needs a CUDA device (B200, sm_100a); no CPU fallback exists")
        self.lib = load_library()
        self.wl = wl
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        g = Grid(wl.dim, wl.nx, wl.ny if wl.dim == 2 else 1, wl.x0, wl.x1, wl.y0, wl.y1, wl.bc, wl.recon)
        fo = (C.c_int32 * 3)(*(list(wl.filter_orders) + [0, 0, 0])[:3])
        p = Params(wl.w, wl.r, wl.h, wl.W, fo, len(wl.filter_orders), wl.filter_max_sweeps, wl.filter_eps,
                   wl.eig_rel_cutoff, wl.lsq_rel_cutoff, wl.f, gram_mode, rebase_period, gather_mode,
                   getattr(wl, "z", 0) if full_period is None else full_period,
                   1 if getattr(wl, "delta", 0.0) > 0.0 else 0, float(getattr(wl, "delta", 0.0)),
                   int(getattr(wl, "n_p", 0)))
        h = C.c_void_p()
        _ck(self.lib.hrom_create(C.byref(g), wl.gamma, wl.cfl, C.byref(p), C.c_void_p(self.stream.cuda_stream),
                                 C.byref(h)), "hrom_create")
        self.h = h
        self.mask_words = int(self.lib.hrom_mask_words(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.hrom_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- state ----
    def set_state(self, q: torch.Tensor):
        assert q.dtype == torch.float64 and q.is_contiguous() and q.numel() == self.wl.D
        _ck(self.lib.hrom_set_state(self.h, _ptr(q)), "hrom_set_state")

    def get_state(self, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if out is None:
            out = torch.empty((self.wl.c, self.wl.N), dtype=torch.float64, device="cuda")
        _ck(self.lib.hrom_get_state(self.h, _ptr(out)), "hrom_get_state")
        return out

    # ---- hot path ----
    def full_step(self, dt: float = 0.0, dt_out: Optional[torch.Tensor] = None):
        _ck(self.lib.hrom_full_step(self.h, dt, _ptr(dt_out)), "hrom_full_step")

    def hybrid_step(self, mask: Optional[torch.Tensor] = None, dt: float = 0.0, dt_out: Optional[torch.Tensor] = None):
        _ck(self.lib.hrom_hybrid_step(self.h, _ptr(mask), dt, _ptr(dt_out)), "hrom_hybrid_step")

    def update_basis(self):
        _ck(self.lib.hrom_update_basis(self.h), "hrom_update_basis")

    def sample(self, fraction: Optional[float] = None, eps: Optional[torch.Tensor] = None,
               mask_out: Optional[torch.Tensor] = None, list_out: Optional[torch.Tensor] = None,
               count_out: Optional[torch.Tensor] = None):
        f = self.wl.f if fraction is None else fraction
        _ck(self.lib.hrom_sample(self.h, f, _ptr(eps), _ptr(mask_out), _ptr(list_out), _ptr(count_out)), "hrom_sample")

    def sample_rre(self, delta: Optional[float] = None, eps: Optional[torch.Tensor] = None,
                   mask_out: Optional[torch.Tensor] = None, list_out: Optional[torch.Tensor] = None,
                   count_out: Optional[torch.Tensor] = None):
        d = self.wl.delta if delta is None else delta
        _ck(self.lib.hrom_sample_rre(self.h, d, _ptr(eps), _ptr(mask_out), _ptr(list_out), _ptr(count_out)),
            "hrom_sample_rre")

    def odeim(self, phi: torch.Tensor, n_p: int):
        """ODEIM points of phi ((m, D) contiguous = D x m column-major): (cells int32, rows int64)."""
        assert phi.dtype == torch.float64 and phi.is_contiguous() and phi.shape[1] == self.wl.D
        cells = torch.empty(n_p, dtype=torch.int32, device="cuda")
        rows = torch.empty(n_p, dtype=torch.int64, device="cuda")
        _ck(self.lib.hrom_odeim(self.h, _ptr(phi), phi.shape[0], n_p, _ptr(cells), _ptr(rows)), "hrom_odeim")
        return cells, rows

    def project(self, phi: torch.Tensor) -> torch.Tensor:
        """Phi^T [gamma_{k-w}, ..., gamma_k] (m x (w+1)) on the FP64 tensor cores."""
        assert phi.dtype == torch.float64 and phi.is_contiguous() and phi.shape[1] == self.wl.D
        out = torch.empty((phi.shape[0], self.wl.w + 1), dtype=torch.float64, device="cuda")
        _ck(self.lib.hrom_project(self.h, _ptr(phi), phi.shape[0], _ptr(out)), "hrom_project")
        return out

    def reconstruct(self, v: torch.Tensor, mask: Optional[torch.Tensor] = None,
                    y_out: Optional[torch.Tensor] = None, eps_out: Optional[torch.Tensor] = None):
        _ck(self.lib.hrom_reconstruct(self.h, _ptr(mask), _ptr(v), _ptr(y_out), _ptr(eps_out)), "hrom_reconstruct")

    def filter(self, v: torch.Tensor, F: torch.Tensor, mask: Optional[torch.Tensor] = None,
               kept_out: Optional[torch.Tensor] = None):
        _ck(self.lib.hrom_filter(self.h, _ptr(mask), _ptr(v), _ptr(F), _ptr(kept_out)), "hrom_filter")

    def step(self, dt: float = 0.0, count_out: Optional[torch.Tensor] = None):
        """One step of Algorithm 1; count_out (device int32, 1 element): |S-hat| used (N if full)."""
        if count_out is None:
            _ck(self.lib.hrom_step(self.h, dt), "hrom_step")
        else:
            assert count_out.dtype == torch.int32 and count_out.is_cuda
            _ck(self.lib.hrom_step_ex(self.h, dt, _ptr(count_out)), "hrom_step_ex")

    def rel_l1_error(self, a: torch.Tensor, b: torch.Tensor) -> float:
        """e = sum|a - b| / sum|b| over the D entries, on the device."""
        assert a.dtype == b.dtype == torch.float64 and a.numel() == b.numel() == self.wl.D
        out = C.c_double()
        _ck(self.lib.hrom_rel_l1_error(self.h, _ptr(a.contiguous()), _ptr(b.contiguous()), C.byref(out)),
            "hrom_rel_l1_error")
        return out.value

    def sync(self):
        code = self.lib.hrom_sync(self.h)
        if code == 3:
            raise HromError(code, f"hrom_sync (cell {self.lib.hrom_error_cell(self.h)})")
        _ck(code, "hrom_sync")

    def set_graph(self, enable: bool = True):
        """Replay steady-state steps from per-ring-phase CUDA graphs (hrom_set_graph)."""
        _ck(self.lib.hrom_set_graph(self.h, int(enable)), "hrom_set_graph")

    def graph_launches(self) -> int:
        return int(self.lib.hrom_graph_launches(self.h))

    def join(self):
        """Context stream waits for the library's side-stream work (no host sync)."""
        _ck(self.lib.hrom_join(self.h), "hrom_join")

    def points_used(self) -> int:
        """ODEIM points (n_p)_k of the latest step; 0 for full steps / S-hat = G."""
        return int(self.lib.hrom_points_used(self.h))

    @property
    def k(self) -> int:
        return int(self.lib.hrom_step_index(self.h))

    def effective_rank(self) -> int:
        return int(self.lib.hrom_effective_rank(self.h))

    # ---- replay / inspection hooks ----
    def set_window(self, k: int, snaps: torch.Tensor, mask_next: Optional[torch.Tensor] = None):
        assert snaps.dtype == torch.float64 and snaps.is_contiguous()
        _ck(self.lib.hrom_set_window(self.h, k, _ptr(snaps), snaps.shape[0], _ptr(mask_next)), "hrom_set_window")

    def put_snapshot(self, k: int, q: torch.Tensor):
        """Write gamma_k into its ring slot (window streaming, no basis work)."""
        assert q.dtype == torch.float64 and q.is_contiguous()
        _ck(self.lib.hrom_put_snapshot(self.h, k, _ptr(q)), "hrom_put_snapshot")

    def rebuild_basis(self, k: int, mask_next: Optional[torch.Tensor] = None):
        """Basis from the window gamma_{k-w}..gamma_k written with put_snapshot."""
        _ck(self.lib.hrom_rebuild_basis(self.h, k, _ptr(mask_next)), "hrom_rebuild_basis")

    def basis(self):
        r = self.effective_rank()
        phi = torch.empty((max(r, 1), self.wl.D), dtype=torch.float64, device="cuda")
        psi = torch.empty((self.wl.c, self.wl.N), dtype=torch.float64, device="cuda")
        _ck(self.lib.hrom_get_basis(self.h, _ptr(phi), _ptr(psi)), "hrom_get_basis")
        return phi[:r], psi

    def indicator(self) -> torch.Tensor:
        e = torch.empty(self.wl.N, dtype=torch.float64, device="cuda")
        _ck(self.lib.hrom_get_indicator(self.h, _ptr(e)), "hrom_get_indicator")
        return e

    def mask(self) -> torch.Tensor:
        m = torch.empty(self.mask_words, dtype=torch.int32, device="cuda")
        _ck(self.lib.hrom_get_mask(self.h, _ptr(m)), "hrom_get_mask")
        return m

    def y(self) -> torch.Tensor:
        y = torch.zeros(self.wl.r, dtype=torch.float64, device="cuda")
        _ck(self.lib.hrom_get_y(self.h, _ptr(y)), "hrom_get_y")
        return y

    def eigenvalues(self) -> torch.Tensor:
        lam = torch.empty(self.wl.w, dtype=torch.float64, device="cuda")
        _ck(self.lib.hrom_get_eigen(self.h, _ptr(lam)), "hrom_get_eigen")
        return lam

    def put_state(self, q: torch.Tensor):
        _ck(self.lib.hrom_put_state(self.h, _ptr(q)), "hrom_put_state")

    def profile(self, enable: bool = True):
        _ck(self.lib.hrom_profile(self.h, int(enable)), "hrom_profile")

    def profile_read(self):
        ms = (C.c_double * len(SECTIONS))()
        cnt = (C.c_int64 * len(SECTIONS))()
        _ck(self.lib.hrom_profile_read(self.h, C.cast(ms, C.c_void_p), C.cast(cnt, C.c_void_p), len(SECTIONS)),
            "hrom_profile_read")
        return {name: (ms[i], cnt[i]) for i, name in enumerate(SECTIONS)}

    def launch_count(self) -> int:
        return int(self.lib.hrom_launch_count(self.h))

    def debug_timers(self, n: int = 32):
        out = (C.c_int64 * n)()
        _ck(self.lib.hrom_debug_timers(self.h, C.cast(out, C.c_void_p), n), "hrom_debug_timers")
        return list(out)

    def debug_counters(self, n: int = 8):
        out = (C.c_int32 * n)()
        _ck(self.lib.hrom_debug_counters(self.h, C.cast(out, C.c_void_p), n), "hrom_debug_counters")
        return list(out)

    def gram(self, cols: torch.Tensor, rho: Optional[torch.Tensor] = None) -> torch.Tensor:
        """C = (S - rho)^T (S - rho) for the rows of a (ncol, rows) tensor (DMMA kernel)."""
        ncol, rows = cols.shape
        ptrs = torch.tensor([cols[i].data_ptr() for i in range(ncol)], dtype=torch.int64, device="cuda")
        out = torch.empty((ncol, ncol), dtype=torch.float64, device="cuda")
        _ck(self.lib.hrom_gram(self.h, _ptr(ptrs), ncol, rows, _ptr(rho), _ptr(out)), "hrom_gram")
        return out


def _params_of(wl, gram_mode=0, rebase_period=0, gather_mode=0, full_period=None) -> Params:
    fo = (C.c_int32 * 3)(*(list(wl.filter_orders) + [0, 0, 0])[:3])
    return Params(wl.w, wl.r, wl.h, wl.W, fo, len(wl.filter_orders), wl.filter_max_sweeps, wl.filter_eps,
                  wl.eig_rel_cutoff, wl.lsq_rel_cutoff, wl.f, gram_mode, rebase_period, gather_mode,
                  getattr(wl, "z", 0) if full_period is None else full_period,
                  1 if getattr(wl, "delta", 0.0) > 0.0 else 0, float(getattr(wl, "delta", 0.0)),
                  int(getattr(wl, "n_p", 0)))


class ImplicitROM:
    """One hrom_imp_ctx: Algorithm 1 with the paper's implicit HDM (NEXT-4) on one grid."""

    def __init__(self, wl, stream: Optional[torch.cuda.Stream] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("libhrom needs a CUDA device (B200, sm_100a); no CPU fallback exists")
        self.lib = load_library()
        self.wl = wl
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        g = Grid(wl.dim, wl.nx, wl.ny if wl.dim == 2 else 1, wl.x0, wl.x1, wl.y0, wl.y1, wl.bc, wl.recon)
        p = _params_of(wl)
        ip = ImpParams(int(wl.flux), float(wl.dt), float(wl.eps_y), int(wl.j_max), float(wl.newton_tol),
                       int(wl.newton_maxit))
        h = C.c_void_p()
        _ck(self.lib.hrom_imp_create(C.byref(g), wl.gamma, C.byref(p), C.byref(ip),
                                     C.c_void_p(self.stream.cuda_stream), C.byref(h)), "hrom_imp_create")
        self.h = h
        self.mask_words = int(self.lib.hrom_imp_mask_words(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.hrom_imp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_state(self, q: torch.Tensor):
        assert q.dtype == torch.float64 and q.is_contiguous() and q.numel() == self.wl.D
        _ck(self.lib.hrom_imp_set_state(self.h, _ptr(q)), "hrom_imp_set_state")

    def get_state(self, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if out is None:
            out = torch.empty((self.wl.c, self.wl.N), dtype=torch.float64, device="cuda")
        _ck(self.lib.hrom_imp_get_state(self.h, _ptr(out)), "hrom_imp_get_state")
        return out

    def step(self, count_out: Optional[torch.Tensor] = None):
        _ck(self.lib.hrom_imp_step(self.h, _ptr(count_out)), "hrom_imp_step")

    def stats(self):
        """(kind, J, Newton iterations, GMRES products, ODEIM points used) of the last step."""
        out = (C.c_int32 * 5)()
        _ck(self.lib.hrom_imp_stats(self.h, C.cast(out, C.c_void_p)), "hrom_imp_stats")
        return tuple(out)

    def mask(self) -> torch.Tensor:
        out = torch.empty(self.mask_words, dtype=torch.int32, device="cuda")
        _ck(self.lib.hrom_imp_get_mask(self.h, _ptr(out)), "hrom_imp_get_mask")
        return out

    def indicator(self) -> torch.Tensor:
        out = torch.empty(self.wl.N, dtype=torch.float64, device="cuda")
        _ck(self.lib.hrom_imp_get_indicator(self.h, _ptr(out)), "hrom_imp_get_indicator")
        return out

    def y(self) -> torch.Tensor:
        out = torch.zeros(self.wl.r, dtype=torch.float64, device="cuda")
        _ck(self.lib.hrom_imp_get_y(self.h, _ptr(out)), "hrom_imp_get_y")
        return out

    def effective_rank(self) -> int:
        return int(self.lib.hrom_imp_effective_rank(self.h))

    def sync(self):
        _ck(self.lib.hrom_imp_sync(self.h), "hrom_imp_sync")

    def residual(self, q, qm1, qm2=None, order=2) -> torch.Tensor:
        R = torch.empty_like(q)
        _ck(self.lib.hrom_imp_residual(self.h, order, _ptr(q), _ptr(qm1), _ptr(qm2), _ptr(R)), "hrom_imp_residual")
        return R

    def newton(self, q: torch.Tensor, qm1, qm2=None, order=2, mask: Optional[torch.Tensor] = None) -> int:
        """Solves in place (q: initial guess + frozen data); returns the Newton iterations."""
        its = C.c_int32()
        _ck(self.lib.hrom_imp_newton(self.h, order, _ptr(qm1), _ptr(qm2), _ptr(mask), _ptr(q), C.byref(its)),
            "hrom_imp_newton")
        return its.value

    def filter(self, v: torch.Tensor, mask: torch.Tensor, qm1, qm2=None, order=2):
        """Filters v in place; returns (kept cells uint8 tensor, sweeps per order)."""
        kept = torch.zeros(self.wl.N, dtype=torch.uint8, device="cuda")
        sw = (C.c_int32 * 3)()
        _ck(self.lib.hrom_imp_filter(self.h, order, _ptr(qm1), _ptr(qm2), _ptr(mask), _ptr(v), _ptr(kept),
                                     C.cast(sw, C.POINTER(C.c_int32))), "hrom_imp_filter")
        return kept, list(sw)

    def debug_timers(self):
        """Newton phase clocks since the last read (block 0, clock64 cycles): products, Gram-Schmidt,
        norms + Givens, line searches, whole kernels, products, solves."""
        out = (C.c_int64 * 10)()
        _ck(self.lib.hrom_imp_debug_timers(self.h, C.cast(out, C.c_void_p)), "hrom_imp_debug_timers")
        return list(out)[:9]

    def band(self):
        """Cells of the filter band of the current sets (ascending)."""
        lst = torch.zeros(self.wl.N, dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
        _ck(self.lib.hrom_imp_get_band(self.h, _ptr(lst), _ptr(cnt)), "hrom_imp_get_band")
        return lst[:int(cnt.item())].cpu().numpy()

    def set_window(self, k: int, snaps: torch.Tensor, mask_next: Optional[torch.Tensor] = None):
        _ck(self.lib.hrom_imp_set_window(self.h, k, _ptr(snaps), snaps.shape[0], _ptr(mask_next)),
            "hrom_imp_set_window")
