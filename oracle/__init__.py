"""ctypes wrapper of the CPU oracle (liboracle.so).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg may import this package.  The product
path (paper_2301_01718_b200) never imports it.  See oracle.h for the contract
and the paper citations of every function.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SOURCES = ["euler.cpp", "linalg.cpp", "sampling_filter.cpp", "driver.cpp", "implicit.cpp"]


def build(force: bool = False) -> str:
    """g++ -O2 -ffp-contract=off (no fast-math, no BLAS), single-threaded."""
    srcs = [os.path.join(_HERE, s) for s in _SOURCES]
    deps = srcs + [os.path.join(_HERE, "oracle.h"), os.path.join(_HERE, "common.hpp")]
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= max(os.path.getmtime(d) for d in deps)):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
           "-shared", "-o", tmp] + srcs
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class Grid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32),
                ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
                ("bc", C.c_int32), ("recon", C.c_int32), ("gamma", C.c_double), ("cfl", C.c_double)]


class Params(C.Structure):
    _fields_ = [("w", C.c_int32), ("r", C.c_int32), ("h", C.c_int32), ("W", C.c_int32),
                ("f", C.c_double), ("filter_orders", C.c_int32 * 3), ("n_filter_orders", C.c_int32),
                ("filter_max_sweeps", C.c_int32), ("filter_eps", C.c_double),
                ("eig_rel_cutoff", C.c_double), ("lsq_rel_cutoff", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        P = C.POINTER
        d, i32, i64, u8 = P(C.c_double), C.c_int32, C.c_int64, P(C.c_uint8)
        sig = {
            "orc_pressure": (C.c_double, [i32, C.c_double, d]),
            "orc_physical_flux": (None, [i32, i32, C.c_double, d, d]),
            "orc_minmod": (C.c_double, [C.c_double, C.c_double]),
            "orc_muscl_faces": (None, [C.c_double, C.c_double, C.c_double, d, d]),
            "orc_rusanov": (None, [i32, i32, C.c_double, d, d, d]),
            "orc_rhs": (None, [P(Grid), d, d]),
            "orc_dt": (C.c_double, [P(Grid), d]),
            "orc_positivity": (i64, [P(Grid), d]),
            "orc_full_step": (None, [P(Grid), d, C.c_double, d]),
            "orc_masked_step": (None, [P(Grid), d, C.c_double, u8, i32, d]),
            "orc_dilate_cross": (None, [P(Grid), u8, i32, u8]),
            "orc_dilate_square": (None, [P(Grid), u8, i32, u8]),
            "orc_select": (i64, [d, i64, i64, u8]),
            "orc_select_rre": (i64, [d, i64, C.c_double, u8]),
            "orc_odeim": (i32, [d, i64, i32, i64, i32, C.c_double, C.c_void_p, C.c_void_p]),
            "orc_n_g": (i64, [C.c_double, i64]),
            "orc_lsq": (i32, [d, i64, i32, d, C.c_double, d]),
            "orc_svd": (None, [d, i64, i32, d, d, d]),
            "orc_pod": (i32, [d, i64, i32, i32, C.c_double, d, d, d]),
            "orc_shapiro_1d": (None, [d, i32, i32, i32, d]),
            "orc_gram": (None, [d, i32, i64, d, d]),
            "orc_project": (None, [d, i64, i32, d, i32, d]),
            "orc_seam_filter": (i64, [P(Grid), P(Params), d, d, u8, u8, P(C.c_int32)]),
            "orc_run_create": (C.c_void_p, [P(Grid), P(Params), d]),
            "orc_run_destroy": (None, [C.c_void_p]),
            "orc_run_step": (i32, [C.c_void_p, C.c_double]),
            "orc_run_set_full_period": (None, [C.c_void_p, i32]),
            "orc_run_set_rre": (None, [C.c_void_p, C.c_double]),
            "orc_run_set_odeim": (None, [C.c_void_p, i32]),
            "orc_run_points": (i32, [C.c_void_p, C.c_void_p]),
            "orc_run_k": (i64, [C.c_void_p]),
            "orc_run_state": (None, [C.c_void_p, d]),
            "orc_run_mask": (None, [C.c_void_p, u8]),
            "orc_run_mask_used": (None, [C.c_void_p, u8]),
            "orc_run_eps": (None, [C.c_void_p, d]),
            "orc_run_reff": (i32, [C.c_void_p]),
            "orc_run_basis": (None, [C.c_void_p, d]),
            "orc_run_psi": (None, [C.c_void_p, d]),
            "orc_run_sigma": (None, [C.c_void_p, d]),
            "orc_run_y": (i32, [C.c_void_p, d]),
            "orc_run_dt": (C.c_double, [C.c_void_p]),
            "orc_run_filter_stats": (None, [C.c_void_p, P(C.c_int64), P(C.c_int32)]),
            "orc_run_set_window": (None, [C.c_void_p, i64, d, i32, u8]),
            "orc_roe": (i32, [i32, i32, C.c_double, d, d, d]),
            "orc_rhs2": (i32, [P(Grid), i32, d, d]),
            "orc_bdf_residual": (None, [P(Grid), i32, i32, C.c_double, d, d, d, d]),
            "orc_newton": (i32, [P(Grid), i32, i32, C.c_double, d, d, C.c_void_p, d, C.c_double, i32, d]),
            "orc_seam_filter_implicit": (i64, [P(Grid), P(Params), i32, i32, C.c_double, d, d, d, u8, u8,
                                               P(C.c_int32)]),
            "orc_run_set_implicit": (None, [C.c_void_p, i32, C.c_double, C.c_double, i32, C.c_double, i32]),
            "orc_run_implicit_stats": (None, [C.c_void_p, P(C.c_int32), P(C.c_int64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], (a.dtype, a.flags)
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u8(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def grid_of(wl) -> Grid:
    return Grid(wl.dim, wl.nx, wl.ny if wl.dim == 2 else 1, wl.x0, wl.x1, wl.y0, wl.y1,
                wl.bc, wl.recon, wl.gamma, wl.cfl)


def params_of(wl) -> Params:
    fo = (C.c_int32 * 3)(*(list(wl.filter_orders) + [0, 0, 0])[:3])
    return Params(wl.w, wl.r, wl.h, wl.W, wl.f, fo, len(wl.filter_orders),
                  wl.filter_max_sweeps, wl.filter_eps, wl.eig_rel_cutoff, wl.lsq_rel_cutoff)


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------- thin functional API ----------------
def pressure(dim, gamma, U):
    U = _c(U)
    return lib().orc_pressure(dim, gamma, _d(U))


def physical_flux(dim, axis, gamma, U):
    U = _c(U)
    F = np.zeros(dim + 2)
    lib().orc_physical_flux(dim, axis, gamma, _d(U), _d(F))
    return F


def minmod(a, b):
    return lib().orc_minmod(a, b)


def muscl_faces(um1, u0, up1):
    lf, rf = C.c_double(), C.c_double()
    lib().orc_muscl_faces(um1, u0, up1, C.byref(lf), C.byref(rf))
    return lf.value, rf.value


def rusanov(dim, axis, gamma, UL, UR):
    UL, UR = _c(UL), _c(UR)
    F = np.zeros(dim + 2)
    lib().orc_rusanov(dim, axis, gamma, _d(UL), _d(UR), _d(F))
    return F


def rhs(wl, q):
    q = _c(q)
    L = np.empty_like(q)
    g = grid_of(wl)
    lib().orc_rhs(C.byref(g), _d(q), _d(L))
    return L


def dt(wl, q):
    q = _c(q)
    g = grid_of(wl)
    return lib().orc_dt(C.byref(g), _d(q))


def positivity(wl, q):
    q = _c(q)
    g = grid_of(wl)
    return lib().orc_positivity(C.byref(g), _d(q))


def full_step(wl, q, dt_):
    q = _c(q)
    out = np.empty_like(q)
    g = grid_of(wl)
    lib().orc_full_step(C.byref(g), _d(q), dt_, _d(out))
    return out


def masked_step(wl, q, dt_, mask_T, h=None):
    q = _c(q)
    out = np.empty_like(q)
    m = np.ascontiguousarray(mask_T, dtype=np.uint8)
    g = grid_of(wl)
    lib().orc_masked_step(C.byref(g), _d(q), dt_, _u8(m), wl.h if h is None else h, _d(out))
    return out


def dilate_cross(wl, mask, h):
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    out = np.empty_like(m)
    g = grid_of(wl)
    lib().orc_dilate_cross(C.byref(g), _u8(m), h, _u8(out))
    return out


def dilate_square(wl, mask, W):
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    out = np.empty_like(m)
    g = grid_of(wl)
    lib().orc_dilate_square(C.byref(g), _u8(m), W, _u8(out))
    return out


def n_g(f, N):
    return lib().orc_n_g(f, N)


def select(eps, n_g_):
    e = _c(eps)
    out = np.empty(e.size, dtype=np.uint8)
    k = lib().orc_select(_d(e), e.size, n_g_, _u8(out))
    return out, k


def odeim(phi, N, n_p, cut=1e-12):
    """ODEIM points of phi (m x D array: column-major D x m), DOF e in cell e mod N (A36)."""
    phi = _c(phi)
    m, D = phi.shape
    cells = np.zeros(n_p, dtype=np.int32)
    rows = np.zeros(n_p, dtype=np.int64)
    k = lib().orc_odeim(_d(phi), D, m, N, n_p, cut, cells.ctypes.data_as(C.c_void_p),
                        rows.ctypes.data_as(C.c_void_p))
    if k < 0:
        raise ValueError("orc_odeim: n_p > N or m < 1")
    return cells, rows


def select_rre(eps, delta):
    e = _c(eps)
    out = np.empty(e.size, dtype=np.uint8)
    k = lib().orc_select_rre(_d(e), e.size, delta, _u8(out))
    return out, k


def _colmajor(A):
    A = np.asarray(A, dtype=np.float64)
    return np.ascontiguousarray(A.T), A.shape  # rows of A.T are columns of A


def lsq(A, b, cut=1e-12):
    At, (m, n) = _colmajor(A)
    b = _c(b)
    x = np.zeros(n)
    rank = lib().orc_lsq(_d(At), m, n, _d(b), cut, _d(x))
    return x, rank


def svd(X):
    Xt, (m, n) = _colmajor(X)
    U = np.zeros((n, m))
    S = np.zeros(n)
    V = np.zeros((n, n))
    lib().orc_svd(_d(Xt), m, n, _d(U), _d(S), _d(V))
    return U.T.copy(), S, V.T.copy()


def pod(X, r, cut=1e-8):
    Xt, (m, w) = _colmajor(X)
    Phi = np.zeros((r, m))
    S = np.zeros(w)
    V = np.zeros((w, w))
    reff = lib().orc_pod(_d(Xt), m, w, r, cut, _d(Phi), _d(S), _d(V))
    return Phi[:reff].T.copy(), S, V.T.copy(), reff


def gram(S, rho=None):
    """S: (ncol, rows) array; C = (S - rho)(S - rho)^T with compensated sums."""
    S = _c(S)
    ncol, rows = S.shape
    C_ = np.zeros((ncol, ncol))
    r = None if rho is None else _c(rho)
    lib().orc_gram(_d(S), ncol, rows, None if r is None else _d(r), _d(C_))
    return C_


def project(Phi, S):
    """Phi: (m, D), S: (ncol, D) arrays; C = Phi S^T (m x ncol) with compensated sums."""
    Phi = _c(Phi)
    S = _c(S)
    m, D = Phi.shape
    ncol = S.shape[0]
    assert S.shape[1] == D
    C_ = np.zeros((m, ncol))
    lib().orc_project(_d(Phi), D, m, _d(S), ncol, _d(C_))
    return C_


def shapiro_1d(line, order, periodic=False):
    line = _c(line)
    out = np.empty_like(line)
    lib().orc_shapiro_1d(_d(line), line.size, order, int(periodic), _d(out))
    return out


def seam_filter(wl, v, F, mask_S):
    v = _c(v).copy()
    F = _c(F)
    m = np.ascontiguousarray(mask_S, dtype=np.uint8)
    kept = np.zeros(wl.N, dtype=np.uint8)
    sweeps = (C.c_int32 * 3)()
    g, p = grid_of(wl), params_of(wl)
    lib().orc_seam_filter(C.byref(g), C.byref(p), _d(v), _d(F), _u8(m), _u8(kept), sweeps)
    return v, kept, list(sweeps)


def roe(dim, axis, gamma, UL, UR):
    UL, UR = _c(UL), _c(UR)
    F = np.zeros(dim + 2)
    rc = lib().orc_roe(dim, axis, gamma, _d(UL), _d(UR), _d(F))
    if rc != 0:
        raise ValueError("orc_roe: non-admissible Roe average")
    return F


def rhs2(wl, q, flux=1):
    q = _c(q)
    L = np.empty_like(q)
    g = grid_of(wl)
    lib().orc_rhs2(C.byref(g), flux, _d(q), _d(L))
    return L


def bdf_residual(wl, q, qm1, qm2, dt_, order=2, flux=1):
    q, qm1 = _c(q), _c(qm1)
    qm2 = _c(qm1 if qm2 is None else qm2)
    R = np.empty_like(q)
    g = grid_of(wl)
    lib().orc_bdf_residual(C.byref(g), flux, order, dt_, _d(q), _d(qm1), _d(qm2), _d(R))
    return R


def newton(wl, q0, qm1, qm2, dt_, order=2, flux=1, mask=None, tol=1e-12, maxit=30):
    """Newton-Krylov root of R_k (cells of mask; None: all).  Returns (q, iterations, stats)."""
    q = _c(q0).copy()
    qm1 = _c(qm1)
    qm2 = _c(qm1 if qm2 is None else qm2)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    st = np.zeros(2)
    g = grid_of(wl)
    its = lib().orc_newton(C.byref(g), flux, order, dt_, _d(qm1), _d(qm2),
                           None if m is None else m.ctypes.data_as(C.c_void_p), _d(q), tol, maxit, _d(st))
    return q, its, st


def seam_filter_implicit(wl, v, qm1, qm2, mask_S, dt_, order=2, flux=1):
    v = _c(v).copy()
    qm1 = _c(qm1)
    qm2 = _c(qm1 if qm2 is None else qm2)
    m = np.ascontiguousarray(mask_S, dtype=np.uint8)
    kept = np.zeros(wl.N, dtype=np.uint8)
    sweeps = (C.c_int32 * 3)()
    g, p = grid_of(wl), params_of(wl)
    lib().orc_seam_filter_implicit(C.byref(g), C.byref(p), flux, order, dt_, _d(qm1), _d(qm2), _d(v),
                                   _u8(m), _u8(kept), sweeps)
    return v, kept, list(sweeps)


class Run:
    """Algorithm 1 (explicit; z = wl.z, 0 = infinity) driver of the oracle."""

    def __init__(self, wl, q0):
        self.wl = wl
        self._g = grid_of(wl)
        self._p = params_of(wl)
        q0 = _c(q0)
        self.h = lib().orc_run_create(C.byref(self._g), C.byref(self._p), _d(q0))
        if getattr(wl, "z", 0) > 0:
            lib().orc_run_set_full_period(self.h, int(wl.z))
        if getattr(wl, "delta", 0.0) > 0.0:
            lib().orc_run_set_rre(self.h, float(wl.delta))
        if getattr(wl, "n_p", 0) > 0:
            lib().orc_run_set_odeim(self.h, int(wl.n_p))
        if getattr(wl, "hdm", "explicit") == "implicit":
            lib().orc_run_set_implicit(self.h, int(wl.flux), float(wl.dt), float(wl.eps_y), int(wl.j_max),
                                       float(wl.newton_tol), int(wl.newton_maxit))

    def implicit_stats(self):
        """(J of the last step, total Newton iterations so far)."""
        J = C.c_int32()
        its = C.c_int64()
        lib().orc_run_implicit_stats(self.h, C.byref(J), C.byref(its))
        return J.value, its.value

    def __del__(self):
        h, self.h = getattr(self, "h", None), None
        if h:
            try:
                lib().orc_run_destroy(h)
            except TypeError:  # interpreter shutdown: module globals already torn down
                pass

    def step(self, dt_override: float = 0.0) -> int:
        return lib().orc_run_step(self.h, dt_override)

    @property
    def k(self):
        return lib().orc_run_k(self.h)

    def state(self):
        q = np.empty((self.wl.c, self.wl.N))
        lib().orc_run_state(self.h, _d(q))
        return q

    def mask(self):
        m = np.empty(self.wl.N, dtype=np.uint8)
        lib().orc_run_mask(self.h, _u8(m))
        return m

    def points(self):
        """DOF rows of the ODEIM points chosen for the next step (empty without ODEIM)."""
        rows = np.zeros(max(int(getattr(self.wl, "n_p", 0)), 1), dtype=np.int64)
        k = lib().orc_run_points(self.h, rows.ctypes.data_as(C.c_void_p))
        return rows[:k]

    def mask_used(self):
        m = np.empty(self.wl.N, dtype=np.uint8)
        lib().orc_run_mask_used(self.h, _u8(m))
        return m

    def eps(self):
        e = np.empty(self.wl.N)
        lib().orc_run_eps(self.h, _d(e))
        return e

    def reff(self):
        return lib().orc_run_reff(self.h)

    def basis(self):
        r = self.reff()
        Phi = np.empty((r, self.wl.D))
        lib().orc_run_basis(self.h, _d(Phi))
        return Phi.T.copy()

    def psi(self):
        p = np.empty((self.wl.c, self.wl.N))
        lib().orc_run_psi(self.h, _d(p))
        return p

    def sigma(self):
        s = np.empty(self.wl.w)
        lib().orc_run_sigma(self.h, _d(s))
        return s

    def y(self):
        y = np.zeros(max(self.wl.r, 1))
        n = lib().orc_run_y(self.h, _d(y))
        return y[:n].copy()

    def dt(self):
        return lib().orc_run_dt(self.h)

    def filter_stats(self):
        kept = C.c_int64()
        sw = (C.c_int32 * 3)()
        lib().orc_run_filter_stats(self.h, C.byref(kept), sw)
        return kept.value, list(sw)

    def set_window(self, k: int, snaps: np.ndarray, mask_next: np.ndarray):
        s = _c(snaps)
        assert s.shape[0] == self.wl.w + 1
        m = np.ascontiguousarray(mask_next, dtype=np.uint8)
        lib().orc_run_set_window(self.h, k, _d(s), s.shape[0], _u8(m))
