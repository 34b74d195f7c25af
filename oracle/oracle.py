"""ctypes front end of the CPU oracle (oracle/clampqp_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's CPU legs.
The product package (paper_2311_18056_b200/) never imports this module.

The classes mirror the reference's public types so that tests read like the reference's own:
  QProblem / Solution / SolveReport / SolverSettings  (problem.hpp:31-71, solver.hpp:43-67)
  Solver                                             (solver.hpp:107-135, solver.cpp:180-218)
Matrices cross the boundary column-major (numpy order="F"), like Eigen::MatrixXd.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBS = {}

c_double_p = C.POINTER(C.c_double)
c_int_p = C.POINTER(C.c_int)


class _Settings(C.Structure):
    _fields_ = [
        ("eps_prim", C.c_double), ("eps_dual", C.c_double),
        ("check_interval", C.c_int), ("max_iters", C.c_int),
        ("sigma", C.c_double), ("grid_points", C.c_int),
        ("rho_switch_threshold", C.c_double), ("adaptive_rho", C.c_int),
        ("eq_enabled", C.c_int), ("eq_max_passes", C.c_int), ("eq_tol", C.c_double),
    ]


class _ReportHead(C.Structure):
    _fields_ = [
        ("status", C.c_int), ("iterations", C.c_int),
        ("r_prim", C.c_double), ("r_dual", C.c_double),
        ("n_trace", C.c_int), ("n_hist", C.c_int), ("wall_ms", C.c_double),
    ]


def build(force: bool = False) -> None:
    """Compile liboracle.so / liboracle_v3.so next to this file (gcc via oracle/Makefile)."""
    if force or not all(os.path.exists(os.path.join(_HERE, n))
                        for n in ("liboracle.so", "liboracle_v3.so")):
        subprocess.check_call(["make", "-C", _HERE, "-s"] + (["-B"] if force else []))


def lib(variant: str = "ref") -> C.CDLL:
    """variant 'ref' = compiled like the reference (-O3 -DNDEBUG); 'v3' = -march=x86-64-v3."""
    if variant in _LIBS:
        return _LIBS[variant]
    name = {"ref": "liboracle.so", "v3": "liboracle_v3.so"}[variant]
    path = os.path.join(_HERE, name)
    if not os.path.exists(path):
        build()
    L = C.CDLL(path)
    L.orc_rng_next_u64.restype = C.c_uint64
    L.orc_rng_uniform.restype = C.c_double
    L.orc_rng_uniform_range.restype = C.c_double
    L.orc_rng_uniform_range.argtypes = [C.c_void_p, C.c_double, C.c_double]
    L.orc_rng_normal.restype = C.c_double
    L.orc_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
    L.orc_gen_random_dense_qp.argtypes = [C.c_int, C.c_uint64] + [c_double_p] * 6
    L.orc_precompute_all.restype = C.c_void_p
    L.orc_precompute_all.argtypes = [C.c_int, C.c_int] + [c_double_p] * 5 + [
        C.c_int, C.c_double, C.c_int, C.c_int, C.c_double, c_int_p]
    L.orc_cache_free.argtypes = [C.c_void_p]
    L.orc_cache_ptr.restype = c_double_p
    L.orc_cache_ptr.argtypes = [C.c_void_p, C.c_int, C.c_int]
    for f in ("orc_cache_n", "orc_cache_m", "orc_cache_L", "orc_cache_initial_index"):
        getattr(L, f).argtypes = [C.c_void_p]
    L.orc_cache_cost_scale.restype = C.c_double
    L.orc_cache_cost_scale.argtypes = [C.c_void_p]
    L.orc_cache_sigma.restype = C.c_double
    L.orc_cache_sigma.argtypes = [C.c_void_p]
    L.orc_refresh_z.argtypes = [C.c_void_p, c_double_p]
    L.orc_cache_update_vectors.argtypes = [C.c_void_p] + [c_double_p] * 3
    L.orc_rho_nominal.restype = C.c_double
    L.orc_rho_nominal.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double] + [c_double_p] * 6 + [C.c_double]
    L.orc_select_layer.argtypes = [C.c_double, c_double_p, C.c_int, C.c_int, C.c_double]
    L.orc_nearest_grid_index.argtypes = [c_double_p, C.c_int, C.c_double]
    L.orc_build_penalty_grid.argtypes = [C.c_int, c_double_p]
    L.orc_build_kkt_inverse.argtypes = [C.c_int, C.c_int, c_double_p, c_double_p, C.c_double,
                                        c_double_p, c_double_p]
    L.orc_build_layer.argtypes = [C.c_int, C.c_int, c_double_p, c_double_p, c_double_p, C.c_double,
                                  c_double_p, c_double_p, c_double_p, c_double_p, c_double_p]
    L.orc_layer_bias.argtypes = [C.c_int, C.c_int] + [c_double_p] * 4
    L.orc_iterate.argtypes = [C.c_int] + [c_double_p] * 6
    L.orc_residuals.argtypes = [C.c_int, C.c_int] + [c_double_p] * 8
    L.orc_warm_start.argtypes = [C.c_void_p, c_double_p, c_double_p, C.c_int, c_double_p]
    L.orc_run_loop.argtypes = [C.c_void_p, C.POINTER(_Settings)] + [c_double_p] * 5 + [
        c_double_p, c_int_p, C.c_int, C.c_int, C.POINTER(_ReportHead),
        c_double_p, c_double_p, c_double_p, c_int_p, c_int_p, c_int_p, c_double_p, c_double_p,
        c_int_p, C.c_int]
    L.orc_validate.argtypes = [C.c_int, C.c_int] + [c_double_p] * 5
    L.orc_ruiz_scaling.argtypes = [C.c_int, C.c_int, c_double_p, c_double_p, C.c_int, C.c_double,
                                   c_double_p, c_double_p, c_double_p]
    L.orc_admm_step_reordered.argtypes = [C.c_int, C.c_int] + [c_double_p] * 5 + [
        C.c_double] + [c_double_p] * 7
    L.orc_check_settings.argtypes = [C.POINTER(_Settings)]
    _LIBS[variant] = L
    return L


def _f(a) -> np.ndarray:
    """float64, column-major, contiguous."""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(c_double_p)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(c_int_p)


# ---------------------------------------------------------------------------------------------
# bench::Rng (bench.hpp:29-47, bench.cpp:58-87)
# ---------------------------------------------------------------------------------------------
class Rng:
    def __init__(self, seed: int, variant: str = "ref"):
        self._L = lib(variant)
        self._buf = C.create_string_buffer(self._L.orc_rng_sizeof())
        self._L.orc_rng_seed(self._buf, C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF))

    def next_u64(self) -> int:
        return int(self._L.orc_rng_next_u64(self._buf))

    def uniform(self, lo: Optional[float] = None, hi: Optional[float] = None) -> float:
        if lo is None:
            return float(self._L.orc_rng_uniform(self._buf))
        return float(self._L.orc_rng_uniform_range(self._buf, lo, hi))

    def normal(self) -> float:
        return float(self._L.orc_rng_normal(self._buf))

    def normal_vector(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self._L.orc_rng_normal_vector(self._buf, C.c_int(n), _p(out))
        return out

    def normal_matrix(self, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), dtype=np.float64, order="F")
        self._L.orc_rng_normal_matrix(self._buf, C.c_int(rows), C.c_int(cols), _p(out))
        return out


# ---------------------------------------------------------------------------------------------
# problem.hpp types
# ---------------------------------------------------------------------------------------------
@dataclass
class QProblem:
    """min 0.5 y'Hy + g'y  s.t.  c <= Gy <= d   (problem.hpp:31-40)."""
    H: np.ndarray
    g: np.ndarray
    G: np.ndarray
    c: np.ndarray
    d: np.ndarray

    def __post_init__(self):
        self.H = _f(self.H)
        self.G = _f(self.G)
        self.g = np.ascontiguousarray(self.g, dtype=np.float64).reshape(-1)
        self.c = np.ascontiguousarray(self.c, dtype=np.float64).reshape(-1)
        self.d = np.ascontiguousarray(self.d, dtype=np.float64).reshape(-1)
        if self.H.ndim != 2:
            self.H = self.H.reshape(1, 1) if self.H.size == 1 else self.H
        if self.G.ndim != 2:
            self.G = self.G.reshape(1, -1)

    @property
    def n(self) -> int:
        return self.H.shape[0]

    @property
    def m(self) -> int:
        return self.G.shape[0]

    def copy(self) -> "QProblem":
        return QProblem(self.H.copy(order="F"), self.g.copy(), self.G.copy(order="F"),
                        self.c.copy(), self.d.copy())


class ProblemError(RuntimeError):
    """problem.hpp:73-92; `code` is the ProblemError::Code name."""
    CODES = {1: "DimensionMismatch", 2: "NonSymmetricH", 3: "NonPositiveDefiniteH",
             4: "InvertedBounds", 5: "NonFiniteEntry"}

    def __init__(self, code: int):
        self.code = self.CODES.get(code, str(code))
        super().__init__(self.code)


SOLVED, MAX_ITERS, INVALID = 0, 1, 2  # SolveStatus (problem.hpp:51)


@dataclass
class Solution:
    y: np.ndarray = field(default_factory=lambda: np.zeros(0))
    z: np.ndarray = field(default_factory=lambda: np.zeros(0))
    lam: np.ndarray = field(default_factory=lambda: np.zeros(0))
    status: int = INVALID
    iterations: int = 0
    r_prim: float = 0.0
    r_dual: float = 0.0
    rho_trace: List[Tuple[int, int]] = field(default_factory=list)  # (iteration, grid_index)


@dataclass
class SolveReport:
    solution: Solution
    wall_ms: float = 0.0
    residual_history: List[Tuple[int, float, float, int]] = field(default_factory=list)


@dataclass
class SolverSettings:
    """solver.hpp:43-53 (defaults identical)."""
    eps_prim: float = 1e-6
    eps_dual: float = 1e-6
    check_interval: int = 25
    max_iters: int = 4000
    sigma: float = 1e-6
    grid_points: int = 13
    rho_switch_threshold: float = 5.0
    adaptive_rho: bool = True
    eq_enabled: bool = True
    eq_max_passes: int = 10
    eq_tol: float = 1e-3

    def _c(self) -> _Settings:
        return _Settings(self.eps_prim, self.eps_dual, self.check_interval, self.max_iters,
                         self.sigma, self.grid_points, self.rho_switch_threshold,
                         int(self.adaptive_rho), int(self.eq_enabled), self.eq_max_passes,
                         self.eq_tol)


def validate(p: QProblem, variant: str = "ref") -> QProblem:
    """problem.cpp:121-164."""
    n, m = p.H.shape[0], p.G.shape[0]
    if (n < 1 or m < 1 or p.H.shape[1] != n or p.g.size != n or p.G.shape[1] != n
            or p.c.size != m or p.d.size != m):
        raise ProblemError(1)
    rc = lib(variant).orc_validate(n, m, _p(p.H), _p(p.g), _p(p.G), _p(p.c), _p(p.d))
    if rc:
        raise ProblemError(rc)
    return p


def gen_random_dense_qp(n: int, seed: int, variant: str = "ref", witness: bool = False):
    """bench.cpp:89-118."""
    if n < 4:
        raise ValueError("gen_random_dense_qp: n must be >= 4")
    m = 2 * (n // 4)
    H = np.empty((n, n), order="F"); g = np.empty(n)
    G = np.empty((m, n), order="F"); c = np.empty(m); d = np.empty(m); w = np.empty(n)
    lib(variant).orc_gen_random_dense_qp(n, C.c_uint64(seed), _p(H), _p(g), _p(G), _p(c), _p(d), _p(w))
    p = QProblem(H, g, G, c, d)
    return (p, w) if witness else p


# ---------------------------------------------------------------------------------------------
# layers.hpp
# ---------------------------------------------------------------------------------------------
def build_penalty_grid(n_points: int, variant: str = "ref") -> Tuple[np.ndarray, int]:
    """layers.cpp:22-36 -> (values, initial_index)."""
    if n_points < 2:
        raise ValueError("penalty grid needs at least 2 points")
    vals = np.empty(n_points)
    idx = lib(variant).orc_build_penalty_grid(n_points, _p(vals))
    return vals, idx


def nearest_grid_index(values, rho: float, variant: str = "ref") -> int:
    v = np.ascontiguousarray(values, dtype=np.float64)
    return int(lib(variant).orc_nearest_grid_index(_p(v), v.size, C.c_double(rho)))


def select_layer(rho_nom: float, values, current_index: int, threshold: float,
                 variant: str = "ref") -> int:
    v = np.ascontiguousarray(values, dtype=np.float64)
    return int(lib(variant).orc_select_layer(C.c_double(rho_nom), _p(v), v.size, current_index,
                                             C.c_double(threshold)))


def build_kkt_inverse(H, G, sigma: float, rho_vec, variant: str = "ref") -> np.ndarray:
    """layers.cpp:122-131; raises RuntimeError on factorisation failure."""
    H = _f(np.atleast_2d(H)); G = _f(np.atleast_2d(G))
    rho = np.ascontiguousarray(rho_vec, dtype=np.float64).reshape(-1)
    n, m = H.shape[0], G.shape[0]
    D = np.empty((n, n), order="F")
    if lib(variant).orc_build_kkt_inverse(n, m, _p(H), _p(G), C.c_double(sigma), _p(rho), _p(D)):
        raise RuntimeError("KKT factorization failed")
    return D


def build_layer(H, G, g, sigma: float, rho_vec, D, variant: str = "ref"):
    """layers.cpp:133-166 -> (W, GD, b)."""
    H = _f(np.atleast_2d(H)); G = _f(np.atleast_2d(G)); D = _f(np.atleast_2d(D))
    g = np.ascontiguousarray(g, dtype=np.float64).reshape(-1)
    rho = np.ascontiguousarray(rho_vec, dtype=np.float64).reshape(-1)
    n, m = H.shape[0], G.shape[0]
    dim = n + 2 * m
    W = np.empty((dim, dim), order="F"); GD = np.empty((m, n), order="F"); b = np.empty(dim)
    lib(variant).orc_build_layer(n, m, _p(H), _p(G), _p(g), C.c_double(sigma), _p(rho), _p(D),
                                 _p(W), _p(GD), _p(b))
    return W, GD, b


def layer_bias(D, GD, g, variant: str = "ref") -> np.ndarray:
    D = _f(np.atleast_2d(D)); GD = _f(np.atleast_2d(GD))
    g = np.ascontiguousarray(g, dtype=np.float64).reshape(-1)
    n, m = D.shape[0], GD.shape[0]
    b = np.empty(n + 2 * m)
    lib(variant).orc_layer_bias(n, m, _p(D), _p(GD), _p(g), _p(b))
    return b


def ruiz_scaling(H, G, max_passes: int = 10, tol: float = 1e-3, variant: str = "ref"):
    """layers.cpp:82-120 -> (E, F, cost_scale)."""
    H = _f(np.atleast_2d(H)); G = _f(np.atleast_2d(G))
    n, m = H.shape[0], G.shape[0]
    E = np.empty(n); F = np.empty(m); cs = C.c_double(0.0)
    lib(variant).orc_ruiz_scaling(n, m, _p(H), _p(G), max_passes, C.c_double(tol), _p(E), _p(F),
                                  C.byref(cs))
    return E, F, cs.value


class LayerCache:
    """layers.hpp:108-127; built by precompute_all (layers.cpp:189-228)."""

    def __init__(self, p: QProblem, grid_points: int = 13, sigma: float = 1e-6,
                 eq_enabled: bool = True, eq_max_passes: int = 10, eq_tol: float = 1e-3,
                 variant: str = "ref"):
        if grid_points < 2:
            raise ValueError("penalty grid needs at least 2 points")
        self._L = lib(variant)
        err = C.c_int(0)
        self._h = self._L.orc_precompute_all(p.n, p.m, _p(p.H), _p(p.g), _p(p.G), _p(p.c),
                                             _p(p.d), grid_points, C.c_double(sigma),
                                             int(eq_enabled), eq_max_passes, C.c_double(eq_tol),
                                             C.byref(err))
        if not self._h:
            raise RuntimeError("KKT factorization failed" if err.value == 1 else "bad grid")
        self.n, self.m, self.L = p.n, p.m, grid_points
        self.dim = self.n + 2 * self.m

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._L.orc_cache_free(h)

    def _arr(self, what: int, k: int, shape) -> np.ndarray:
        ptr = self._L.orc_cache_ptr(self._h, what, k)
        count = int(np.prod(shape))
        flat = np.ctypeslib.as_array(ptr, shape=(count,)).copy()
        return flat.reshape(shape, order="F")

    def W(self, k): return self._arr(0, k, (self.dim, self.dim))
    def D(self, k): return self._arr(1, k, (self.n, self.n))
    def GD(self, k): return self._arr(2, k, (self.m, self.n))
    def rho_vec(self, k): return self._arr(3, k, (self.m,))
    def b(self, k): return self._arr(4, k, (self.dim,))
    @property
    def Hs(self): return self._arr(5, 0, (self.n, self.n))
    @property
    def gs(self): return self._arr(6, 0, (self.n,))
    @property
    def Gs(self): return self._arr(7, 0, (self.m, self.n))
    @property
    def cs(self): return self._arr(8, 0, (self.m,))
    @property
    def ds(self): return self._arr(9, 0, (self.m,))
    @property
    def E(self): return self._arr(10, 0, (self.n,))
    @property
    def F(self): return self._arr(11, 0, (self.m,))
    @property
    def grid(self): return self._arr(12, 0, (self.L,))
    @property
    def c_tilde(self): return self._arr(13, 0, (self.dim,))
    @property
    def d_tilde(self): return self._arr(14, 0, (self.dim,))
    @property
    def initial_index(self): return int(self._L.orc_cache_initial_index(self._h))
    @property
    def cost_scale(self): return float(self._L.orc_cache_cost_scale(self._h))
    @property
    def sigma(self): return float(self._L.orc_cache_sigma(self._h))

    def update_vectors(self, g, c, d) -> None:
        """layers.cpp:177-187."""
        g = np.ascontiguousarray(g, dtype=np.float64).reshape(-1)
        c = np.ascontiguousarray(c, dtype=np.float64).reshape(-1)
        d = np.ascontiguousarray(d, dtype=np.float64).reshape(-1)
        if g.size != self.n or c.size != self.m or d.size != self.m:
            raise ValueError("update_vectors: dimension mismatch")
        self._L.orc_cache_update_vectors(self._h, _p(g), _p(c), _p(d))


def precompute_all(p: QProblem, grid_points: int = 13, sigma: float = 1e-6,
                   eq_enabled: bool = True, eq_max_passes: int = 10, eq_tol: float = 1e-3,
                   variant: str = "ref") -> LayerCache:
    return LayerCache(p, grid_points, sigma, eq_enabled, eq_max_passes, eq_tol, variant)


# ---------------------------------------------------------------------------------------------
# solver.hpp free functions
# ---------------------------------------------------------------------------------------------
def iterate(v, W, b, c_tilde, d_tilde, variant: str = "ref") -> np.ndarray:
    """solver.cpp:109-117."""
    W = _f(np.atleast_2d(W))
    v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1)
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
    lo = np.ascontiguousarray(c_tilde, dtype=np.float64).reshape(-1)
    hi = np.ascontiguousarray(d_tilde, dtype=np.float64).reshape(-1)
    dim = W.shape[0]
    if v.size != W.shape[1] or b.size != dim or lo.size != dim or hi.size != dim:
        raise ValueError("iterate: dimension mismatch")
    out = np.empty(dim)
    lib(variant).orc_iterate(dim, _p(v), _p(W), _p(b), _p(lo), _p(hi), _p(out))
    return out


def residuals(y, z, lam, p: QProblem, variant: str = "ref") -> Tuple[float, float]:
    """solver.cpp:119-124."""
    y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
    z = np.ascontiguousarray(z, dtype=np.float64).reshape(-1)
    lam = np.ascontiguousarray(lam, dtype=np.float64).reshape(-1)
    rp, rd = C.c_double(0), C.c_double(0)
    lib(variant).orc_residuals(p.n, p.m, _p(y), _p(z), _p(lam), _p(p.H), _p(p.g), _p(p.G),
                               C.byref(rp), C.byref(rd))
    return rp.value, rd.value


def rho_nominal(r_prim, r_dual, y, z, lam, p: QProblem, current_rho, variant: str = "ref") -> float:
    """solver.cpp:126-134."""
    y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
    z = np.ascontiguousarray(z, dtype=np.float64).reshape(-1)
    lam = np.ascontiguousarray(lam, dtype=np.float64).reshape(-1)
    return float(lib(variant).orc_rho_nominal(p.n, p.m, C.c_double(r_prim), C.c_double(r_dual),
                                              _p(y), _p(z), _p(lam), _p(p.H), _p(p.g), _p(p.G),
                                              C.c_double(current_rho)))


def admm_step_reordered(y, z, lam, H, g, G, c, d, sigma, rho_vec, variant: str = "ref"):
    """oracle.cpp:63-74 -- independent sequential ADMM step."""
    H = _f(np.atleast_2d(H)); G = _f(np.atleast_2d(G))
    arrs = [np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in (g, c, d, rho_vec, y, z, lam)]
    g, c, d, rho, y, z, lam = arrs
    n, m = H.shape[0], G.shape[0]
    yo, zo, lo = np.empty(n), np.empty(m), np.empty(m)
    rc = lib(variant).orc_admm_step_reordered(n, m, _p(H), _p(g), _p(G), _p(c), _p(d),
                                              C.c_double(sigma), _p(rho), _p(y), _p(z), _p(lam),
                                              _p(yo), _p(zo), _p(lo))
    if rc:
        raise RuntimeError("oracle: KKT factorization failed")
    return yo, zo, lo


def _run_loop(cache: LayerCache, s: SolverSettings, p: QProblem, v: np.ndarray,
              layer_index: int, early_exit: bool, total_iters: int):
    """solver.cpp:43-105. Returns (report, new_layer_index); v is updated in place."""
    n, m = cache.n, cache.m
    cap = total_iters // max(1, s.check_interval) + 2
    head = _ReportHead()
    y, z, lam = np.empty(n), np.empty(m), np.empty(m)
    t_it = np.zeros(cap, dtype=np.int32); t_ix = np.zeros(cap, dtype=np.int32)
    h_it = np.zeros(cap, dtype=np.int32); h_ix = np.zeros(cap, dtype=np.int32)
    h_rp = np.zeros(cap); h_rd = np.zeros(cap)
    idx = C.c_int(layer_index)
    cs = s._c()
    cache._L.orc_run_loop(cache._h, C.byref(cs), _p(p.H), _p(p.g), _p(p.G), _p(p.c), _p(p.d),
                          _p(v), C.byref(idx), int(early_exit), int(total_iters), C.byref(head),
                          _p(y), _p(z), _p(lam), _ip(t_it), _ip(t_ix), _ip(h_it), _p(h_rp),
                          _p(h_rd), _ip(h_ix), cap)
    sol = Solution(y, z, lam, head.status, head.iterations, head.r_prim, head.r_dual,
                   [(int(t_it[i]), int(t_ix[i])) for i in range(head.n_trace)])
    rep = SolveReport(sol, head.wall_ms,
                      [(int(h_it[i]), float(h_rp[i]), float(h_rd[i]), int(h_ix[i]))
                       for i in range(head.n_hist)])
    return rep, idx.value


def check_settings(s: SolverSettings) -> None:
    """solver.cpp:29-34."""
    if s.check_interval < 1:
        raise ValueError("check_interval must be >= 1")
    if s.max_iters < s.check_interval:
        raise ValueError("max_iters must be >= check_interval")


def warm_start(prev: Solution, cache: LayerCache) -> Tuple[np.ndarray, int]:
    """solver.cpp:144-156 -> (v, layer_index)."""
    y = np.ascontiguousarray(prev.y, dtype=np.float64).reshape(-1)
    lam = np.ascontiguousarray(prev.lam, dtype=np.float64).reshape(-1)
    if y.size != cache.n or lam.size != cache.m:
        raise ValueError("warm_start: dimension mismatch")
    v = np.zeros(cache.dim)
    last = prev.rho_trace[-1][1] if prev.rho_trace else -1
    idx = cache._L.orc_warm_start(cache._h, _p(y), _p(lam), last, _p(v))
    return v, int(idx)


def solve(p: QProblem, cache: LayerCache, s: SolverSettings,
          warm: Optional[Solution] = None) -> SolveReport:
    """solver.cpp:158-166."""
    check_settings(s)
    if p.n != cache.n or p.m != cache.m:
        return SolveReport(Solution(status=INVALID), 0.0, [])
    v, idx = np.zeros(cache.dim), cache.initial_index
    if warm is not None:
        v, idx = warm_start(warm, cache)
    rep, _ = _run_loop(cache, s, p, v, idx, True, s.max_iters)
    return rep


def fixed_iters(p: QProblem, cache: LayerCache, s: SolverSettings, k: int,
                warm: Optional[Solution] = None) -> SolveReport:
    """solver.cpp:168-178."""
    check_settings(s)
    if k < 1:
        raise ValueError("fixed_iters: k must be >= 1")
    if p.n != cache.n or p.m != cache.m:
        return SolveReport(Solution(status=INVALID), 0.0, [])
    v, idx = np.zeros(cache.dim), cache.initial_index
    if warm is not None:
        v, idx = warm_start(warm, cache)
    rep, _ = _run_loop(cache, s, p, v, idx, False, k)
    return rep


class Solver:
    """solver.hpp:107-135 / solver.cpp:180-218 (CPU oracle)."""

    def __init__(self, p: QProblem, settings: Optional[SolverSettings] = None,
                 variant: str = "ref"):
        self.settings = settings or SolverSettings()
        self.problem = validate(p.copy(), variant)
        check_settings(self.settings)
        s = self.settings
        self.cache = LayerCache(self.problem, s.grid_points, s.sigma, s.eq_enabled,
                                s.eq_max_passes, s.eq_tol, variant)
        self.cold_start()

    def cold_start(self) -> None:
        self.v = np.zeros(self.cache.dim)
        self.layer_index = self.cache.initial_index

    def warm_start(self, prev: Solution) -> None:
        self.v, self.layer_index = warm_start(prev, self.cache)

    def refresh_z(self) -> None:
        """solver.cpp:197-200: z_s <- G_s y_s."""
        self.cache._L.orc_refresh_z(self.cache._h, _p(self.v))

    def solve(self) -> SolveReport:
        rep, self.layer_index = _run_loop(self.cache, self.settings, self.problem, self.v,
                                          self.layer_index, True, self.settings.max_iters)
        return rep

    def fixed_iters(self, k: int) -> SolveReport:
        if k < 1:
            raise ValueError("fixed_iters: k must be >= 1")
        rep, self.layer_index = _run_loop(self.cache, self.settings, self.problem, self.v,
                                          self.layer_index, False, k)
        return rep

    def update_vectors(self, g, c, d) -> None:
        self.cache.update_vectors(g, c, d)
        self.problem.g = np.ascontiguousarray(g, dtype=np.float64).reshape(-1).copy()
        self.problem.c = np.ascontiguousarray(c, dtype=np.float64).reshape(-1).copy()
        self.problem.d = np.ascontiguousarray(d, dtype=np.float64).reshape(-1).copy()

    @property
    def state(self) -> np.ndarray:
        return self.v
