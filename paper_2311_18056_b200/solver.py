"""Host-side mirror of the reference's `clampqp::Solver` over the C ABI (include/cqp_b200.h).

Same names, argument meaning and error behaviour as
/root/reference/proj/include/clampqp/solver.hpp:107-135 and the Python module the reference
ships (python/bindings.cpp:101-112), so tests read like the reference's own.  All compute runs
in libcqp_b200.so on the GPU; this file only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _lib
from ._lib import CqpResidualSample, CqpResult, CqpRhoSwitch, CqpSettings, c_double_p

SOLVED, MAX_ITERS, INVALID = 0, 1, 2  # SolveStatus, problem.hpp:51


class ProblemError(RuntimeError):
    """problem.hpp:73-92."""
    CODES = {1: "DimensionMismatch", 2: "NonSymmetricH", 3: "NonPositiveDefiniteH",
             4: "InvertedBounds", 5: "NonFiniteEntry"}

    def __init__(self, code: int, msg: str):
        self.code = self.CODES.get(code, str(code))
        super().__init__(f"{self.code}: {msg}")


class CudaError(RuntimeError):
    pass


def _raise(rc: int) -> None:
    """Map cqp_status onto the reference's exception types."""
    if rc == 0:
        return
    msg = _lib.last_error()
    if 1 <= rc <= 5:
        raise ProblemError(rc, msg)
    if rc in (6, 8):
        raise ValueError(msg)              # std::invalid_argument
    if rc == 7:
        raise RuntimeError(msg)            # std::runtime_error (factorisation)
    if rc == 10:
        raise MemoryError(msg)
    raise CudaError(msg)


@dataclass
class SolverSettings:
    """solver.hpp:43-53 (identical defaults)."""
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

    def _c(self) -> CqpSettings:
        return CqpSettings(self.eps_prim, self.eps_dual, self.check_interval, self.max_iters,
                           self.sigma, self.grid_points, self.rho_switch_threshold,
                           int(self.adaptive_rho), int(self.eq_enabled), self.eq_max_passes,
                           self.eq_tol)


@dataclass
class Solution:
    """problem.hpp:62-71."""
    y: np.ndarray
    z: np.ndarray
    lam: np.ndarray
    status: int = INVALID
    iterations: int = 0
    r_prim: float = 0.0
    r_dual: float = 0.0
    rho_trace: List[Tuple[int, int]] = field(default_factory=list)


@dataclass
class SolveReport:
    """solver.hpp:63-67 (+ the kernel-only CUDA-event time)."""
    solution: Solution
    wall_ms: float = 0.0
    residual_history: List[Tuple[int, float, float, int]] = field(default_factory=list)
    kernel_us: float = 0.0


def _vec(a, size: Optional[int] = None, name: str = "vector") -> np.ndarray:
    v = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    if size is not None and v.size != size:
        raise ValueError(f"{name}: dimension mismatch")
    return v


def _mat(a) -> np.ndarray:
    return np.asfortranarray(np.atleast_2d(np.asarray(a, dtype=np.float64)))


def _p(a: np.ndarray):
    return a.ctypes.data_as(c_double_p)


class Solver:
    """GPU `clampqp::Solver`: build once, then solve / update_vectors + refresh_z + fixed_iters."""

    def __init__(self, H, g, G, c, d, settings: Optional[SolverSettings] = None,
                 device: int = -1, layers: Optional[dict] = None):
        """Solver(QProblem, SolverSettings) (solver.cpp:180-186).

        `layers`: optional precomputed LayerCache fields (W, D, GD lists, grid, initial_index,
        Gs, E, F, cost_scale) -> cqp_create_from_layers; otherwise the offline stage runs on
        the device (cqp_create)."""
        self._L = _lib.load()
        self._h = C.c_void_p()
        self.settings = settings or SolverSettings()
        H, G = _mat(H), _mat(G)
        g, c, d = _vec(g), _vec(c), _vec(d)
        n, m = H.shape[0], G.shape[0]
        if (n < 1 or m < 1 or H.shape[1] != n or g.size != n or G.shape[1] != n or c.size != m
                or d.size != m):
            raise ProblemError(1, "inconsistent problem dimensions")
        self.n, self.m = n, m
        cs = self.settings._c()
        if layers is None:
            rc = self._L.cqp_create(C.byref(self._h), n, m, _p(H), _p(g), _p(G), _p(c), _p(d),
                                    C.byref(cs), device)
        else:
            Lk = len(layers["W"])
            keep = []

            def ptr_array(mats):
                arr = (c_double_p * Lk)()
                for k, a in enumerate(mats):
                    a = _mat(a)
                    keep.append(a)
                    arr[k] = _p(a)
                return arr

            Wp, Dp, GDp = ptr_array(layers["W"]), ptr_array(layers["D"]), ptr_array(layers["GD"])
            grid = _vec(layers["grid"], Lk)
            Gs, E, F = _mat(layers["Gs"]), _vec(layers["E"], n), _vec(layers["F"], m)
            rc = self._L.cqp_create_from_layers(
                C.byref(self._h), n, m, Lk, Wp, Dp, GDp, _p(grid), int(layers["initial_index"]),
                _p(H), _p(g), _p(G), _p(c), _p(d), _p(Gs), _p(E), _p(F),
                C.c_double(float(layers["cost_scale"])), C.byref(cs), device)
        if rc:
            self._h = C.c_void_p()
            _raise(rc)
        Lc = C.c_int()
        self._L.cqp_dims(self._h, None, None, C.byref(Lc))
        self.L = Lc.value

    def close(self) -> None:
        """Frees the handle.  BatchSolvers built on this solver share its ladder: they are closed
        first, so that none is left holding a dangling handle."""
        for ref in list(self.__dict__.get("_dependents", [])):
            dep = ref()
            if dep is not None:
                dep.close()
        self.__dict__["_dependents"] = []
        h, self._h = getattr(self, "_h", None), C.c_void_p()
        if h:
            self._L.cqp_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- solver.hpp:111-121 ----
    def cold_start(self) -> None:
        _raise(self._L.cqp_cold_start(self._h))

    def warm_start(self, prev: Solution) -> None:
        y, lam = _vec(prev.y), _vec(prev.lam)
        if y.size != self.n or lam.size != self.m:
            raise ValueError("warm_start: dimension mismatch")
        last = prev.rho_trace[-1][1] if prev.rho_trace else -1
        _raise(self._L.cqp_warm_start(self._h, _p(y), _p(lam), last))

    def refresh_z(self) -> None:
        _raise(self._L.cqp_refresh_z(self._h))

    def update_vectors(self, g, c, d) -> None:
        g = _vec(g, self.n, "update_vectors")
        c = _vec(c, self.m, "update_vectors")
        d = _vec(d, self.m, "update_vectors")
        _raise(self._L.cqp_update_vectors(self._h, _p(g), _p(c), _p(d)))

    def _result(self, cap: int):
        # result buffers are cached per capacity (the MPC step path calls this at kHz rates); only
        # the most recent few capacities are kept
        cache = self.__dict__.setdefault("_res_cache", {})
        if cap not in cache:
            while len(cache) >= 4:
                cache.pop(next(iter(cache)))
            y, z, lam = np.empty(self.n), np.empty(self.m), np.empty(self.m)
            trace = (CqpRhoSwitch * cap)()
            hist = (CqpResidualSample * cap)()
            res = CqpResult(_p(y), _p(z), _p(lam), trace, cap, 0, hist, cap, 0, INVALID, 0, 0.0, 0.0,
                            0.0, 0.0)
            cache[cap] = (res, (y, z, lam, trace, hist))
        return cache[cap]

    @staticmethod
    def _report(res: CqpResult, bufs) -> SolveReport:
        y, z, lam, trace, hist = bufs
        y, z, lam = y.copy(), z.copy(), lam.copy()
        nt = min(res.rho_trace_len, res.rho_trace_cap)
        nh = min(res.history_len, res.history_cap)
        sol = Solution(y, z, lam, res.status, res.iterations, res.r_prim, res.r_dual,
                       [(trace[i].iteration, trace[i].grid_index) for i in range(nt)])
        return SolveReport(sol, res.wall_ms,
                           [(hist[i].iteration, hist[i].r_prim, hist[i].r_dual, hist[i].grid_index)
                            for i in range(nh)], res.kernel_us)

    def solve(self) -> SolveReport:
        s = self.settings
        res, bufs = self._result(s.max_iters // s.check_interval + 2)
        _raise(self._L.cqp_solve(self._h, C.byref(res)))
        return self._report(res, bufs)

    def fixed_iters(self, k: int) -> SolveReport:
        if k < 1:
            raise ValueError("fixed_iters: k must be >= 1")
        res, bufs = self._result(k // self.settings.check_interval + 2)
        _raise(self._L.cqp_fixed_iters(self._h, int(k), C.byref(res)))
        return self._report(res, bufs)

    def mpc_step(self, g, c, d, k: int) -> SolveReport:
        """update_vectors + refresh_z + fixed_iters(k) as one upload + one launch
        (the per-step protocol of bench.cpp:157-167)."""
        if k < 1:
            raise ValueError("mpc_step: k must be >= 1")
        g = _vec(g, self.n, "mpc_step")
        c = _vec(c, self.m, "mpc_step")
        d = _vec(d, self.m, "mpc_step")
        res, bufs = self._result(k // self.settings.check_interval + 2)
        _raise(self._L.cqp_mpc_step(self._h, _p(g), _p(c), _p(d), int(k), C.byref(res)))
        return self._report(res, bufs)

    def set_mpc_template(self, tmpl, limits) -> None:
        """Hand the condensed-MPC template (mpc.hpp CondensedTemplate: offset_g, offset_c, c_base,
        d_base, K) and the control limits to the device, so that `mpc_step_x0` can instantiate the
        step QP (mpc.cpp:260-270) and extract the control (bench.cpp:169-175) there."""
        f = lambda a: np.asfortranarray(np.asarray(a, dtype=np.float64))  # noqa: E731
        og, oc, K = f(tmpl.offset_g), f(tmpl.offset_c), f(tmpl.K)
        nx, nu = og.shape[1], K.shape[0]
        if og.shape != (self.n, nx) or oc.shape != (self.m, nx) or K.shape != (nu, nx):
            raise ValueError("set_mpc_template: dimension mismatch")
        cb, db = _vec(tmpl.c_base, self.m, "set_mpc_template"), _vec(tmpl.d_base, self.m, "set_mpc_template")
        ulo, uhi = _vec(limits.u_lo, nu, "set_mpc_template"), _vec(limits.u_hi, nu, "set_mpc_template")
        _raise(self._L.cqp_mpc_set_template(self._h, nx, nu, _p(og), _p(oc), _p(cb), _p(db), _p(K), _p(ulo), _p(uhi)))
        self._mpc_nx, self._mpc_nu = nx, nu

    def mpc_step_x0(self, x0, k: int):
        """(u0, report) of one control step from the measured state x0; everything between the
        upload of x0 and the download of u0 runs on the device."""
        if k < 1:
            raise ValueError("mpc_step_x0: k must be >= 1")
        x0 = _vec(x0, getattr(self, "_mpc_nx", -1), "mpc_step_x0")
        u0 = np.empty(self._mpc_nu)
        res, bufs = self._result(k // self.settings.check_interval + 2)
        _raise(self._L.cqp_mpc_step_x0(self._h, _p(x0), int(k), _p(u0), C.byref(res)))
        return u0, self._report(res, bufs)

    def mpc_server_start(self, k: int, idle_timeout_ms: float = 100.0) -> None:
        """Keep the solve kernel resident and serve `mpc_step_x0(x0, k)` from a host-mapped mailbox
        (no CUDA call per control step; same results bit for bit).  Any other method of this Solver
        retires the resident kernel first; it also leaves by itself after `idle_timeout_ms` without
        a request and is restarted by the next step."""
        if k < 1:
            raise ValueError("mpc_server_start: k must be >= 1")
        _raise(self._L.cqp_mpc_server_start(self._h, int(k), float(idle_timeout_ms)))

    def mpc_server_stop(self) -> None:
        _raise(self._L.cqp_mpc_server_stop(self._h))

    def mpc_server_last_timing(self) -> Tuple[float, float]:
        """(wall_us inside the C ABI call, device-side step duration in us) of the last served step."""
        w, d = C.c_double(), C.c_double()
        _raise(self._L.cqp_mpc_server_last_timing(self._h, C.byref(w), C.byref(d)))
        return w.value, d.value

    def mpc_step_x0_fast(self, x0: np.ndarray, k: int, u0: np.ndarray) -> None:
        """`mpc_step_x0` without the report and without allocations (x0, u0: contiguous float64
        arrays the caller keeps): what a control loop calls at kHz rates."""
        _raise(self._L.cqp_mpc_step_x0(self._h, _p(x0), int(k), _p(u0), None))

    # ---- accessors, solver.hpp:123-127 ----
    @property
    def state(self) -> np.ndarray:
        v = np.empty(self.n + 2 * self.m)
        _raise(self._L.cqp_get_state(self._h, _p(v), None))
        return v

    @property
    def layer_index(self) -> int:
        idx = C.c_int()
        _raise(self._L.cqp_get_state(self._h, None, C.byref(idx)))
        return idx.value

    def layer(self, k: int) -> dict:
        """cache().layers[k]: W, D, GD, b (for the current g), rho_vec."""
        n, m = self.n, self.m
        dim = n + 2 * m
        W = np.empty((dim, dim), order="F"); D = np.empty((n, n), order="F")
        GD = np.empty((m, n), order="F"); b = np.empty(dim); rho = np.empty(m)
        _raise(self._L.cqp_get_layer(self._h, k, _p(W), _p(D), _p(GD), _p(b), _p(rho)))
        return {"W": W, "D": D, "GD": GD, "b": b, "rho_vec": rho}

    def scaling(self) -> dict:
        """cache().scaling, grid and clamp bounds."""
        n, m = self.n, self.m
        E, F, grid = np.empty(n), np.empty(m), np.empty(self.L)
        lo, hi = np.empty(n + 2 * m), np.empty(n + 2 * m)
        cs, idx = C.c_double(), C.c_int()
        _raise(self._L.cqp_get_scaling(self._h, _p(E), _p(F), C.byref(cs), _p(grid), C.byref(idx),
                                       _p(lo), _p(hi)))
        return {"E": E, "F": F, "cost_scale": cs.value, "grid": grid, "initial_index": idx.value,
                "c_tilde": lo, "d_tilde": hi}

    def launch_info(self) -> dict:
        a, b, c, d = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _raise(self._L.cqp_launch_info(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        wb, st = C.c_double(), C.c_int()
        _raise(self._L.cqp_layer_traffic(self._h, C.byref(wb), C.byref(st)))
        return {"ctas": a.value, "rows_per_cta": b.value, "tier": c.value, "smem_bytes": d.value,
                "w_bytes_per_iteration": wb.value, "structured": st.value}


class BatchSolver:
    """Many QPs sharing (H, G) -- MPC instances that differ in x0, i.e. in (g, c, d) -- solved
    together from a cold start: column j of the result equals what `Solver.solve()` returns
    after `update_vectors(g[:, j], c[:, j], d[:, j]); cold_start()` (solver.cpp:158-166)."""

    def __init__(self, solver: Solver, capacity: int):
        import weakref
        self._L = solver._L
        self._solver = solver          # keeps the shared ladder alive
        self._b = C.c_void_p()
        self.capacity = int(capacity)
        if not solver._h:
            raise ValueError("BatchSolver: the Solver has been closed")
        _raise(self._L.cqp_batch_create(C.byref(self._b), solver._h, self.capacity))
        solver.__dict__.setdefault("_dependents", []).append(weakref.ref(self))
        self.n, self.m = solver.n, solver.m
        self._rec_cap = solver.settings.max_iters // solver.settings.check_interval + 2
        self._pinned = []     # page-locked output buffers, allocated once
        self._out = None
        self._last_B = 0

    def _pinned_array(self, shape, dtype, order="C"):
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        ptr = C.c_void_p()
        _raise(self._L.cqp_pinned_alloc(C.byref(ptr), max(nbytes, 1)))
        self._pinned.append(ptr)
        buf = (C.c_char * max(nbytes, 1)).from_address(ptr.value)
        return np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape, order=order)

    def close(self) -> None:
        b, self._b = getattr(self, "_b", None), C.c_void_p()
        if b:
            self._L.cqp_batch_destroy(b)
        self._out = None
        for ptr in getattr(self, "_pinned", []):
            self._L.cqp_pinned_free(ptr)
        self._pinned = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve(self, g_cols, c_cols, d_cols, zero_copy: bool = False) -> dict:
        """Solves the B columns.  The result arrays are COPIES by default.  With `zero_copy=True`
        they are views of this object's page-locked result buffers: valid only until the next
        `solve()` (which overwrites them) or `close()` (which frees them) -- the caller must not
        touch them afterwards."""
        if not self._b:
            raise ValueError("BatchSolver: closed (or its Solver was closed)")
        g = np.asfortranarray(np.asarray(g_cols, dtype=np.float64))
        c = np.asfortranarray(np.asarray(c_cols, dtype=np.float64))
        d = np.asfortranarray(np.asarray(d_cols, dtype=np.float64))
        if g.ndim != 2 or g.shape[0] != self.n or c.shape != (self.m, g.shape[1]) or d.shape != c.shape:
            raise ValueError("batch solve: dimension mismatch")
        B = g.shape[1]
        if B > self.capacity:
            raise MemoryError("batch solve: B exceeds the batch capacity")
        if self._out is None:
            # page-locked result buffers for `capacity` columns, reused by every solve: the arrays
            # returned below are views that the NEXT solve overwrites (copy them to keep them)
            cap = self.capacity
            self._out = (self._pinned_array((self.n, cap), np.float64, "F"), self._pinned_array((self.m, cap), np.float64, "F"),
                         self._pinned_array((self.m, cap), np.float64, "F"), self._pinned_array((cap,), np.int32),
                         self._pinned_array((cap,), np.int32), self._pinned_array((cap,), np.int32),
                         self._pinned_array((cap,), np.int32), self._pinned_array((cap,), np.float64),
                         self._pinned_array((cap,), np.float64))
        y, z, lam, status, iters, final, nsw, rp, rd = (a[..., :B] for a in self._out)
        self._last_B = B
        ms = C.c_double()
        ip = lambda a: a.ctypes.data_as(_lib.c_int_p)  # noqa: E731
        _raise(self._L.cqp_batch_solve(self._b, B, _p(g), _p(c), _p(d), _p(y), _p(z), _p(lam),
                                       ip(status), ip(iters), ip(final), _p(rp), _p(rd), ip(nsw),
                                       C.byref(ms)))
        comp, tot, launches = C.c_double(), C.c_double(), C.c_longlong()
        self._L.cqp_batch_last_timing(self._b, C.byref(comp), C.byref(tot), C.byref(launches))
        gms, gfl, rounds = C.c_double(), C.c_double(), C.c_int()
        self._L.cqp_batch_last_profile(self._b, C.byref(gms), C.byref(gfl), C.byref(rounds))
        ract = np.zeros(max(rounds.value, 1), dtype=np.int32); rms = np.zeros(max(rounds.value, 1))
        self._L.cqp_batch_round_profile(self._b, rounds.value, ip(ract), _p(rms))
        if not zero_copy:
            y, z, lam, status, iters, final, nsw, rp, rd = (
                np.array(a, copy=True, order="F" if a.ndim == 2 else "C") for a in (y, z, lam, status, iters, final, nsw, rp, rd))
        return {"round_active": ract, "round_ms": rms,
                "y": y, "z": z, "lam": lam, "status": status, "iterations": iters,
                "final_index": final, "n_switches": nsw, "r_prim": rp, "r_dual": rd,
                "device_ms": ms.value, "compute_ms": comp.value, "launches": launches.value,
                "gemm_ms": gms.value, "gemm_flops": gfl.value, "rounds": rounds.value}

    def solve_into(self, B: int, g_ptr: int, c_ptr: int, d_ptr: int, y_ptr: int, z_ptr: int, lam_ptr: int,
                   status_ptr: int, iterations_ptr: int, final_index_ptr: int, r_prim_ptr: int,
                   r_dual_ptr: int, n_switches_ptr: int) -> dict:
        """cqp_batch_solve on raw addresses (host or device memory of this GPU; 0 = not wanted for
        an output): the caller owns every buffer.  Used by the multi-GPU gather
        (sharding.solve_sharded_device), which hands device buffers straight to NCCL."""
        if not self._b:
            raise ValueError("BatchSolver: closed (or its Solver was closed)")
        if not 1 <= B <= self.capacity:
            raise MemoryError("batch solve: B exceeds the batch capacity")
        dp = lambda a: C.cast(C.c_void_p(a or None), c_double_p)          # noqa: E731
        ip = lambda a: C.cast(C.c_void_p(a or None), _lib.c_int_p)        # noqa: E731
        ms = C.c_double()
        _raise(self._L.cqp_batch_solve(self._b, B, dp(g_ptr), dp(c_ptr), dp(d_ptr), dp(y_ptr), dp(z_ptr),
                                       dp(lam_ptr), ip(status_ptr), ip(iterations_ptr), ip(final_index_ptr),
                                       dp(r_prim_ptr), dp(r_dual_ptr), ip(n_switches_ptr), C.byref(ms)))
        self._last_B = B
        comp, tot, launches = C.c_double(), C.c_double(), C.c_longlong()
        self._L.cqp_batch_last_timing(self._b, C.byref(comp), C.byref(tot), C.byref(launches))
        gms, gfl, rounds = C.c_double(), C.c_double(), C.c_int()
        self._L.cqp_batch_last_profile(self._b, C.byref(gms), C.byref(gfl), C.byref(rounds))
        return {"device_ms": ms.value, "compute_ms": comp.value, "launches": launches.value,
                "gemm_ms": gms.value, "gemm_flops": gfl.value, "rounds": rounds.value}

    def traces(self) -> List[List[Tuple[int, int]]]:
        """Per-column `Solution.rho_trace` of the last solve (problem.hpp:57-70): a list of
        (iteration, grid_index) per column, entry 0 = (0, start index)."""
        B, cap = self._last_B, self._rec_cap
        rec = (CqpRhoSwitch * (B * cap))()
        ln = np.zeros(B, dtype=np.int32)
        _raise(self._L.cqp_batch_get_traces(self._b, B, cap, rec, ln.ctypes.data_as(_lib.c_int_p)))
        flat = np.frombuffer(rec, dtype=np.int32).reshape(B, cap, 2)
        return [[(int(a), int(b)) for a, b in flat[j, :min(int(ln[j]), cap)]] for j in range(B)]

    def histories(self) -> List[List[Tuple[int, float, float, int]]]:
        """Per-column `SolveReport.residual_history` of the last solve (solver.hpp:56-67):
        (iteration, r_prim, r_dual, grid_index before the check's switch) per convergence check."""
        B, cap = self._last_B, self._rec_cap
        rec = (CqpResidualSample * (B * cap))()
        ln = np.zeros(B, dtype=np.int32)
        _raise(self._L.cqp_batch_get_history(self._b, B, cap, rec, ln.ctypes.data_as(_lib.c_int_p)))
        dt = np.dtype([("iteration", np.int32), ("pad0", np.int32), ("r_prim", np.float64),
                       ("r_dual", np.float64), ("grid_index", np.int32), ("pad1", np.int32)])
        flat = np.frombuffer(rec, dtype=dt).reshape(B, cap)
        return [[(int(r["iteration"]), float(r["r_prim"]), float(r["r_dual"]), int(r["grid_index"]))
                 for r in flat[j, :min(int(ln[j]), cap)]] for j in range(B)]
