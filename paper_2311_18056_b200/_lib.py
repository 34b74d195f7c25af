"""Loader of the C-ABI library libcqp_b200.so (include/cqp_b200.h).

There is no CPU fallback: if the library is missing, or no CUDA device is present when a
solver is constructed, the call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
# CQP_B200_LIB: load another build of the same library (tools/: instrumented -DCQP_TRACE builds)
LIB_PATH = os.environ.get("CQP_B200_LIB") or os.path.join(_HERE, "libcqp_b200.so")

c_double_p = C.POINTER(C.c_double)
c_int_p = C.POINTER(C.c_int)


class CqpSettings(C.Structure):
    """cqp_settings (SolverSettings + Equilibration, solver.hpp:43-53)."""
    _fields_ = [
        ("eps_prim", C.c_double), ("eps_dual", C.c_double),
        ("check_interval", C.c_int), ("max_iters", C.c_int),
        ("sigma", C.c_double), ("grid_points", C.c_int),
        ("rho_switch_threshold", C.c_double), ("adaptive_rho", C.c_int),
        ("eq_enabled", C.c_int), ("eq_max_passes", C.c_int), ("eq_tol", C.c_double),
    ]


class CqpRhoSwitch(C.Structure):
    _fields_ = [("iteration", C.c_int), ("grid_index", C.c_int)]


class CqpResidualSample(C.Structure):
    _fields_ = [("iteration", C.c_int), ("r_prim", C.c_double), ("r_dual", C.c_double),
                ("grid_index", C.c_int)]


class CqpResult(C.Structure):
    _fields_ = [
        ("y", c_double_p), ("z", c_double_p), ("lam", c_double_p),
        ("rho_trace", C.POINTER(CqpRhoSwitch)), ("rho_trace_cap", C.c_int), ("rho_trace_len", C.c_int),
        ("history", C.POINTER(CqpResidualSample)), ("history_cap", C.c_int), ("history_len", C.c_int),
        ("status", C.c_int), ("iterations", C.c_int),
        ("r_prim", C.c_double), ("r_dual", C.c_double),
        ("wall_ms", C.c_double), ("kernel_us", C.c_double),
    ]


# Every symbol include/cqp_b200.h declares (tests/test_cabi_symbols.py checks the list against
# the header and the built library).
EXPORTS = [
    "cqp_default_settings", "cqp_last_error", "cqp_device_count", "cqp_create",
    "cqp_create_from_layers", "cqp_destroy", "cqp_update_vectors", "cqp_cold_start",
    "cqp_warm_start", "cqp_refresh_z", "cqp_solve", "cqp_fixed_iters", "cqp_mpc_step",
    "cqp_mpc_set_template", "cqp_mpc_step_x0", "cqp_mpc_server_start", "cqp_mpc_server_stop", "cqp_mpc_server_last_timing",
    "cqp_get_state", "cqp_set_state", "cqp_get_layer", "cqp_get_scaling", "cqp_dims", "cqp_debug_words",
    "cqp_launch_info", "cqp_layer_traffic", "cqp_measure_read_bandwidth", "cqp_pinned_alloc", "cqp_pinned_free",
    "cqp_batch_create", "cqp_batch_destroy", "cqp_batch_solve", "cqp_batch_last_timing", "cqp_batch_last_profile", "cqp_batch_round_profile",
    "cqp_batch_get_traces", "cqp_batch_get_history",
]

_lib = None


def build(force: bool = False) -> str:
    """Compile csrc/*.cu into libcqp_b200.so with nvcc for sm_100a (csrc/Makefile)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.check_call(["make", "-C", os.path.join(_HERE, "csrc"), "-j8", "-s"]
                              + (["-B"] if force else []))
    return LIB_PATH


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback for the solve path)")
    L = C.CDLL(LIB_PATH)
    L.cqp_last_error.restype = C.c_char_p
    L.cqp_default_settings.argtypes = [C.POINTER(CqpSettings)]
    L.cqp_create.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int] + [c_double_p] * 5 + [
        C.POINTER(CqpSettings), C.c_int]
    L.cqp_create_from_layers.argtypes = [
        C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int,
        C.POINTER(c_double_p), C.POINTER(c_double_p), C.POINTER(c_double_p),
        c_double_p, C.c_int] + [c_double_p] * 8 + [C.c_double, C.POINTER(CqpSettings), C.c_int]
    L.cqp_destroy.argtypes = [C.c_void_p]
    L.cqp_destroy.restype = None
    L.cqp_update_vectors.argtypes = [C.c_void_p] + [c_double_p] * 3
    L.cqp_cold_start.argtypes = [C.c_void_p]
    L.cqp_warm_start.argtypes = [C.c_void_p, c_double_p, c_double_p, C.c_int]
    L.cqp_refresh_z.argtypes = [C.c_void_p]
    L.cqp_solve.argtypes = [C.c_void_p, C.POINTER(CqpResult)]
    L.cqp_fixed_iters.argtypes = [C.c_void_p, C.c_int, C.POINTER(CqpResult)]
    L.cqp_mpc_step.argtypes = [C.c_void_p] + [c_double_p] * 3 + [C.c_int, C.POINTER(CqpResult)]
    L.cqp_mpc_set_template.argtypes = [C.c_void_p, C.c_int, C.c_int] + [c_double_p] * 7
    L.cqp_mpc_step_x0.argtypes = [C.c_void_p, c_double_p, C.c_int, c_double_p, C.POINTER(CqpResult)]
    L.cqp_mpc_server_start.argtypes = [C.c_void_p, C.c_int, C.c_double]
    L.cqp_mpc_server_stop.argtypes = [C.c_void_p]
    L.cqp_mpc_server_last_timing.argtypes = [C.c_void_p, c_double_p, c_double_p]
    L.cqp_get_state.argtypes = [C.c_void_p, c_double_p, c_int_p]
    L.cqp_set_state.argtypes = [C.c_void_p, c_double_p, C.c_int]
    L.cqp_get_layer.argtypes = [C.c_void_p, C.c_int] + [c_double_p] * 5
    L.cqp_get_scaling.argtypes = [C.c_void_p, c_double_p, c_double_p, c_double_p, c_double_p,
                                  c_int_p, c_double_p, c_double_p]
    L.cqp_dims.argtypes = [C.c_void_p, c_int_p, c_int_p, c_int_p]
    L.cqp_debug_words.argtypes = [C.c_void_p, c_int_p]
    L.cqp_launch_info.argtypes = [C.c_void_p, c_int_p, c_int_p, c_int_p, c_int_p]
    L.cqp_layer_traffic.argtypes = [C.c_void_p, c_double_p, c_int_p]
    L.cqp_measure_read_bandwidth.argtypes = [C.c_int, C.c_ulonglong, C.c_int, c_double_p]
    L.cqp_pinned_alloc.argtypes = [C.POINTER(C.c_void_p), C.c_ulonglong]
    L.cqp_pinned_free.argtypes = [C.c_void_p]
    L.cqp_pinned_free.restype = None
    L.cqp_batch_create.argtypes = [C.POINTER(C.c_void_p), C.c_void_p, C.c_int]
    L.cqp_batch_destroy.argtypes = [C.c_void_p]
    L.cqp_batch_destroy.restype = None
    L.cqp_batch_solve.argtypes = [C.c_void_p, C.c_int] + [c_double_p] * 6 + [
        c_int_p, c_int_p, c_int_p, c_double_p, c_double_p, c_int_p, c_double_p]
    L.cqp_batch_last_timing.argtypes = [C.c_void_p, c_double_p, c_double_p, C.POINTER(C.c_longlong)]
    L.cqp_batch_last_profile.argtypes = [C.c_void_p, c_double_p, c_double_p, c_int_p]
    L.cqp_batch_round_profile.argtypes = [C.c_void_p, C.c_int, c_int_p, c_double_p]
    L.cqp_batch_get_traces.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(CqpRhoSwitch), c_int_p]
    L.cqp_batch_get_history.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(CqpResidualSample), c_int_p]
    _lib = L
    return L


def last_error() -> str:
    return load().cqp_last_error().decode("utf-8", "replace")
