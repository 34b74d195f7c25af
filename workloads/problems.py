"""Synthetic problem generators for the BASELINE.json workloads (host side, offline, numpy).

Mirrors the reference's benchmark generators and sampling rules
(/root/reference/proj/src/bench.cpp):

  gen_random_dense_qp        bench.cpp:89-118
  gen_random_linear_system   bench.cpp:120-137   (nx = 3 nu there; nx is a parameter here because
                                                  BASELINE.json's configs use nx = 2 nu)
  x0 start scale             bench.cpp:205-221   (3x LQR push of the control limits)
  x0 stream seed             bench.cpp:35        (seed ^ 0x9e3779b97f4a7c15)
  MPC suite weights/limits   bench.cpp:264-275   (Q = I, R = I, Q_N = P, |u| <= 1)

Both the GPU path and the CPU oracle are fed the arrays produced here, byte for byte.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from paper_2311_18056_b200.problem_io import DenseQP  # noqa: F401  (re-exported: problems.DenseQP)

from . import mpc
from .rng import Rng

X0_STREAM = 0x9E3779B97F4A7C15


def gen_random_dense_qp(n: int, seed: int) -> DenseQP:
    """bench.cpp:89-118: H = M'M + 0.1 I, floor(n/4) equality + floor(n/4) inequality rows."""
    if n < 4:
        raise ValueError("gen_random_dense_qp: n must be >= 4")
    rng = Rng(seed)
    M = rng.normal_matrix(n, n)
    H = M.T @ M + 0.1 * np.eye(n)
    H = 0.5 * (H + H.T)
    g = rng.normal_vector(n)
    n_side = n // 4
    m = 2 * n_side
    y0 = rng.normal_vector(n)
    G = rng.normal_matrix(m, n)
    gy0 = G @ y0
    c = np.empty(m)
    d = np.empty(m)
    c[:n_side] = gy0[:n_side]
    d[:n_side] = gy0[:n_side]
    for i in range(n_side, m):
        slack = abs(rng.normal()) + 0.1
        c[i] = gy0[i] - slack
        d[i] = gy0[i] + slack
    return DenseQP(np.asfortranarray(H), g, np.asfortranarray(G), c, d)


def gen_random_linear_system(nu: int, seed: int, unstable: bool,
                             nx: Optional[int] = None) -> mpc.LinearSystem:
    """bench.cpp:120-137 (nx defaults to the reference's 3 nu)."""
    if nu < 1:
        raise ValueError("gen_random_linear_system: nu must be >= 1")
    nx = 3 * nu if nx is None else nx
    rng = Rng(seed)
    for _ in range(10):
        A = rng.normal_matrix(nx, nx)
        B = rng.normal_matrix(nx, nu)
        target = rng.uniform(1.05, 1.3) if unstable else rng.uniform(0.8, 0.95)
        radius = mpc.spectral_radius(A)
        if radius <= 0.0:
            continue
        A = A * (target / radius)
        sys = mpc.LinearSystem(np.asfortranarray(A), np.asfortranarray(B))
        if mpc.controllability_rank(sys) == nx:
            return sys
    raise RuntimeError("gen_random_linear_system: controllability check failed after resampling")


@dataclass
class MpcWorkload:
    """One condensed-MPC family: shared (H, G), per-instance (g, c, d) via instantiate(x0)."""
    sys: mpc.LinearSystem
    tmpl: mpc.CondensedTemplate
    limits: mpc.BoxLimits
    seed: int
    name: str

    @property
    def n(self) -> int:
        return self.tmpl.Hbar.shape[0]

    @property
    def m(self) -> int:
        return self.tmpl.Gbar.shape[0]

    def base_problem(self) -> DenseQP:
        """The QP the Solver is constructed on: instantiate(tmpl, 0) (bench.cpp:275)."""
        return self.problem_at(np.zeros(self.sys.nx))

    def problem_at(self, x0: np.ndarray) -> DenseQP:
        H, g, G, c, d = mpc.instantiate(self.tmpl, x0)
        return DenseQP(H, g, G, c, d)

    def x0_direction(self, seed: Optional[int] = None) -> np.ndarray:
        """bench.cpp:208-211: normal direction from the x0 stream, infinity-normalised."""
        s = self.seed if seed is None else seed
        d = Rng((s ^ X0_STREAM) & 0xFFFFFFFFFFFFFFFF).normal_vector(self.sys.nx)
        nrm = float(np.abs(d).max())
        return d / nrm if nrm > 0 else d

    def push_scale(self, direction: np.ndarray) -> float:
        """bench.cpp:213-221: scale at which the LQR control exceeds the limits 3x."""
        limit_mag = 0.0
        for v in list(self.limits.u_hi) + list(self.limits.u_lo):
            if np.isfinite(v):
                limit_mag = max(limit_mag, abs(float(v)))
        if limit_mag == 0.0:
            return 1.0
        push = float(np.abs(self.tmpl.K @ direction).max())
        return 3.0 * limit_mag / push if push > 0 else 1.0

    def x0(self, hardness: float = 1.0, seed: Optional[int] = None) -> np.ndarray:
        d = self.x0_direction(seed)
        return hardness * self.push_scale(d) * d


def make_mpc_workload(nu: int, nx: int, horizon: int, seed: int, unstable: bool = False,
                      limits: Optional[mpc.BoxLimits] = None, name: str = "") -> MpcWorkload:
    """bench.cpp:259-275 recipe: Q = I, R = I, Q_N = DARE P, |u| <= 1, LQR-preconditioned."""
    sys = gen_random_linear_system(nu, seed, unstable, nx=nx)
    P, K = mpc.lqr_gain(sys, np.eye(nx), np.eye(nu))
    weights = mpc.MpcWeights(np.eye(nx), np.eye(nu), P, horizon)
    lim = limits if limits is not None else mpc.BoxLimits.symmetric_control(nu, 1.0)
    tmpl = mpc.build_condensed_mpc(sys, weights, lim, K)
    return MpcWorkload(sys, tmpl, lim, seed, name or f"mpc_nu{nu}_nx{nx}_N{horizon}")


# ---- the BASELINE.json configs ----------------------------------------

def config1(seed: int = 0, unstable: bool = False) -> MpcWorkload:
    """configs[0]: nx=20, nu=10, N=10, control limits."""
    return make_mpc_workload(10, 20, 10, seed, unstable, name="random_mpc_nu10")


def config2(nu: int, seed: int = 0, unstable: bool = False) -> MpcWorkload:
    """configs[1]: sweep nu=10..50, nx=2 nu, N=10."""
    return make_mpc_workload(nu, 2 * nu, 10, seed, unstable, name=f"random_mpc_nu{nu}")


def config3_atlas(horizon: int = 30, seed: int = 0) -> MpcWorkload:
    """configs[2]: Atlas-sized synthetic linearisation: 58 states, 29 controls,
    open-loop unstable; horizon 0.3/0.4/0.5 s at dt = 0.01 s -> N = 30/40/50."""
    return make_mpc_workload(29, 58, horizon, seed, unstable=True, name=f"atlas_sized_N{horizon}")


def config4_quadruped(horizon: int = 30, seed: int = 0) -> MpcWorkload:
    """configs[3]: quadruped + arm sized: 52 states, 20+12 inputs, 52 constraint rows per step
    (PAPER.md:828): 32 control rows + the first 20 state rows, long horizon."""
    nx, nu = 52, 32
    lim = mpc.BoxLimits(np.full(nu, -1.0), np.full(nu, 1.0), np.full(nx, -50.0),
                        np.full(nx, 50.0), x_rows=list(range(20)))
    return make_mpc_workload(nu, nx, horizon, seed, unstable=False, limits=lim,
                             name=f"quadruped_sized_N{horizon}")


def batch_instances(wl: MpcWorkload, count: int, first: int = 0, lo: float = 0.3,
                    hi: float = 10.0):
    """configs[4]: `count` instances of one family; instance j has x0_j = s_j * push * dir_j with
    dir_j from Rng(1000 + j) and s_j log-uniform in [lo, hi].
    Returns column-major (n x count) g and (m x count) c, d, plus the x0 matrix (nx x count)."""
    n, m, nx = wl.n, wl.m, wl.sys.nx
    X0 = np.empty((nx, count), order="F")
    for j in range(count):
        rng = Rng(1000 + first + j)
        d = rng.normal_vector(nx)
        d = d / float(np.abs(d).max())
        s = float(np.exp(np.log(lo) + (np.log(hi) - np.log(lo)) * rng.uniform()))
        X0[:, j] = s * wl.push_scale(d) * d
    g = np.asfortranarray(wl.tmpl.offset_g @ X0)
    shift = wl.tmpl.offset_c @ X0
    c = np.asfortranarray(wl.tmpl.c_base[:, None] - shift)
    d_ = np.asfortranarray(wl.tmpl.d_base[:, None] - shift)
    assert g.shape == (n, count) and c.shape == (m, count)
    return g, c, d_, X0
