"""Host-side (offline) MPC front end: LQR-preconditioned condensed MPC templates.

Mirrors the subset of the reference's `clampqp::mpc` that produces the QPs the solve path
consumes (/root/reference/proj/include/clampqp/mpc.hpp, src/mpc.cpp):

  lqr_gain             mpc.cpp:192-216   fixed-point Riccati iteration
  build_limit_rows     mpc.cpp:65-89     control (and optional state) selector rows
  build_cost_hessian   mpc.cpp:91-101
  build_sm             mpc.cpp:105-134   S, M of the substitution u_k = -K x_k + du_k
  build_condensed_mpc  mpc.cpp:227-258
  instantiate          mpc.cpp:260-270   g = offset_g x0, bounds shifted by offset_c x0

This is input production (numpy, offline), not the solve loop.  The per-step `instantiate`
also exists as a device kernel (csrc/cqp_single.cu, cqp_mpc_step) -- SURVEY.md section 8(f) rank 1.

One extension over the reference: `BoxLimits.x_rows` selects a subset of state rows, which the
reference's all-or-nothing state limits (mpc.cpp:70) cannot express; it is needed to build the
"52 constraint rows per step" quadruped-sized workload.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np


@dataclass
class LinearSystem:
    """x+ = A x + B u  (mpc.hpp:25-32)."""
    A: np.ndarray
    B: np.ndarray

    @property
    def nx(self) -> int:
        return self.A.shape[0]

    @property
    def nu(self) -> int:
        return self.B.shape[1]


@dataclass
class MpcWeights:
    """mpc.hpp:37-42."""
    Q: np.ndarray
    R: np.ndarray
    Q_N: np.ndarray
    horizon: int = 1


@dataclass
class BoxLimits:
    """mpc.hpp:44-54 (+ optional x_rows subset, see module docstring)."""
    u_lo: np.ndarray
    u_hi: np.ndarray
    x_lo: Optional[np.ndarray] = None
    x_hi: Optional[np.ndarray] = None
    x_rows: Optional[Sequence[int]] = None

    @staticmethod
    def symmetric_control(nu: int, magnitude: float) -> "BoxLimits":
        return BoxLimits(np.full(nu, -magnitude), np.full(nu, magnitude))


@dataclass
class CondensedTemplate:
    """mpc.hpp:73-87."""
    K: np.ndarray
    Abar: np.ndarray
    S: np.ndarray
    M: np.ndarray
    Hbar: np.ndarray
    Gbar: np.ndarray
    offset_g: np.ndarray
    offset_c: np.ndarray
    c_base: np.ndarray
    d_base: np.ndarray
    nx: int
    nu: int
    horizon: int


def spectral_radius(a: np.ndarray) -> float:
    """types.hpp:41-47 (Eigen::EigenSolver there, LAPACK dgeev here)."""
    if a.shape[0] == 0:
        return 0.0
    return float(np.abs(np.linalg.eigvals(a)).max())


def controllability_rank(sys: LinearSystem) -> int:
    """mpc.cpp:144-154 (ColPivHouseholderQR rank there, SVD rank here)."""
    nx, nu = sys.nx, sys.nu
    ctrb = np.empty((nx, nx * nu))
    block = sys.B.copy()
    for j in range(nx):
        ctrb[:, j * nu:(j + 1) * nu] = block
        block = sys.A @ block
    return int(np.linalg.matrix_rank(ctrb))


def lqr_gain(sys: LinearSystem, Q: np.ndarray, R: np.ndarray, tol: float = 1e-10,
             max_iters: int = 10000):
    """mpc.cpp:192-216 -> (P, K). Raises RuntimeError when the iteration does not converge."""
    A, B = sys.A, sys.B
    At, Bt = A.T, B.T
    P = Q.copy()
    defect = np.inf
    for _ in range(max_iters):
        BtPA = Bt @ P @ A
        gain_term = np.linalg.solve(R + Bt @ P @ B, BtPA)
        P_next = Q + At @ P @ A - BtPA.T @ gain_term
        P_next = 0.5 * (P_next + P_next.T)
        defect = float(np.abs(P_next - P).max())
        P = P_next
        if defect <= tol:
            break
    if defect > tol:
        raise RuntimeError("lqr_gain: Riccati iteration did not converge")
    K = np.linalg.solve(R + Bt @ P @ B, Bt @ P @ A)
    return P, K


def _u_offset(k: int, nx: int, nu: int) -> int:
    return k * (nx + nu)


def _x_offset(k: int, nx: int, nu: int) -> int:
    return k * (nx + nu) + nu


def build_limit_rows(sys: LinearSystem, lim: BoxLimits, N: int):
    """mpc.cpp:65-89 -> (G, c, d) over the direct layout y = [u0; x1; u1; ...; xN]."""
    nx, nu = sys.nx, sys.nu
    n = N * (nx + nu)
    m_u = N * nu
    rows = list(range(nx)) if lim.x_rows is None else list(lim.x_rows)
    per_x = len(rows) if lim.x_lo is not None else 0
    m_x = N * per_x
    G = np.zeros((m_u + m_x, n))
    c = np.empty(m_u + m_x)
    d = np.empty(m_u + m_x)
    for k in range(N):
        uo = _u_offset(k, nx, nu)
        G[k * nu:(k + 1) * nu, uo:uo + nu] = np.eye(nu)
        c[k * nu:(k + 1) * nu] = lim.u_lo
        d[k * nu:(k + 1) * nu] = lim.u_hi
    if lim.x_lo is not None:
        x_lo = np.asarray(lim.x_lo, dtype=np.float64)
        x_hi = np.asarray(lim.x_hi, dtype=np.float64)
        for k in range(N):
            xo = _x_offset(k, nx, nu)
            for r, xi in enumerate(rows):
                G[m_u + k * per_x + r, xo + xi] = 1.0
                c[m_u + k * per_x + r] = x_lo[xi]
                d[m_u + k * per_x + r] = x_hi[xi]
    return G, c, d


def build_cost_hessian(w: MpcWeights, nx: int, nu: int) -> np.ndarray:
    """mpc.cpp:91-101."""
    N = w.horizon
    n = N * (nx + nu)
    H = np.zeros((n, n))
    for k in range(N):
        uo, xo = _u_offset(k, nx, nu), _x_offset(k, nx, nu)
        H[uo:uo + nu, uo:uo + nu] = w.R
        H[xo:xo + nx, xo:xo + nx] = w.Q_N if k == N - 1 else w.Q
    return H


def build_sm(sys: LinearSystem, K: np.ndarray, N: int):
    """mpc.cpp:105-134."""
    nx, nu = sys.nx, sys.nu
    Abar = sys.A - sys.B @ K
    AjB = [sys.B]
    Aj = [np.eye(nx)]
    for _ in range(1, N):
        AjB.append(Abar @ AjB[-1])
    for _ in range(1, N + 1):
        Aj.append(Abar @ Aj[-1])
    S = np.zeros((N * (nx + nu), N * nu))
    M = np.empty((N * (nx + nu), nx))
    for k in range(N):
        uo, xo = _u_offset(k, nx, nu), _x_offset(k, nx, nu)
        M[uo:uo + nu, :] = -K @ Aj[k]
        S[uo:uo + nu, k * nu:(k + 1) * nu] = np.eye(nu)
        for j in range(k):
            S[uo:uo + nu, j * nu:(j + 1) * nu] = -K @ AjB[k - 1 - j]
        M[xo:xo + nx, :] = Aj[k + 1]
        for j in range(k + 1):
            S[xo:xo + nx, j * nu:(j + 1) * nu] = AjB[k - j]
    return S, M


def build_condensed_mpc(sys: LinearSystem, weights: MpcWeights, limits: BoxLimits,
                        K: np.ndarray) -> CondensedTemplate:
    """mpc.cpp:227-258. Raises ValueError when K is not stabilising."""
    nx, nu = sys.nx, sys.nu
    if K.shape != (nu, nx):
        raise ValueError("gain dimensions inconsistent")
    if weights.horizon < 1:
        raise ValueError("horizon must be >= 1")
    Abar = sys.A - sys.B @ K
    if spectral_radius(Abar) >= 1.0:
        raise ValueError("build_condensed_mpc: K is not stabilizing")
    S, M = build_sm(sys, K, weights.horizon)
    H = build_cost_hessian(weights, nx, nu)
    HS = H @ S
    Hbar = S.T @ HS
    Hbar = 0.5 * (Hbar + Hbar.T)
    offset_g = HS.T @ M
    G_lim, c, d = build_limit_rows(sys, limits, weights.horizon)
    return CondensedTemplate(K=K, Abar=Abar, S=S, M=M, Hbar=np.asfortranarray(Hbar),
                             Gbar=np.asfortranarray(G_lim @ S),
                             offset_g=np.asfortranarray(offset_g),
                             offset_c=np.asfortranarray(G_lim @ M), c_base=c, d_base=d,
                             nx=nx, nu=nu, horizon=weights.horizon)


def instantiate(tmpl: CondensedTemplate, x0: np.ndarray):
    """mpc.cpp:260-270 -> (H, g, G, c, d); H and G are the template's (shared) matrices."""
    x0 = np.asarray(x0, dtype=np.float64).reshape(-1)
    if x0.size != tmpl.nx:
        raise ValueError("instantiate: x0 dimension mismatch")
    g = tmpl.offset_g @ x0
    shift = tmpl.offset_c @ x0
    return tmpl.Hbar, g, tmpl.Gbar, tmpl.c_base - shift, tmpl.d_base - shift
