"""Bit-exact Python/numpy restatement of the reference's benchmark RNG.

Reference: `bench::Rng` (/root/reference/proj/include/clampqp/bench.hpp:29-47,
src/bench.cpp:58-87): `std::mt19937_64` plus a hand-rolled Box-Muller with a cached spare, so
that input streams are identical across implementations.  This module only produces synthetic
INPUTS (host side, offline); it is not on the solve path.
"""
from __future__ import annotations

import math

import numpy as np

_NN, _MM = 312, 156
_MATRIX_A = np.uint64(0xB5026F5AA96619E9)
_UM = np.uint64(0xFFFFFFFF80000000)
_LM = np.uint64(0x7FFFFFFF)
_MASK64 = 0xFFFFFFFFFFFFFFFF
_TWO_PI = 6.283185307179586  # bench.cpp:27


class Rng:
    """mt19937_64 (bit-specified by the C++ standard) + Box-Muller, as bench.hpp:29-47."""

    def __init__(self, seed: int):
        mt = [0] * _NN
        mt[0] = seed & _MASK64
        for i in range(1, _NN):
            prev = mt[i - 1]
            mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _MASK64
        self._mt = np.array(mt, dtype=np.uint64)
        self._out = None
        self._idx = _NN
        self._has_spare = False
        self._spare = 0.0

    def _twist(self) -> None:
        mt = self._mt
        one = np.uint64(1)

        def mix(upper, lower, far):
            x = (upper & _UM) | (lower & _LM)
            return far ^ (x >> one) ^ ((x & one) * _MATRIX_A)

        # i in [0, NN-MM): reads only not-yet-updated words
        mt[: _NN - _MM] = mix(mt[: _NN - _MM], mt[1: _NN - _MM + 1], mt[_MM:])
        # i in [NN-MM, NN-1): far word mt[i + MM - NN] was updated above
        mt[_NN - _MM: _NN - 1] = mix(mt[_NN - _MM: _NN - 1], mt[_NN - _MM + 1:], mt[: _MM - 1])
        mt[_NN - 1] = mix(mt[_NN - 1: _NN], mt[0:1], mt[_MM - 1: _MM])[0]
        x = mt.copy()
        x ^= (x >> np.uint64(29)) & np.uint64(0x5555555555555555)
        x ^= (x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        x ^= (x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        x ^= x >> np.uint64(43)
        self._out = x
        self._idx = 0

    def next_u64(self) -> int:
        if self._idx >= _NN:
            self._twist()
        v = int(self._out[self._idx])
        self._idx += 1
        return v

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        """bench.hpp:36-37."""
        u = float(self.next_u64() >> 11) * 2.0 ** -53
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def normal(self) -> float:
        """bench.cpp:58-73."""
        if self._has_spare:
            self._has_spare = False
            return self._spare
        u1 = 0.0
        while u1 <= 0.0:
            u1 = self.uniform()
        u2 = self.uniform()
        radius = math.sqrt(-2.0 * math.log(u1))
        angle = _TWO_PI * u2
        self._spare = radius * math.sin(angle)
        self._has_spare = True
        return radius * math.cos(angle)

    def normal_vector(self, n: int) -> np.ndarray:
        """bench.cpp:75-79."""
        return np.array([self.normal() for _ in range(n)], dtype=np.float64)

    def normal_matrix(self, rows: int, cols: int) -> np.ndarray:
        """bench.cpp:81-87: filled row by row; returned column-major like Eigen::MatrixXd."""
        flat = np.array([self.normal() for _ in range(rows * cols)], dtype=np.float64)
        return np.asfortranarray(flat.reshape(rows, cols))
