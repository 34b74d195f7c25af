"""JSON problem documents and the `solve` command: the on-disk format
either side of the solve path, so that problem files and solver output can be exchanged with a
machine that runs the reference itself.

  parse_problem / serialize_problem   /root/reference/proj/src/problem.cpp:166-203
      {"n", "m", "H" (n rows), "g", "G" (m rows), "c", "d"}; scalars are numbers or the tokens
      "inf" / "-inf"; magnitudes >= 1e30 read as infinity (problem.cpp:25,31-46); canonical key
      order and two-space indentation on output; values round-trip bit for bit.
  cmd_solve                           /root/reference/proj/tools/main.cpp:43-74
      `python -m paper_2311_18056_b200.problem_io solve problem.json` prints the reference CLI's
      key: value lines (status, iterations, r_prim, r_dual, y, z, lambda, wall_ms; %.12g) and exits
      0 when solved, 2 otherwise, 1 on a malformed document.  The solve runs on the GPU through
      the C ABI (no CPU fallback).
"""
from __future__ import annotations

import json
import math
import sys
from dataclasses import dataclass

import numpy as np


@dataclass
class DenseQP:
    """QProblem of the reference (/root/reference/proj/include/clampqp/problem.hpp:31-40): min 1/2 y'Hy + g'y
    subject to c <= Gy <= d, dense, column-major on the device side."""
    H: np.ndarray
    g: np.ndarray
    G: np.ndarray
    c: np.ndarray
    d: np.ndarray

    @property
    def n(self) -> int:
        return self.H.shape[0]

    @property
    def m(self) -> int:
        return self.G.shape[0]


INF_THRESHOLD = 1e30  # problem.cpp:25


class ProblemFormatError(ValueError):
    """ProblemError codes MalformedDocument / MissingField / DimensionMismatch (problem.hpp:75-83)."""

    def __init__(self, code: str, message: str):
        super().__init__(f"{code}: {message}")
        self.code = code


def _scalar(j, field: str) -> float:
    if isinstance(j, str):
        if j == "inf":
            return math.inf
        if j == "-inf":
            return -math.inf
        raise ProblemFormatError("MalformedDocument", f'unrecognized token "{j}" in field {field}')
    if isinstance(j, bool) or not isinstance(j, (int, float)):
        raise ProblemFormatError("MalformedDocument", f"non-numeric entry in field {field}")
    v = float(j)
    if v >= INF_THRESHOLD:
        return math.inf
    if v <= -INF_THRESHOLD:
        return -math.inf
    return v


def _vector(j, field: str, length: int) -> np.ndarray:
    if not isinstance(j, list):
        raise ProblemFormatError("MalformedDocument", f"{field} must be an array")
    if len(j) != length:
        raise ProblemFormatError("MissingField", f"{field} has length {len(j)}, expected {length}")
    return np.array([_scalar(x, field) for x in j], dtype=np.float64)


def _matrix(j, field: str, rows: int, cols: int) -> np.ndarray:
    if not isinstance(j, list):
        raise ProblemFormatError("MalformedDocument", f"{field} must be an array")
    if len(j) != rows:
        raise ProblemFormatError("MissingField", f"{field} has {len(j)} rows, expected {rows}")
    out = np.empty((rows, cols), order="F")
    for i, row in enumerate(j):
        out[i, :] = _vector(row, field, cols)
    return out


def parse_problem(text: str) -> DenseQP:
    """problem.cpp:166-190 (validation of H / bounds happens in the Solver constructor, on the GPU
    path: cqp_create reports NonSymmetricH / NonPositiveDefiniteH / InvertedBounds / NonFiniteEntry)."""
    try:
        doc = json.loads(text, parse_constant=lambda tok: (_ for _ in ()).throw(ValueError(tok)))
    except ValueError as e:
        raise ProblemFormatError("MalformedDocument", f"parse error: {e}") from None
    if not isinstance(doc, dict):
        raise ProblemFormatError("MalformedDocument", "document must be an object")
    for field in ("n", "m"):
        if field not in doc:
            raise ProblemFormatError("MissingField", f"missing field {field}")
    n, m = doc["n"], doc["m"]
    if isinstance(n, bool) or isinstance(m, bool) or not isinstance(n, int) or not isinstance(m, int):
        raise ProblemFormatError("MalformedDocument", "n and m must be integers")
    if n < 1 or m < 1:
        raise ProblemFormatError("DimensionMismatch", "n and m must be >= 1")
    for field in ("H", "g", "G", "c", "d"):
        if field not in doc:
            raise ProblemFormatError("MissingField", f"missing field {field}")
    return DenseQP(_matrix(doc["H"], "H", n, n), _vector(doc["g"], "g", n), _matrix(doc["G"], "G", m, n),
                   _vector(doc["c"], "c", m), _vector(doc["d"], "d", m))


def _enc(v: float):
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return float(v)


def serialize_problem(p: DenseQP) -> str:
    """problem.cpp:192-203: canonical key order, indent 2, trailing newline.  Python's float repr is
    the shortest string that round-trips, like the reference's JSON library."""
    H, G = np.asarray(p.H, dtype=np.float64), np.asarray(p.G, dtype=np.float64)
    doc = {"n": int(H.shape[0]), "m": int(G.shape[0]),
           "H": [[_enc(x) for x in row] for row in H.tolist()],
           "g": [_enc(x) for x in np.asarray(p.g, dtype=np.float64).tolist()],
           "G": [[_enc(x) for x in row] for row in G.tolist()],
           "c": [_enc(x) for x in np.asarray(p.c, dtype=np.float64).tolist()],
           "d": [_enc(x) for x in np.asarray(p.d, dtype=np.float64).tolist()]}
    return json.dumps(doc, indent=2) + "\n"


_STATUS = {0: "solved", 1: "max-iters", 2: "invalid"}  # to_string(SolveStatus), problem.cpp:108-119


def format_vector(v) -> str:
    return " ".join("%.12g" % x for x in np.asarray(v, dtype=np.float64))  # main.cpp:32-40


def format_report(report) -> str:
    """The key: value lines of `clampqp solve` (main.cpp:64-71)."""
    sol = report.solution
    return "\n".join([f"status: {_STATUS.get(sol.status, 'invalid')}", f"iterations: {sol.iterations}",
                      "r_prim: %.12g" % sol.r_prim, "r_dual: %.12g" % sol.r_dual,
                      "y: " + format_vector(sol.y), "z: " + format_vector(sol.z),
                      "lambda: " + format_vector(sol.lam), "wall_ms: %.3f" % report.wall_ms]) + "\n"


def cmd_solve(path: str, settings=None, out=sys.stdout, err=sys.stderr) -> int:
    """main.cpp:43-74 with the GPU Solver behind it."""
    from . import solver as S
    try:
        text = open(path).read()
    except OSError:
        err.write(f"error: cannot open {path}\n")
        return 1
    try:
        p = parse_problem(text)
        gpu = S.Solver(p.H, p.g, p.G, p.c, p.d, settings or S.SolverSettings())
    except (ProblemFormatError, S.ProblemError) as e:
        err.write(f"error: {e}\n")
        return 1
    report = gpu.solve()
    out.write(format_report(report))
    gpu.close()
    return 0 if report.solution.status == S.SOLVED else 2


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    if len(argv) == 2 and argv[0] == "solve":
        return cmd_solve(argv[1])
    sys.stderr.write("usage: python -m paper_2311_18056_b200.problem_io solve <problem.json>\n")
    return 1


if __name__ == "__main__":
    sys.exit(main())
