"""JSON problem documents and the `solve` command.  The CPU part re-asserts
the reference's own format tests (/root/reference/proj/tests/test_problem.cpp:116-197); the GPU part
runs `solve` on a document through the C ABI and checks the printed report against the oracle."""
import io
import math

import numpy as np
import pytest

from paper_2311_18056_b200 import problem_io as IO
from workloads import problems


def box_1d():
    return problems.DenseQP(np.array([[2.0]]), np.array([-2.0]), np.array([[1.0]]), np.array([0.0]), np.array([0.5]))


def test_parse_maps_inf_tokens_and_huge_magnitudes():          # test_problem.cpp:116-129
    doc = '{"n": 1, "m": 2, "H": [[2.0]], "g": [-2.0], "G": [[1.0], [1.0]], "c": ["-inf", -1e31], "d": ["inf", 0.5]}'
    p = IO.parse_problem(doc)
    assert p.c[0] == -math.inf and p.c[1] == -math.inf and p.d[0] == math.inf and p.d[1] == 0.5


def test_serialize_emits_inf_tokens_and_canonical_key_order():   # test_problem.cpp:131-143
    p = box_1d()
    p.c[0] = -math.inf
    doc = IO.serialize_problem(p)
    assert '"-inf"' in doc
    order = [doc.find(f'"{k}"') for k in ("n", "m", "H", "g", "G", "c", "d")]
    assert order == sorted(order) and min(order) >= 0


def test_serialize_then_parse_is_the_identity():                 # test_problem.cpp:145-157
    p = box_1d()
    doc = IO.serialize_problem(p)
    q = IO.parse_problem(doc)
    for k in "HgGcd":
        assert np.array_equal(getattr(p, k), getattr(q, k))
    assert IO.serialize_problem(q) == doc


def test_parse_reports_missing_field_short_c_and_garbage():      # test_problem.cpp:159-177
    with pytest.raises(IO.ProblemFormatError):
        IO.parse_problem('{"n": 1, "m": 1}')
    short_c = '{"n": 1, "m": 2, "H": [[2.0]], "g": [-2.0], "G": [[1.0], [1.0]], "c": [0.0], "d": [0.5, 0.5]}'
    with pytest.raises(IO.ProblemFormatError) as e:
        IO.parse_problem(short_c)
    assert e.value.code == "MissingField"
    with pytest.raises(IO.ProblemFormatError):
        IO.parse_problem("not json")
    with pytest.raises(IO.ProblemFormatError):
        IO.parse_problem('{"n": 1, "m": 1, "H": [["x"]], "g": [0], "G": [[1]], "c": [0], "d": [1]}')
    with pytest.raises(IO.ProblemFormatError):
        IO.parse_problem('{"n": 1.5, "m": 1, "H": [[1]], "g": [0], "G": [[1]], "c": [0], "d": [1]}')


def test_all_equality_problem_round_trips():                     # test_problem.cpp:179-187
    p = box_1d()
    p.G = np.array([[1.0], [2.0]])
    p.c = np.array([0.3, 0.6])
    p.d = p.c.copy()
    q = IO.parse_problem(IO.serialize_problem(p))
    assert np.array_equal(q.c, q.d) and np.array_equal(q.c, p.c)


def test_round_trip_is_bit_exact_on_random_problems():           # test_problem.cpp:189-197
    for seed in range(10):
        p = problems.gen_random_dense_qp(8, seed)
        q = IO.parse_problem(IO.serialize_problem(p))
        for k in "HgGcd":
            assert np.array_equal(getattr(p, k), getattr(q, k))


def test_format_vector_matches_printf_12g():
    assert IO.format_vector([0.5, -1.0 / 3.0, 1e-20, 12345678901234.0]) == "0.5 -0.333333333333 1e-20 1.23456789012e+13"


@pytest.mark.gpu
def test_solve_command_on_a_document(tmp_path, oracle):
    """`solve problem.json` (main.cpp:43-74): document -> GPU Solver -> the reference CLI's report."""
    p = problems.gen_random_dense_qp(20, 4)
    path = tmp_path / "qp.json"
    path.write_text(IO.serialize_problem(p))
    out, err = io.StringIO(), io.StringIO()
    rc = IO.cmd_solve(str(path), out=out, err=err)
    ref = oracle.Solver(oracle.QProblem(p.H, p.g, p.G, p.c, p.d), variant="ref").solve()
    fields = dict(line.split(": ", 1) for line in out.getvalue().strip().split("\n"))
    assert rc == 0 and fields["status"] == "solved"
    assert int(fields["iterations"]) == ref.solution.iterations
    y = np.array([float(x) for x in fields["y"].split()])
    lam = np.array([float(x) for x in fields["lambda"].split()])
    assert np.abs(y - ref.solution.y).max() <= 1e-6 * max(1.0, np.abs(ref.solution.y).max())
    assert np.abs(lam - ref.solution.lam).max() <= 1e-6 * max(1.0, np.abs(ref.solution.lam).max())
    assert float(fields["r_prim"]) <= 1e-6 and float(fields["r_dual"]) <= 1e-6
    # malformed documents and invalid problems exit with 1 and an "error:" line
    bad = tmp_path / "bad.json"
    bad.write_text('{"n": 1, "m": 1, "H": [[-1.0]], "g": [0.0], "G": [[1.0]], "c": [0.0], "d": [1.0]}')
    err = io.StringIO()
    assert IO.cmd_solve(str(bad), out=io.StringIO(), err=err) == 1 and "NonPositiveDefiniteH" in err.getvalue()
    assert IO.cmd_solve(str(tmp_path / "missing.json"), out=io.StringIO(), err=io.StringIO()) == 1
