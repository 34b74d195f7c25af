"""Synthetic workload generators (bench / test inputs, host side, numpy).

Not part of the product package: `paper_2311_18056_b200/` holds only the solve path.  These
modules restate the reference's out-of-scope generators (`proj/src/bench.cpp`, `proj/src/mpc.cpp`,
`proj/src/rng.hpp` sampling rules) so that the GPU path and the CPU oracle are fed the same
bit-specified inputs.
"""
