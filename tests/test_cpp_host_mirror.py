"""The C++ host-side mirror of clampqp::Solver (csrc/host/clampqp_gpu.hpp) over the C ABI:
compiles everywhere; on a GPU box the reference-style C++ checks in tests/cpp run green."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2311_18056_b200")
EXE = os.path.join(ROOT, "tests", "cpp", "test_solver_gpu.bin")


def build_exe():
    from paper_2311_18056_b200 import _lib
    _lib.build()
    cmd = ["g++", "-std=c++17", "-O2", f"-I{ROOT}/include", f"-I{PKG}/csrc/host",
           os.path.join(ROOT, "tests", "cpp", "test_solver_gpu.cpp"), "-o", EXE, f"-L{PKG}", "-lcqp_b200",
           f"-Wl,-rpath,{PKG}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.check_call(cmd)


def test_cpp_mirror_compiles_and_fails_loudly_without_gpu():
    from paper_2311_18056_b200 import _lib
    build_exe()
    if _lib.load().cqp_device_count() > 0:
        pytest.skip("a CUDA device is present")
    r = subprocess.run([EXE], capture_output=True, text=True)
    assert r.returncode != 0
    assert "no CPU fallback" in (r.stderr + r.stdout)


@pytest.mark.gpu
def test_cpp_mirror_reference_style_checks():
    build_exe()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL C++ HOST-MIRROR CHECKS PASSED" in r.stdout
