"""Runs the C++ drop-in test (tests/cpp/test_gpu_kernels.cpp): the reference's own
kernel tests against afmm::gpu::afmm_case_{a,b}, linked to libafmm_b200.so and
compiled against the reference headers in the build container."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "test_gpu_kernels")


@pytest.mark.gpu
def test_cpp_dropin_against_reference_tests(cuda):
    if not os.path.exists(BIN):
        pytest.skip("build/test_gpu_kernels not built (needs the reference headers)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_cpp_dropin_builds():
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference headers not present")
    r = subprocess.run(["make", "-C", ROOT, "cpptest"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert os.path.exists(BIN)
