"""MT19937-64 jump-ahead of the device generator (CPU).

The device generates the reference's one std::mt19937_64 stream
(random.hpp:111-129) in parallel stretches whose start windows come from
jump-ahead polynomials x^J mod phi (paper_1308_2400_b200/csrc/mt64jump.h).
tests/cpp/test_mt64jump.cpp checks, against std::mt19937_64 itself
(discard(J) then 312 draws), that phi has degree 19937 and that jumped
windows -- single, chained and via a product of jump polynomials -- equal the
stream's outputs; built with the carry-less-multiply instructions the library
uses and with the portable fallback.
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("flags", [["-mpclmul"], []], ids=["pclmul", "portable"])
def test_jump_ahead_matches_std_mt19937_64(tmp_path, flags):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    exe = tmp_path / "test_mt64jump"
    subprocess.run(["g++", "-std=c++17", "-O2", *flags,
                    "-I", os.path.join(ROOT, "paper_1308_2400_b200", "csrc"),
                    "-o", str(exe), os.path.join(ROOT, "tests", "cpp", "test_mt64jump.cpp")],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stdout + r.stderr
