"""The SFU-free quotient of the QSGD quantiser (div_rn_fma, csrc/nebula_internal.cuh) against
the IEEE division, exhaustively over every binary32 significand of p in 30 binades around each
of 4096 scales s (random significands and the edge ones), both signs: bit-identical.  The
parity tests then check the whole QSGD codec against the oracle (R32: x = fl(p / s))."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_div_rn_fma_is_ieee_division(tmp_path):
    exe = tmp_path / "div_check"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false", "-prec-div=true",
                    "-std=c++17", "-o", str(exe), os.path.join(ROOT, "tests", "cuda", "div_check.cu")],
                   check=True, timeout=300)
    r = subprocess.run([str(exe), "4096"], capture_output=True, text=True, timeout=600)
    assert "DIV_CHECK mismatches=0" in r.stdout, r.stdout + r.stderr
    assert r.returncode == 0
