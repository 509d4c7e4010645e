"""Regression for the two-stream TOPK step at BASELINE config 2 size (ERNIE-M-base, LOOPBACK
P = 2, 25 MiB buckets) with more buckets on the multi-CTA resolve path (threshold lowered to
32768 candidates through the NEBULA_DEBUG_WIDE_MIN hook, read once per process — hence the
subprocesses).  Before the halves' multi-CTA resolve sections were ordered, 2 % and 5 % density
faulted (illegal address) in 4 of 4 runs of the loop below.  Now: no fault, and the two-stream
outputs equal the one-stream outputs bit for bit at every step."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(script, *args):
    env = dict(os.environ, NEBULA_DEBUG_WIDE_MIN="32768")
    return subprocess.run([sys.executable, os.path.join(ROOT, "scripts", script), *map(str, args)],
                          capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)


@pytest.mark.gpu
@pytest.mark.parametrize("rho", [0.02, 0.05])
def test_two_stream_topk_no_fault(rho):
    r = _run("topk_pipeline_loop.py", rho, 20, 1)
    assert "LOOP OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_two_stream_topk_equals_one_stream():
    r = _run("topk_pipeline_stress.py", 0.05, 8)
    assert r.returncode == 0 and "differ" not in r.stdout and r.stdout.count(" ok") == 8, r.stdout[-2000:] + r.stderr[-2000:]
