"""Bounds-checked build (BFS200_CHECKS=1: every flist / tile table / tile record / CSC position /
row id / CSR scan result / finalize offset checked against its array's capacity, a violation
traps the kernel).  compute-sanitizer is closed on the GPU pool, so this build plus the oracle
comparison is the memory-safety check: tools/sanitize_run.py runs host- and graph-driven level
loops on the 1x1 and 2x2 loopback grids (s12: sparse and P1 levels; s18: the hot-copy K1 path
and long-tile pipeline) through the checked library and compares every output with the oracle."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("scale", [12, 18])
def test_checked_build_parity(scale):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1408_1605_b200 import _build
    lib = _build.build_variant("checked", ["BFS200_CHECKS=1"])
    env = dict(os.environ, BFS200_LIB=lib, SAN_SCALE=str(scale))
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], capture_output=True, text=True,
                       timeout=900, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    assert "sanitize_run OK" in p.stdout
