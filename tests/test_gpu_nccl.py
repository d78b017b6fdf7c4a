"""NCCL transport parity (one process per GPU through torchrun); needs >= 2 GPUs, else skipped.
The same 2D logic is covered on one GPU by the loopback grids of test_gpu_parity.py."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nproc,grid,exchange", [(2, "1x2", "bitmap"), (2, "2x1", "bitmap"), (4, "2x2", "bitmap"),
                                                 (2, "1x2", "list"), (2, "2x1", "auto"), (4, "2x2", "list"),
                                                 (4, "2x2", "auto"), (2, "1x2", "peer"), (2, "2x1", "peer"),
                                                 (4, "2x2", "peer"), (4, "1x4", "peer"), (4, "4x1", "peer")])
def test_nccl_parity(nproc, grid, exchange):
    if not torch.cuda.is_available() or torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", str(nproc),
           os.path.join(ROOT, "tools", "nccl_check.py"), "--scale", "15", "--roots", "6", "--grid", grid,
           *(["--peer"] if exchange == "peer" else ["--exchange", exchange])]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    rep = json.loads(lines[-1])
    assert rep["ok"] and rep["grid"] == grid
