"""Small BFS workload for memory-safety runs (the BFS200_CHECKS=1 bounds-checked build through
BFS200_LIB -- tests/test_gpu_checked.py -- or compute-sanitizer where a pool allows it):
Kronecker s12 on the 1x1 and 2x2 loopback grids, host-driven and CUDA-graph level loops, every
K1/K3/K4/K2 path (P1, mode 3, P2 levels; long and short tiles), outputs checked against the
oracle so a sanitizer-perturbed run is also a parity run.

    BFS200_LIB=paper_1408_1605_b200/build/variants/libchecked.so SAN_SCALE=18 python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1408_1605_b200 import bfs, inputs  # noqa: E402

scale = int(os.environ.get("SAN_SCALE", "12"))
s, d = inputs.generate(scale)
n = 1 << scale
og = oracle.Graph(n, s, d)
roots = inputs.sample_roots(n, 3, inputs.nonisolated_mask(n, s, d))
ts = torch.from_numpy(s.view(np.int64)).cuda()
td = torch.from_numpy(d.view(np.int64)).cuda()
bad = 0
for R, C in ((1, 1), (2, 2)):
    g = bfs.Graph(ts, td, n, R, C, comm=bfs.make_comm(loopback=True))
    for phase in (False, True):
        g.set_opts(bfs.make_opts(edges_per_thread=4, phase_timing=phase))
        for r in roots:
            lv, pa = g.bfs(r)
            ol, op = og.bfs(r)
            if not (np.array_equal(lv[:n], ol) and np.array_equal(pa[:n], op)):
                bad += 1
    g.close()
print("sanitize_run", "OK" if bad == 0 else f"MISMATCH {bad}")
sys.exit(1 if bad else 0)
