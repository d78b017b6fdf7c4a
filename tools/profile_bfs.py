"""Profiling driver: build the scale-S Kronecker graph on one GPU and run a few BFS roots
(the bench workload, bench launch options).  Used under ncu; prints per-level phase times."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1408_1605_b200 import bfs, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--roots", type=int, default=1)
ap.add_argument("--E", type=int, default=4)
ap.add_argument("--grid", default="1x1")
a = ap.parse_args()
R, C = (int(x) for x in a.grid.split("x"))
n = 1 << a.scale
ds, dd = inputs.generate_device(a.scale)
stream = torch.cuda.current_stream()
g = bfs.Graph(ds, dd, n, R, C, comm=bfs.make_comm(loopback=True),
              opts=bfs.make_opts(edges_per_thread=a.E, phase_timing=True, stream=stream.cuda_stream))
del ds, dd
torch.cuda.empty_cache()
roots, t = [], 0
while len(roots) < a.roots:
    v = inputs.root_candidate(inputs.ROOT_SEED, t, n)
    t += 1
    if g.degree(v) > 0:
        roots.append(v)
parent = torch.empty(g.info.nout, dtype=torch.int64, device="cuda")
level = torch.empty(g.info.nout, dtype=torch.int32, device="cuda")
for r in roots:
    st = g.run(r, parent, level)
    recs = g.level_times()
    print(f"root {r}: levels {st.nlevels} edges {st.edges_scanned} mcomp {g.mcomp()} "
          f"finalize {st.finalize_ms:.3f} ms resolve {st.resolve_ms:.3f} ms")
    for i, x in enumerate(recs):
        print(f"  L{i}: frontier {x.frontier:>10} edges {x.edges:>12} scan {x.scan:7.3f} expand {x.expand:7.3f} "
              f"parent {x.parent:6.3f} update {x.update:6.3f} ms  -> "
              f"{((4*x.edges+40*x.frontier)/1e9)/(max(x.expand,1e-6)*1e-3):8.1f} GB/s (4E+40F over K1)")
g.close()
