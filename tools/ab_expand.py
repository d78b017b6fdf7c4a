"""A/B driver for kernel experiments: one library build (BFS200_LIB or the default) on the bench
workload (Kronecker s26, 1x1 unless --grid), prints per-level phase times of a few roots, the
CUDA-graph BFS time (hmean GTEPS over the roots) and a digest of the outputs so variants can be
checked for identical results.

    BFS200_LIB=paper_1408_1605_b200/build/variants/libpipe3.so python tools/ab_expand.py --roots 8
"""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1408_1605_b200 import bfs, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--roots", type=int, default=8)
ap.add_argument("--grid", default="1x1")
ap.add_argument("--levels", action="store_true", help="print per-level phase times of the first root")
a = ap.parse_args()
R, C = (int(x) for x in a.grid.split("x"))
n = 1 << a.scale
ds, dd = inputs.generate_device(a.scale)
stream = torch.cuda.current_stream()
g = bfs.Graph(ds, dd, n, R, C, comm=bfs.make_comm(loopback=True),
              opts=bfs.make_opts(edges_per_thread=4, stream=stream.cuda_stream))
del ds, dd
torch.cuda.empty_cache()
roots, t = [], 0
while len(roots) < a.roots:
    v = inputs.root_candidate(inputs.ROOT_SEED, t, n)
    t += 1
    if v not in roots and g.degree(v) > 0:
        roots.append(v)
parent = torch.empty(g.info.nout, dtype=torch.int64, device="cuda")
level = torch.empty(g.info.nout, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in roots[:2]:  # warm-up (first run: host loop; graph built on the second)
    g.run(r, parent, level)
teps, dig = [], hashlib.sha1()
for r in roots:
    flush.zero_()
    torch.cuda.synchronize()
    e0.record(stream)
    g.run(r, parent, level)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    teps.append(g.mcomp() / (ms * 1e-3))
    dig.update(parent.cpu().numpy().tobytes())
    dig.update(level.cpu().numpy().tobytes())
hm = len(teps) / sum(1 / x for x in teps) / 1e9
# phase-timed replay
g.set_opts(bfs.make_opts(edges_per_thread=4, phase_timing=True, stream=stream.cuda_stream))
tot = {"scan": 0.0, "expand": 0.0, "parent": 0.0, "update": 0.0}
peak_e, peak_ms = 0.0, 0.0
for i, r in enumerate(roots):
    flush.zero_()
    torch.cuda.synchronize()
    st = g.run(r, parent, level)
    recs = g.level_times()
    for x in recs:
        for k in tot:
            tot[k] += getattr(x, k)
    top = max(recs, key=lambda x: x.edges)
    peak_e += 4.0 * top.edges + 40.0 * top.frontier
    peak_ms += top.expand
    if a.levels and i == 0:
        for li, x in enumerate(recs):
            print(f"  L{li}: frontier {x.frontier:>10} edges {x.edges:>12} scan {x.scan:7.3f} expand {x.expand:7.3f} "
                  f"parent {x.parent:6.3f} update {x.update:6.3f} ms")
lib = os.environ.get("BFS200_LIB", "default")
print(f"{os.path.basename(lib)}: {hm:.1f} GTEPS (graph loop, {len(roots)} roots); per BFS ms: " +
      " ".join(f"{k} {v / len(roots):.3f}" for k, v in tot.items()) +
      f"; peak-level K1 {peak_ms / len(roots):.3f} ms = {peak_e / 1e9 / (peak_ms * 1e-3):.0f} GB/s; digest {dig.hexdigest()[:12]}",
      flush=True)
g.close()
