"""Write tests/golden/snap_small.txt: a small graph in the SNAP text format (SPEC.md S:55-63,
External Interfaces) for the loader tests -- '#' header lines as SNAP files have them, tab- and
space-separated ids, sparse non-contiguous ids, duplicates, reversed duplicates, self-loops, a
second component, isolated ids only implied by max id, CRLF on some lines and no newline after
the last line.  Seeded; the expected BFS results come from the oracle at test time."""
import os

import numpy as np

rng = np.random.default_rng(1408)
ids = np.sort(rng.choice(5000, size=300, replace=False)) + 7  # sparse ids, max < 5008
# component A: 240 vertices, preferential-attachment-like; component B: 40 vertices, a cycle + chords
A, B = ids[:240], ids[240:280]
edges = []
for k in range(1, len(A)):
    for _ in range(1 + (k % 3 == 0)):
        j = int(rng.integers(0, k)) if rng.random() < 0.5 else int(min(k - 1, rng.zipf(1.6) - 1))
        edges.append((int(A[k]), int(A[j])))
for k in range(len(B)):
    edges.append((int(B[k]), int(B[(k + 1) % len(B)])))
    if k % 7 == 0:
        edges.append((int(B[k]), int(B[(k + 13) % len(B)])))
edges += [edges[5], (edges[9][1], edges[9][0]), (int(A[3]), int(A[3])), (int(B[2]), int(B[2]))]
order = rng.permutation(len(edges))
lines = ["# Undirected graph (each unordered pair of nodes is saved once): snap_small.txt",
         "# Synthetic fixture for the loader tests (tools/make_snap_fixture.py, seed 1408)",
         f"# Nodes: {len(set(a for e in edges for a in e))} Edges: {len(edges)}",
         "# FromNodeId\tToNodeId"]
for n, k in enumerate(order):
    a, b = edges[k]
    sep = "\t" if n % 2 == 0 else "  "
    end = "\r" if n % 11 == 0 else ""
    lines.append(f"{a}{sep}{b}{end}")
    if n == 100:
        lines.append("")  # a blank line inside the body
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "snap_small.txt")
with open(out, "w", newline="") as f:
    f.write("\n".join(lines))  # no newline after the last line
print(out, len(edges), "tuples")
