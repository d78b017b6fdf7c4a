"""Host-side logic of the N>1 path on CPU: two gloo ranks (world_size 2, 127.0.0.1).

Covers bench.py's max-over-ranks step time, the collective root sampling (every rank must get
the same roots from the same candidate stream) and the weak-scaling workload per world size."""
import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import numpy as np
    from paper_1408_1605_b200 import inputs
    # max over ranks of per-rank times
    t = bench.max_over_ranks_dist(1.0 + rank, world, "cpu")
    # collective degree: each rank holds half of the tuple list; the degree of v is the sum
    scale = 10
    n = 1 << scale
    M = inputs.num_tuples(scale)
    s, d = inputs.generate(scale, k0=M * rank // world, count=M * (rank + 1) // world - M * rank // world)

    def degree(v):
        local = int(np.count_nonzero((s == v) & (d != v)) + np.count_nonzero((d == v) & (s != v)))
        x = torch.tensor([local], dtype=torch.int64)
        dist.all_reduce(x)
        return int(x.item())

    roots = bench.sample_roots_collective(n, 16, degree)
    allr = [None] * world
    dist.all_gather_object(allr, roots)
    q.put((rank, t, roots, allr))
    dist.destroy_process_group()


def test_two_gloo_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_1408_1605_b200 import inputs
    s, d = inputs.generate(10)
    elig = inputs.nonisolated_mask(1 << 10, s, d)
    expect = inputs.sample_roots(1 << 10, 16, elig)
    for rank, t, roots, allr in out:
        assert t == 2.0                      # max over ranks
        assert roots == expect               # collective degree == full-graph eligibility
        assert allr[0] == allr[1] == expect  # identical on every rank


def test_weak_scaling_workloads():
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    a = argparse.Namespace(scale=0, E=4, grid="")
    cfgs = {w: bench.workload_config(a, w) for w in (1, 2, 4, 8)}
    assert [cfgs[w]["scale"] for w in (1, 2, 4, 8)] == [26, 27, 28, 29]
    assert [cfgs[w]["grid"] for w in (1, 2, 4, 8)] == ["1x1", "1x2", "2x2", "2x4"]
