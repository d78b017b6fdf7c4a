"""Multi-GPU parity run (one process per GPU, NCCL transport), launched with torchrun:

    torchrun --standalone --nproc-per-node N tools/nccl_check.py --scale 16 --roots 8

Every rank contributes its slice of the tuple list; the per-rank outputs (owned vertex blocks)
are gathered on rank 0 and compared element by element with the CPU oracle.  Prints one JSON
line on rank 0 and exits non-zero on any mismatch.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1408_1605_b200 import bfs, inputs  # noqa: E402

GRIDS = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=16)
    ap.add_argument("--roots", type=int, default=8)
    ap.add_argument("--grid", default="")
    ap.add_argument("--device-gen", action="store_true", help="generate the slice on the GPU")
    ap.add_argument("--exchange", default="bitmap", choices=["bitmap", "list", "auto"])
    ap.add_argument("--peer", action="store_true", help="NVLink peer-memory exchange (opts.peer_exchange)")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    R, C = (int(x) for x in a.grid.split("x")) if a.grid else GRIDS[world]
    n = 1 << a.scale
    M = inputs.num_tuples(a.scale)
    k0, k1 = M * rank // world, M * (rank + 1) // world
    if a.device_gen:
        s, d = inputs.generate_device(a.scale, k0=k0, count=k1 - k0)
    else:
        s, d = inputs.generate(a.scale, k0=k0, count=k1 - k0)
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.tensor(list(bfs.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    comm = bfs.make_comm(rank, world, local, loopback=False, nccl_id=bytes(uid.cpu().tolist()))
    g = bfs.Graph(s, d, n, R, C, comm=comm, opts=bfs.make_opts(edges_per_thread=4, exchange=a.exchange, peer_exchange=a.peer))
    info = g.info
    roots, t = [], 0
    while len(roots) < a.roots:
        v = inputs.root_candidate(inputs.ROOT_SEED, t, n)
        t += 1
        if v not in roots and g.degree(v) > 0:
            roots.append(v)
    results = []
    for r in roots:
        lv, pa = g.bfs(r)
        mc = g.mcomp()
        tl = torch.from_numpy(lv).cuda()
        tp = torch.from_numpy(pa).cuda()
        gl = [torch.empty_like(tl) for _ in range(world)] if rank == 0 else None
        gp = [torch.empty_like(tp) for _ in range(world)] if rank == 0 else None
        dist.gather(tl, gl, 0)
        dist.gather(tp, gp, 0)
        if rank == 0:
            results.append((r, torch.cat(gl).cpu().numpy(), torch.cat(gp).cpu().numpy(), mc))
    g.close()
    ok = True
    report = {"world": world, "grid": f"{R}x{C}", "scale": a.scale, "roots": len(roots), "block": int(info.block)}
    if rank == 0:
        import oracle
        hs, hd = inputs.generate(a.scale)
        og = oracle.Graph(n, hs, hd)
        bad = []
        for r, lv, pa, mc in results:
            ol, op = og.bfs(r)
            if not (np.array_equal(lv[:n], ol) and np.array_equal(pa[:n], op) and mc == og.mcomp(ol)):
                bad.append(r)
        ok = not bad
        report.update({"ok": ok, "mismatched_roots": bad})
        print(json.dumps(report), flush=True)
    okt = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(okt, 0)
    dist.destroy_process_group()
    sys.exit(0 if okt.item() else 1)


if __name__ == "__main__":
    main()
