"""Multi-GPU parity run (one process per GPU, NCCL transport), launched with torchrun:

    torchrun --standalone --nproc-per-node N tools/nccl_check.py --scale 16 --roots 8 [--peer]
    torchrun ... tools/nccl_check.py --scale 28 --roots 1 --peer --device-gen --stream-validate

Every rank contributes its slice of the tuple list; the per-rank outputs (owned vertex blocks)
are gathered on rank 0 through the C ABI's bfs_gather and checked there:
  default            element by element against the CPU oracle's level[] / parent[] / m_comp;
  --stream-validate  with the oracle's streaming Graph500 validator V1-V6 + m_comp, which
                     regenerates the tuples from the seed chunk by chunk (full-size graphs:
                     V1-V6 passing is equivalent to bit-exact equality).
Prints one JSON line on rank 0 and exits non-zero on any mismatch.
"""
import argparse
import json
import os
import sys
import time

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
    ap.add_argument("--stream-validate", action="store_true", help="V1-V6 streaming validator instead of the oracle BFS")
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
    g = bfs.Graph(s, d, n, R, C, comm=comm,
                  opts=bfs.make_opts(edges_per_thread=4, exchange=a.exchange, peer_exchange=a.peer))
    del s, d
    torch.cuda.empty_cache()
    info = g.info
    roots, t = [], 0
    while len(roots) < a.roots:
        v = inputs.root_candidate(inputs.ROOT_SEED, t, n)
        t += 1
        if v not in roots and g.degree(v) > 0:
            roots.append(v)
    # rank-local outputs in HBM; bfs_gather collects them on rank 0 (host buffers there)
    parent = torch.empty(info.nout, dtype=torch.int64, device="cuda")
    level = torch.empty(info.nout, dtype=torch.int32, device="cuda")
    pall = np.empty(info.npad, dtype=np.int64) if rank == 0 else None
    lall = np.empty(info.npad, dtype=np.int32) if rank == 0 else None
    ok, bad, checked = True, [], []
    og = None
    batch_check = a.scale <= 20  # bfs_run_batch vs the single runs (rank-local outputs kept on the host)
    single = []
    for r in roots:
        g.run(r, parent, level)  # the first root runs the host-driven loop, later roots the graph loop
        mc = g.mcomp()
        if batch_check:
            single.append((parent.cpu().numpy().copy(), level.cpu().numpy().copy()))
        g.gather(parent, level, pall, lall)
        if rank != 0:
            continue
        t0 = time.time()
        if a.stream_validate:
            import oracle
            step = 1 << 26
            chunks = (inputs.generate(a.scale, k0=k, count=min(step, M - k)) for k in range(0, M, step))
            mask, omc = oracle.validate_stream(n, r, lall[:n], pall[:n], chunks)
            good = mask == 0 and omc == mc
            checked.append({"root": r, "mask": mask, "failed": oracle.failed_names(mask), "mcomp": mc,
                            "oracle_mcomp": omc, "check_s": round(time.time() - t0, 1)})
        else:
            import oracle
            if og is None:
                hs, hd = inputs.generate(a.scale)
                og = oracle.Graph(n, hs, hd)
            ol, op = og.bfs(r)
            good = (np.array_equal(lall[:n], ol) and np.array_equal(pall[:n], op) and mc == og.mcomp(ol)
                    and (lall[n:] == -1).all() and (pall[n:] == -1).all())
        if not good:
            bad.append(r)
    batch_bad = []
    if batch_check:  # the same roots through bfs_run_batch into pinned host buffers (copies overlap searches)
        pb = [torch.empty(info.nout, dtype=torch.int64).pin_memory() for _ in roots]
        lb = [torch.empty(info.nout, dtype=torch.int32).pin_memory() for _ in roots]
        g.run_batch(roots, pb, lb)
        batch_bad = [r for r, (sp, sl), p_, l_ in zip(roots, single, pb, lb)
                     if not (np.array_equal(p_.numpy(), sp) and np.array_equal(l_.numpy(), sl))]
        flag = torch.tensor([len(batch_bad)], device="cuda")
        dist.all_reduce(flag)
        if flag.item():
            bad.append("run_batch")
    dist.barrier()
    g.close()
    report = {"world": world, "grid": f"{R}x{C}", "scale": a.scale, "roots": len(roots), "block": int(info.block),
              "transport": "peer" if a.peer else "nccl", "exchange": a.exchange,
              "check": "stream-validator V1-V6 + m_comp" if a.stream_validate else "bit-exact vs oracle",
              "run_batch_checked": batch_check}
    if rank == 0:
        ok = not bad
        report.update({"ok": ok, "mismatched_roots": bad})
        if checked:
            report["validated"] = checked
        print(json.dumps(report), flush=True)
    okt = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(okt, 0)
    dist.destroy_process_group()
    sys.exit(0 if okt.item() else 1)


if __name__ == "__main__":
    main()
