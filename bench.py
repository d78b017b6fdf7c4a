#!/usr/bin/env python
"""bench.py -- harmonic-mean GTEPS of the 2D-partitioned top-down BFS (arXiv 1408.1605) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--scale S]

One step = one BFS (bfs_run: init, every level's expand exchange / scan / expansion / fold
exchange / update / termination, parent resolution, outputs written to HBM) from one of the
64 sampled roots of a Graph500 Kronecker graph (ef 16, A,B,C = .57,.19,.19; synthetic, seeded).
N=1 runs configs[2] (scale 26, 1x1); N>1 (torchrun, one rank per GPU) runs weak scaling at
scale 26 + log2(N) on the grids 1x2, 2x2, 2x4 (configs[4]'s grid shapes).  TEPS_i = m_comp_i /
t_i, t_i = max over ranks of the CUDA-event time of bfs_run on the library's
stream; value = harmonic mean of the K timed steps in GTEPS.  L2 is flushed between
steps (and the graph is > L2).  --impl reference times the CPU oracle on a bounded sample.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GTEPS (harmonic mean, 64 roots) Graph500 Kronecker ef16 at 1/2/4/8 B200"
UNIT = "GTEPS"
GRIDS = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}
REF_SAMPLE_SCALE = 20  # oracle sample graph for --impl reference / cpu_baseline steps


def hmean(xs):
    xs = [x for x in xs]
    return len(xs) / sum(1.0 / x for x in xs)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU oracle leg
def oracle_sample(steps: int, warmup: int, scale: int = REF_SAMPLE_SCALE):
    """Time the CPU oracle (as it stands) on `steps` roots of a scale-`scale` Kronecker graph."""
    import oracle
    from paper_1408_1605_b200 import inputs
    s, d = inputs.generate(scale)
    n = 1 << scale
    g = oracle.Graph(n, s, d)
    roots = inputs.sample_roots(n, 64, lambda v: g.degree(v) > 0)
    teps = []
    for k in range(warmup + steps):
        r = roots[k % len(roots)]
        t0 = time.perf_counter()
        lv, _ = g.bfs(r)
        t = time.perf_counter() - t0
        if k >= warmup:
            teps.append(g.mcomp(lv) / t)
    return hmean(teps) / 1e9, f"oracle BFS+parent pass, Kronecker scale {scale} ef16, {steps} roots (graph seed 1)"


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = workload_config(args, world)
    steps = max(1, args.steps)
    v, sample = oracle_sample(steps, max(0, args.warmup))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def max_over_ranks_dist(x: float, world: int, device) -> float:
    """Max of a per-rank scalar over all ranks (the step time of a multi-GPU run)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    tt = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return float(tt.item())


def sample_roots_collective(n, count, degree):
    """The first `count` distinct candidates of the root stream with degree(v) > 0.  `degree` is
    collective (bfs_degree), so every rank walks the same candidate sequence and gets the same
    roots."""
    from paper_1408_1605_b200 import inputs
    roots, seen, t = [], set(), 0
    while len(roots) < count and t < (1 << 22):
        v = inputs.root_candidate(inputs.ROOT_SEED, t, n)
        t += 1
        if v in seen:
            continue
        seen.add(v)
        if degree(v) > 0:
            roots.append(v)
    return roots


def grid_of(args, world):
    if getattr(args, "grid", ""):
        R, C = (int(x) for x in args.grid.lower().split("x"))
        if R * C != world:
            raise SystemExit(f"--grid {args.grid} needs {R * C} ranks, have {world}")
        return R, C
    return GRIDS.get(world, (1, world))


def workload_config(args, world):
    R, C = grid_of(args, world)
    scale = args.scale if args.scale else 26 + int(round(math.log2(world)))
    return {"workload": f"graph500-kronecker-s{scale}-ef16-{R}x{C}", "scale": scale, "edgefactor": 16,
            "grid": f"{R}x{C}", "roots": 64, "parallelism": f"2d-{R}x{C}", "edges_per_thread": args.E,
            "exchange": getattr(args, "exchange", "bitmap"),
            "transport": ("nvlink-peer" if getattr(args, "transport", "peer") == "peer" and
                          getattr(args, "exchange", "bitmap") == "bitmap" else "nccl") if world > 1 else "none",
            "l2": "flushed between steps (256 MiB write); graph > L2"}


# ---------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1408_1605_b200 import bfs, inputs

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        return max_over_ranks_dist(x, world, dev)

    cfg = workload_config(args, world)
    scale = cfg["scale"]
    R, C = grid_of(args, world)
    n = 1 << scale
    M = inputs.num_tuples(scale)
    # this rank's slice of the tuple list, generated in HBM
    k0 = M * rank // world
    k1 = M * (rank + 1) // world
    torch.cuda.synchronize()
    barrier()
    t_gen = time.perf_counter()
    ds, dd = inputs.generate_device(scale, k0=k0, count=k1 - k0, device=dev)
    torch.cuda.synchronize()
    t_gen = max_over_ranks(time.perf_counter() - t_gen)
    stream = torch.cuda.current_stream(dev)
    # timed steps: the level loop runs as one CUDA graph (no phase events); the per-phase CUDA-event
    # times (roofline of the expansion kernel) come from a replay of the same roots afterwards
    opts = bfs.make_opts(edges_per_thread=args.E, phase_timing=False, stream=stream.cuda_stream,
                         exchange=args.exchange, peer_exchange=args.transport == "peer" and args.exchange == "bitmap")
    opts_phase = bfs.make_opts(edges_per_thread=args.E, phase_timing=True, stream=stream.cuda_stream,
                               exchange=args.exchange, peer_exchange=args.transport == "peer" and args.exchange == "bitmap")
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.tensor(list(bfs.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        comm = bfs.make_comm(rank, world, local_rank, loopback=False, nccl_id=bytes(uid.cpu().tolist()))
    else:
        comm = bfs.make_comm(0, 1, local_rank, loopback=True)
    torch.cuda.synchronize()
    barrier()
    t_build = time.perf_counter()
    g = bfs.Graph(ds, dd, n, R, C, comm=comm, opts=opts)  # returns after the graph is resident
    t_build = max_over_ranks(time.perf_counter() - t_build)
    del ds, dd
    torch.cuda.empty_cache()
    info = g.info
    # 64 timed roots + W warm-up roots: degree >= 1, distinct, root stream of seed 2
    roots = sample_roots_collective(n, 64 + args.warmup, g.degree)
    timed_roots = roots[:64]
    warm_roots = roots[64:] or roots[:1]
    parent = torch.empty(info.nout, dtype=torch.int64, device=dev)
    level = torch.empty(info.nout, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)

    for k in range(args.warmup):
        g.run(warm_roots[k % len(warm_roots)], parent, level)
    torch.cuda.synchronize()

    times, mcomps, launches, xbytes, xlists = [], [], 0, 0, 0
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            r = timed_roots[k % len(timed_roots)]
            flush.zero_()
            torch.cuda.synchronize()
            barrier()
            ev0.record(stream)
            st = g.run(r, parent, level)
            ev1.record(stream)
            torch.cuda.synchronize()
            barrier()
            t_ms = max_over_ranks(ev0.elapsed_time(ev1))
            times.append(t_ms)
            launches += st.kernel_launches
            xbytes += st.bytes_exchanged
            xlists += st.list_messages
            mcomps.append(g.mcomp())
    clocks = clk.summary()
    teps = [m / (t * 1e-3) for m, t in zip(mcomps, times)]
    value = hmean(teps) / 1e9

    # phase-timed replay of the same roots (host-driven level loop, CUDA events around every phase)
    exp_bytes, exp_ms, lvl_tot, replay_ms = 0.0, 0.0, 0, 0.0
    tail = {"finalize": 0.0, "resolve": 0.0}
    phase = {"expand_comm": 0.0, "scan": 0.0, "expand": 0.0, "parent": 0.0, "fold_comm": 0.0, "update": 0.0,
             "allreduce": 0.0}
    if not args.no_phase_timing:
        g.set_opts(opts_phase)
        for k in range(args.steps):
            r = timed_roots[k % len(timed_roots)]
            flush.zero_()
            torch.cuda.synchronize()
            barrier()
            ev0.record(stream)
            st = g.run(r, parent, level)
            ev1.record(stream)
            torch.cuda.synchronize()
            replay_ms += ev0.elapsed_time(ev1)
            tail["finalize"] += st.finalize_ms
            tail["resolve"] += st.resolve_ms
            recs = g.level_times()
            lvl_tot += len(recs)
            for rec in recs:
                for key in phase:
                    phase[key] += getattr(rec, key)
                # algorithmic bytes of one expansion launch: 4 B row entry per scanned edge +
                # 20 B per frontier column (list 4 + cumul 8 + row offset 8)
                exp_bytes += 4.0 * rec.edges + 20.0 * rec.frontier
                exp_ms += rec.expand
        g.set_opts(opts)

    # e2e: same metric through the C ABI with a HOST output buffer (D2H inside the timed region).
    # The result read back is the BFS tree (parent array, Graph500's output); levels are optional
    # in the API and not requested here.
    ph = torch.empty(info.nout, dtype=torch.int64).pin_memory()
    e2e_teps = []
    for k in range(args.steps):
        r = timed_roots[k % len(timed_roots)]
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        g.run(r, ph)  # returns after the host buffer is complete
        t_s = max_over_ranks(time.perf_counter() - t0)
        e2e_teps.append(mcomps[k % len(mcomps)] / t_s)
    e2e = hmean(e2e_teps) / 1e9

    peak, peak_kind = measured_peaks()
    per_rank_exp_ms = exp_ms  # phase times are per rank; expansion kernel of this rank
    achieved = (exp_bytes / 1e9) / (per_rank_exp_ms * 1e-3) if per_rank_exp_ms > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "expand_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    step_ms = sum(times) / len(times)
    g.close()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded Graph500-style Kronecker, graph seed 1, "
                                                     "root seed 2)",
        "config": cfg,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8,
                "d2h_bytes_per_step": int(info.nout) * 8 * world, "result": "parent array (int64 per vertex)"},
        "gpu_launches": int(launches),
        "exchange": {"mode": args.exchange, "bytes_per_step_rank0": xbytes / max(1, args.steps),
                     "list_messages_per_step_rank0": xlists / max(1, args.steps)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "kernel": "k_expand (frontier expansion, Alg.3)", "peak_kind": peak_kind,
                     "alg_bytes_per_step": exp_bytes / max(1, args.steps),
                     "kernel_ms_per_step": per_rank_exp_ms / max(1, args.steps),
                     "kernel_share_of_step": per_rank_exp_ms / replay_ms if replay_ms else None,
                     "timing": "CUDA events around every k_expand launch in a phase-timed replay of the K "
                               "timed roots (the timed steps run the level loop as one CUDA graph)"},
        "phase_ms_per_step": {**{k: v / max(1, args.steps) for k, v in phase.items()},
                              **{k: v / max(1, args.steps) for k, v in tail.items()}},
        "levels_per_step": lvl_tot / max(1, args.steps),
        "replay_ms_per_step": replay_ms / max(1, args.steps),
        "clocks": clocks,
        "graph": {"nverts": n, "tuples": M, "nnz_rank0": int(info.nnz_local), "build_s": t_build,
                  "device_bytes_rank0": int(info.device_bytes)},
        # Graph500 kernel 1 (§8(f) NEXT-3): tuple generation in HBM + partition/shuffle/CSC+CSR
        # build, wall clock, max over ranks
        "construction": {"generate_s": t_gen, "build_s": t_build,
                         "tuples_per_s": M / (t_gen + t_build) if t_gen + t_build > 0 else None},
    }
    if world == 1 and not args.no_cpu_baseline:
        ns = int(os.environ.get("BENCH_CPU_ROOTS", "4"))
        v, sample = oracle_sample(ns, 0)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=0)
    ap.add_argument("--E", type=int, default=4)
    ap.add_argument("--grid", default="", help="RxC override of the default grid (1x1, 1x2, 2x2, 2x4)")
    ap.add_argument("--exchange", default="bitmap", choices=["bitmap", "list", "auto"],
                    help="per-level message encoding (bitmap: CUDA-graph level loop; list/auto: host-sized)")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="N > 1: per-level exchanges over NVLink peer memory (opts.peer_exchange, default) "
                         "or NCCL collectives")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-phase-timing", action="store_true", help="(diagnostic) no per-phase events")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world == 1 and args.gpus > 1:
        print(json.dumps({"error": f"--gpus {args.gpus} needs torchrun with {args.gpus} ranks"}), flush=True)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
