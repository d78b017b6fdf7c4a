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
steps (and the graph is > L2).  --impl reference times the CPU oracle (as it stands) on the
same graph: one root per step, the roots spread over the host cores (one process each).
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
# The oracle (oracle/oracle.c, serial) timed as it stands on the host cores: its adjacency is
# built once (untimed, like GPU graph construction), then roots run one per process on separate
# cores (forked workers share the adjacency copy-on-write); per root TEPS = m_comp / t with t the
# BFS + min-parent pass (oracle steps 2-3), m_comp counted outside the timed region.
_OG = None


def _oracle_root(r):
    t0 = time.perf_counter()
    lv, _ = _OG.bfs(r)
    t = time.perf_counter() - t0
    return r, t, _OG.mcomp(lv)


def cpu_info():
    cores = len(os.sched_getaffinity(0))
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return cores, model


class OracleLeg:
    """Build the scale-S oracle adjacency (untimed), then time roots spread over the host cores."""

    def __init__(self, scale: int, gen_threads: int = 0):
        global _OG
        import oracle
        from paper_1408_1605_b200 import inputs
        self.scale, self.n = scale, 1 << scale
        t0 = time.perf_counter()
        if gen_threads:
            os.environ["OMP_NUM_THREADS"] = str(gen_threads)
        self.src, self.dst = inputs.generate(scale)
        self.g = oracle.Graph(self.n, self.src, self.dst)
        _OG = self.g
        self.build_s = time.perf_counter() - t0

    def roots(self, count):
        from paper_1408_1605_b200 import inputs
        return inputs.sample_roots(self.n, count, lambda v: self.g.degree(v) > 0)

    def run(self, roots, procs):
        import multiprocessing as mp
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_oracle_root, roots, chunksize=1)
        return res, time.perf_counter() - t0


def oracle_measure(scale: int, timed: int, warm: int = 0, gen_threads: int = 0):
    """Harmonic-mean GTEPS of the oracle over `timed` roots of the scale-`scale` graph (the
    first `timed` roots of the bench's root stream; `warm` further roots run alongside, untimed)."""
    cores, model = cpu_info()
    leg = OracleLeg(scale, gen_threads)
    roots = leg.roots(timed + warm)
    procs = max(1, min(cores, len(roots)))
    res, wall = leg.run(roots, procs)
    res = res[:timed]
    teps = [mc / t for _, t, mc in res]
    per_root_s = [t for _, t, _ in res]
    return {"value": hmean(teps) / 1e9, "unit": UNIT, "cores": procs, "cores_available": cores, "cpu_model": model,
            "kind": "oracle",
            "sample": (f"oracle BFS + min-parent pass (oracle/oracle.c steps 2-3), Graph500 Kronecker scale {scale} "
                       f"ef16 (graph seed 1), {timed} timed roots of root seed 2 (+{warm} untimed), one root per "
                       f"process on {procs} of {cores} host cores, adjacency built once untimed "
                       f"({leg.build_s:.0f} s)"),
            "per_root_s": {"min": min(per_root_s), "max": max(per_root_s)},
            "aggregate_gteps": sum(mc for _, _, mc in res) / wall / 1e9 if len(res) == len(roots) else None,
            "wall_s": wall}


def cpu_leg_main(args):
    """Subprocess body of the cpu_baseline leg: build, print 'ready', wait for 'go' on stdin (the
    GPU arm's timed regions are over), time the roots, print the result as one JSON line."""
    cores, _ = cpu_info()
    leg = OracleLeg(args.scale, gen_threads=4)
    roots = leg.roots(args.cpu_roots)
    print("ready", flush=True)
    sys.stdin.readline()
    procs = max(1, min(cores, len(roots)))
    res, wall = leg.run(roots, procs)
    teps = [mc / t for _, t, mc in res]
    _, model = cpu_info()
    print(json.dumps({"value": hmean(teps) / 1e9, "unit": UNIT, "cores": procs, "cores_available": cores,
                      "cpu_model": model, "kind": "oracle",
                      "sample": (f"oracle BFS + min-parent pass (oracle/oracle.c steps 2-3), Graph500 Kronecker "
                                 f"scale {args.scale} ef16 (graph seed 1; the bench graph), the first {len(roots)} "
                                 f"roots of root seed 2, one root per process on {procs} of {cores} host cores "
                                 f"(forked workers sharing the adjacency, built once untimed in {leg.build_s:.0f} s)"),
                      "per_root_s": {"min": min(r[1] for r in res), "max": max(r[1] for r in res)},
                      "aggregate_gteps": sum(r[2] for r in res) / wall / 1e9, "wall_s": wall}), flush=True)


def cpu_leg_start(scale: int, roots: int):
    """Start the oracle leg in a subprocess: its untimed adjacency build overlaps the GPU work."""
    return subprocess.Popen([sys.executable, os.path.abspath(__file__), "--cpu-leg", "--scale", str(scale),
                             "--cpu-roots", str(roots)], stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True)


def cpu_leg_finish(proc):
    try:
        line = proc.stdout.readline()  # 'ready' (build done)
        if line.strip() != "ready":
            raise RuntimeError(f"oracle leg failed to build: {line!r}")
        proc.stdin.write("go\n")
        proc.stdin.flush()
        out = proc.stdout.readline()
        proc.wait(timeout=60)
        return json.loads(out)
    except Exception as e:  # reported, never fatal for the GPU line
        proc.kill()
        return {"value": None, "unit": UNIT, "kind": "oracle", "error": str(e)[:200]}


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = workload_config(args, world)
    steps = max(1, args.steps)
    cb = oracle_measure(cfg["scale"], steps, max(0, args.warmup))
    cfg = dict(cfg, roots=steps)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world,
            "steps": steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (seeded Graph500-style Kronecker, graph seed 1, root seed 2)",
            "config": cfg, "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
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
    # cpu_baseline (rank 0, N = 1): the oracle leg's untimed adjacency build overlaps the GPU work;
    # its roots run after the GPU's timed regions
    cpu_proc = None
    if world == 1 and not args.no_cpu_baseline:
        cpu_proc = cpu_leg_start(scale, min(16, cpu_info()[0]))
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
    cfg["roots"] = min(args.steps, len(timed_roots))  # distinct roots actually timed
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
    # Algorithmic bytes of level L: B_L = 4 E_L + 40 F_L -- a 4-B `row` entry per
    # scanned edge, and per frontier column 16 B of `col` offsets + 24 B of frontier list / scan
    # entries written and read.
    def alg_bytes(rec):
        return 4.0 * rec.edges + 40.0 * rec.frontier

    exp_bytes, exp_ms, lvl_tot, replay_ms = 0.0, 0.0, 0, 0.0
    pk = {"bytes": 0.0, "k1_ms": 0.0, "level_ms": 0.0, "edges": 0}
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
                exp_bytes += alg_bytes(rec)
                exp_ms += rec.expand
            top = max(recs, key=lambda x: x.edges)  # the peak level of this root
            pk["bytes"] += alg_bytes(top)
            pk["k1_ms"] += top.expand
            pk["level_ms"] += top.scan + top.expand + top.parent + top.update
            pk["edges"] += top.edges
        g.set_opts(opts)

    # NVLink (N > 1): peer bandwidth measured in-run at the per-level message size (one bitmap
    # segment, block/8 bytes, to every other rank: all-to-all over the world), against the bytes
    # the per-level exchanges move (bfs_stats.bytes_exchanged)
    nvl = None
    if world > 1:
        msg = int(info.block) // 8
        a2a_in = torch.zeros(world * msg, dtype=torch.uint8, device=dev)
        a2a_out = torch.empty_like(a2a_in)
        for _ in range(3):
            dist.all_to_all_single(a2a_out, a2a_in)
        torch.cuda.synchronize()
        barrier()
        ev0.record(stream)
        reps = 10
        for _ in range(reps):
            dist.all_to_all_single(a2a_out, a2a_in)
        ev1.record(stream)
        torch.cuda.synchronize()
        t_a2a = max_over_ranks(ev0.elapsed_time(ev1) / reps)
        bw_nvl = (world - 1) * msg / (t_a2a * 1e-3) / 1e9  # GB/s sent per GPU
        b_nvl = xbytes / max(1, args.steps) / max(1, int(info.nlocal))
        step_s = sum(times) / len(times) * 1e-3
        nvl = {"bw_measured_gbs": bw_nvl, "msg_bytes": msg, "how": "torch.distributed all_to_all_single (NCCL), "
               "block/8 bytes per peer, 10 reps after 3 warm-up, max over ranks",
               "bytes_per_step_per_gpu": b_nvl, "achieved_gbs": b_nvl / step_s / 1e9,
               "frac": (b_nvl / step_s / 1e9) / bw_nvl if bw_nvl else None,
               "roofline_ms_per_step": b_nvl / (bw_nvl * 1e9) * 1e3 if bw_nvl else None,
               "note": "per-level fold/expand bitmaps only (the end-of-search resolution is excluded); the "
                       "exchange is fused into K4/K2 as NVLink peer stores, so it overlaps the kernels"}
        del a2a_in, a2a_out

    # e2e: same metric through the C ABI with HOST output buffers (D2H inside the timed region).
    # The result read back is the BFS tree (parent array, Graph500's output); levels are optional
    # in the API and not requested here.  Headline: the K timed roots in one bfs_run_batch call
    # (root k's copy to pinned host memory overlaps root k+1's search; two host buffers in turn),
    # value = sum of m_comp / wall time of the call, max over ranks.  Also reported: one bfs_run
    # per root (search, then copy; L2 flushed before each), harmonic mean.
    ph = [torch.empty(info.nout, dtype=torch.int64).pin_memory() for _ in range(2)]
    e2e_teps = []
    for k in range(args.steps):
        r = timed_roots[k % len(timed_roots)]
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        g.run(r, ph[0])  # returns after the host buffer is complete
        t_s = max_over_ranks(time.perf_counter() - t0)
        e2e_teps.append(mcomps[k % len(mcomps)] / t_s)
    e2e_sync = hmean(e2e_teps) / 1e9
    batch_roots = [timed_roots[k % len(timed_roots)] for k in range(args.steps)]
    g.run_batch(batch_roots[:2], [ph[0], ph[1]])  # first batch: staging buffers and copy stream
    flush.zero_()
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    g.run_batch(batch_roots, [ph[k % 2] for k in range(args.steps)])
    t_b = max_over_ranks(time.perf_counter() - t0)
    e2e = sum(mcomps[k % len(mcomps)] for k in range(args.steps)) / t_b / 1e9

    peak, peak_kind = measured_peaks()
    per_rank_exp_ms = exp_ms  # phase times are per rank; expansion kernel of this rank
    achieved = (exp_bytes / 1e9) / (per_rank_exp_ms * 1e-3) if per_rank_exp_ms > 0 else 0.0
    peak_levels = None
    if pk["k1_ms"] > 0:
        a_k1 = pk["bytes"] / 1e9 / (pk["k1_ms"] * 1e-3)
        a_lv = pk["bytes"] / 1e9 / (pk["level_ms"] * 1e-3)
        peak_levels = {"alg_bytes_per_step": pk["bytes"] / args.steps, "edges_per_step": pk["edges"] / args.steps,
                       "k1_ms_per_step": pk["k1_ms"] / args.steps, "level_ms_per_step": pk["level_ms"] / args.steps,
                       "k1_gbs": a_k1, "k1_frac": a_k1 / peak, "level_gbs": a_lv, "level_frac": a_lv / peak,
                       "definition": "per root the level with the most scanned edges; B_L = 4 E_L + 40 F_L; "
                                     "k1 = k_expand time, level = K3 scan + K1 expand + K4 parent + K2 update"}
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
                "d2h_bytes_per_step": int(info.nout) * 8 * world, "result": "parent array (int64 per vertex)",
                "how": "bfs_run_batch over the K timed roots into pinned host memory (root k's D2H overlaps "
                       "root k+1's search), sum m_comp / wall time of the call, max over ranks",
                "per_call_value": e2e_sync,
                "per_call_how": "one bfs_run per root (search then D2H), L2 flushed before each, harmonic mean"},
        "gpu_launches": int(launches),
        "exchange": {"mode": args.exchange, "bytes_per_step_rank0": xbytes / max(1, args.steps),
                     "list_messages_per_step_rank0": xlists / max(1, args.steps)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": None,
                     "traffic_note": "not measured in-run (needs ncu); the ncu capture of this config's peak "
                                     "k_expand launch is in profiles/ (DRAM vs algorithmic bytes)",
                     "kernel": "k_expand (frontier expansion, Alg.3)", "peak_kind": peak_kind,
                     "alg_bytes_per_step": exp_bytes / max(1, args.steps),
                     "alg_bytes_definition": "sum over levels of 4 E_L + 40 F_L (SURVEY.md §8(d))",
                     "kernel_ms_per_step": per_rank_exp_ms / max(1, args.steps),
                     "kernel_share_of_step": per_rank_exp_ms / replay_ms if replay_ms else None,
                     "peak_levels": peak_levels,
                     "timing": "CUDA events around every k_expand launch in a phase-timed replay of the K "
                               "timed roots (the timed steps run the level loop as one CUDA graph); rank 0"},
        "nvlink": nvl,
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
    if world == 1 and cpu_proc is not None:
        line["cpu_baseline"] = cpu_leg_finish(cpu_proc)
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
    ap.add_argument("--cpu-leg", action="store_true", help=argparse.SUPPRESS)  # cpu_baseline subprocess
    ap.add_argument("--cpu-roots", type=int, default=16, help=argparse.SUPPRESS)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world == 1 and args.gpus > 1:
        print(json.dumps({"error": f"--gpus {args.gpus} needs torchrun with {args.gpus} ranks"}), flush=True)
        sys.exit(2)
    if args.cpu_leg:
        cpu_leg_main(args)
        return
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
