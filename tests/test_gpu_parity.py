"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

level[] and parent[] must be bit-identical (integer path; parent = minimum-id neighbour one
level up, R1).  Grids other than 1x1 run on one GPU with the loopback transport
(R*C logical ranks, same kernels).  Full-size (s26, the bench launch configuration) outputs are
checked with the Graph500 invariants V1-V6, which hold at any size and together are equivalent
to bit-exact equality with the oracle.
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_1408_1605_b200 import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


@pytest.fixture(scope="module")
def bfs():
    _need_gpu()
    from paper_1408_1605_b200 import _build, bfs as b
    _build.build_all()
    return b


def make_graph(bfs, s, d, n, R=1, C=1, E=4, on_device=True):
    if on_device:
        ts = torch.from_numpy(np.ascontiguousarray(s, dtype=np.uint64).view(np.int64)).cuda()
        td = torch.from_numpy(np.ascontiguousarray(d, dtype=np.uint64).view(np.int64)).cuda()
    else:
        ts = np.ascontiguousarray(s, dtype=np.uint64)
        td = np.ascontiguousarray(d, dtype=np.uint64)
    return bfs.Graph(ts, td, n, R, C, comm=bfs.make_comm(loopback=True, device=0),
                     opts=bfs.make_opts(edges_per_thread=E))


def check_root(g, og, r, n):
    lv, pa = g.bfs(r)
    ol, op = og.bfs(r)
    assert np.array_equal(lv[:n], ol), f"level mismatch root {r}: {np.flatnonzero(lv[:n] != ol)[:10]}"
    assert np.array_equal(pa[:n], op), f"parent mismatch root {r}: {np.flatnonzero(pa[:n] != op)[:10]}"
    assert (lv[n:] == -1).all() and (pa[n:] == -1).all()  # padding vertices never reached
    assert g.mcomp() == og.mcomp(ol)


# ---------------------------------------------------------------- worked examples
def _golden():
    with open(GOLDEN) as f:
        return json.load(f)["examples"]


@pytest.mark.parametrize("ex", _golden(), ids=lambda e: e["name"])
@pytest.mark.parametrize("grid", [(1, 1), "own", (2, 2), (1, 4), (4, 1)])
def test_worked_examples(bfs, ex, grid):
    R, C = tuple(ex["grid"]) if grid == "own" else grid
    t = np.asarray(ex["tuples"], dtype=np.uint64).reshape(-1, 2)
    g = make_graph(bfs, t[:, 0], t[:, 1], ex["n"], R, C)
    lv, pa = g.bfs(ex["root"])
    n = ex["n"]
    assert lv[:n].tolist() == ex["level"]
    assert pa[:n].tolist() == ex["parent"]
    assert g.mcomp() == ex["m_comp"]


# ---------------------------------------------------------------- Kronecker graphs vs oracle
@pytest.mark.parametrize("grid", [(1, 1), (1, 2), (2, 1), (2, 2), (2, 4), (4, 2), (4, 4)])
def test_kron_s10_all_grids(bfs, grid):
    scale = 10
    s, d = inputs.generate(scale)
    n = 1 << scale
    og = oracle.Graph(n, s, d)
    g = make_graph(bfs, s, d, n, *grid)
    elig = inputs.nonisolated_mask(n, s, d)
    roots = inputs.sample_roots(n, 64 if grid == (1, 1) else 16, elig)
    for r in roots:
        check_root(g, og, r, n)


def test_kron_s10_every_root_1x1(bfs):
    scale = 10
    s, d = inputs.generate(scale)
    n = 1 << scale
    og = oracle.Graph(n, s, d)
    g = make_graph(bfs, s, d, n)
    for r in range(n):  # includes isolated roots (only r visited)
        check_root(g, og, r, n)


@pytest.mark.parametrize("E", [1, 2, 4, 8, 16])
def test_edges_per_thread_invariance(bfs, E):
    scale = 14
    s, d = inputs.generate(scale)
    n = 1 << scale
    og = oracle.Graph(n, s, d)
    g = make_graph(bfs, s, d, n, E=E)
    for r in inputs.sample_roots(n, 8, inputs.nonisolated_mask(n, s, d)):
        check_root(g, og, r, n)


@pytest.mark.parametrize("scale,nroots,grid", [(16, 64, (1, 1)), (20, 8, (1, 1)), (18, 8, (2, 4)), (18, 8, (4, 4))])
def test_kron_larger(bfs, scale, nroots, grid):
    s, d = inputs.generate(scale)
    n = 1 << scale
    og = oracle.Graph(n, s, d)
    g = make_graph(bfs, s, d, n, *grid)
    for r in inputs.sample_roots(n, nroots, inputs.nonisolated_mask(n, s, d)):
        check_root(g, og, r, n)


def test_host_buffers_and_host_edges(bfs):
    scale = 12
    s, d = inputs.generate(scale)
    n = 1 << scale
    og = oracle.Graph(n, s, d)
    g = make_graph(bfs, s, d, n, 2, 2, on_device=False)  # host edge arrays
    r = inputs.sample_roots(n, 1, inputs.nonisolated_mask(n, s, d))[0]
    ol, op = og.bfs(r)
    # device outputs
    pd = torch.empty(g.info.nout, dtype=torch.int64, device="cuda")
    ld = torch.empty(g.info.nout, dtype=torch.int32, device="cuda")
    g.run(r, pd, ld)
    assert np.array_equal(ld.cpu().numpy()[:n], ol) and np.array_equal(pd.cpu().numpy()[:n], op)
    # pinned host outputs
    ph = torch.empty(g.info.nout, dtype=torch.int64).pin_memory()
    lh = torch.empty(g.info.nout, dtype=torch.int32).pin_memory()
    g.run(r, ph, lh)
    assert np.array_equal(lh.numpy()[:n], ol) and np.array_equal(ph.numpy()[:n], op)


def test_degree_matches_oracle(bfs):
    scale = 11
    s, d = inputs.generate(scale)
    n = 1 << scale
    og = oracle.Graph(n, s, d)
    for grid in ((1, 1), (2, 4)):
        g = make_graph(bfs, s, d, n, *grid)
        keep = s != d
        a = np.concatenate([s[keep], d[keep]]).astype(np.int64)
        b = np.concatenate([d[keep], s[keep]]).astype(np.int64)
        uniq = np.unique(a * n + b)
        deg = np.bincount(uniq // n, minlength=n)
        for v in list(range(0, n, 97)) + [int(np.argmax(deg))]:
            assert g.degree(v) == deg[v]


# ---------------------------------------------------------------- list <-> bitmap exchange (NEXT-1)
@pytest.mark.parametrize("exchange", ["list", "auto"])
@pytest.mark.parametrize("grid", [(1, 2), (2, 1), (2, 2), (2, 4), (4, 2)])
def test_exchange_modes(bfs, exchange, grid):
    """Index-list and auto (P:874-897 threshold T = block/32) messages give the same outputs;
    byte counts follow the encoding."""
    scale = 12
    s, d = inputs.generate(scale)
    n = 1 << scale
    og = oracle.Graph(n, s, d)
    g = make_graph(bfs, s, d, n, *grid)
    roots = inputs.sample_roots(n, 6, inputs.nonisolated_mask(n, s, d))
    g.set_opts(bfs.make_opts(edges_per_thread=4))
    bitmap_bytes = g.run(roots[0]).bytes_exchanged
    g.set_opts(bfs.make_opts(edges_per_thread=4, exchange=exchange))
    for r in roots:
        check_root(g, og, r, n)
    st = g.run(roots[0])
    R, C = grid
    nmsg = st.nlevels * R * C * ((R - 1) + (C - 1))  # per-level messages of all ranks
    if exchange == "list":
        assert st.list_messages == nmsg
        # every list entry is one discovered/frontier vertex: at most 4 B per reached vertex per
        # receiving peer and level
        assert 0 < st.bytes_exchanged <= 4 * n * max(R, C) * st.nlevels
    else:
        assert 0 < st.list_messages < nmsg  # sparse levels as lists, the dense ones as bitmaps
        assert st.bytes_exchanged < bitmap_bytes


def test_exchange_threshold_rule(bfs):
    """a message is a list iff n <= T = L/32 words (L = block), strictly '>' for
    the bitmap.  A 2x1 grid (one column phase message per rank and level) on a star whose hub's
    frontier sizes are known exactly."""
    R, C = 2, 1
    nverts = 4096  # block = 2048 vertices, T = 64 words
    hub = 0
    # level 1 frontier on the owner of block 1: exactly 64 leaves there (list), then 65 (bitmap)
    for k, expect_list in ((64, True), (65, False)):
        leaves = np.arange(2048, 2048 + k, dtype=np.uint64)
        t = np.stack([np.full(k, hub, dtype=np.uint64), leaves], 1)
        og = oracle.Graph(nverts, t[:, 0], t[:, 1])
        g = make_graph(bfs, t[:, 0], t[:, 1], nverts, R, C)
        g.set_opts(bfs.make_opts(edges_per_thread=4, exchange="auto"))
        check_root(g, og, hub, nverts)
        st = g.run(hub)
        # one all-gather per level, 2 messages, both encoded by the larger count: frontier sizes
        # per level are 1 (the hub), k (the leaves), then 0
        f = [1, k] + [0] * st.nlevels
        assert st.list_messages == sum(2 for lv in range(st.nlevels) if f[lv] <= 64)
        assert (f[1] <= 64) == expect_list


def test_exchange_invalid(bfs):
    s = np.array([0], dtype=np.uint64)
    d = np.array([1], dtype=np.uint64)
    g = make_graph(bfs, s, d, 8)
    with pytest.raises(bfs.BfsError) as e:
        g.set_opts(bfs.make_opts(exchange=3))
    assert e.value.status == bfs.BFS_EINVAL


# ---------------------------------------------------------------- edge cases
def test_padding_and_tiny_graphs(bfs):
    # nverts not a multiple of 32*R*C; single vertex; no edges
    for n, tuples, root, grid in [(37, [(0, 36), (36, 5), (5, 6)], 0, (2, 2)), (1, [(0, 0)], 0, (1, 1)),
                                  (5, [], 3, (1, 2)), (100, [(i, i + 1) for i in range(99)], 50, (2, 4))]:
        t = np.asarray(tuples, dtype=np.uint64).reshape(-1, 2)
        og = oracle.Graph(n, t[:, 0], t[:, 1])
        g = make_graph(bfs, t[:, 0], t[:, 1], n, *grid)
        check_root(g, og, root, n)


def test_errors(bfs):
    s = np.array([0, 1], dtype=np.uint64)
    d = np.array([1, 9], dtype=np.uint64)
    with pytest.raises(bfs.BfsError) as e:
        make_graph(bfs, s, d, 8)
    assert e.value.status == bfs.BFS_ERANGE
    g = make_graph(bfs, s[:1], d[:1], 8)
    with pytest.raises(bfs.BfsError) as e:
        g.bfs(8)
    assert e.value.status == bfs.BFS_ERANGE
    with pytest.raises(bfs.BfsError):
        g.set_opts(bfs.make_opts(edges_per_thread=5))
    lv, pa = g.bfs(1)  # graph still usable after argument errors
    assert lv[:2].tolist() == [1, 0] and pa[:2].tolist() == [1, 1]


def test_repeat_determinism_and_phase_timing(bfs):
    scale = 16
    s, d = inputs.generate(scale)
    n = 1 << scale
    g = make_graph(bfs, s, d, n)
    g.set_opts(bfs.make_opts(edges_per_thread=4, phase_timing=True))
    r = inputs.sample_roots(n, 1, inputs.nonisolated_mask(n, s, d))[0]
    a = g.bfs(r)
    b = g.bfs(r)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    recs = g.level_times()
    assert len(recs) >= 3 and all(x.expand >= 0 for x in recs)
    st = g.run(r)
    assert st.edges_scanned == sum(x.edges for x in recs)


# ---------------------------------------------------------------- generator twins
def test_device_generator_matches_host(bfs):
    for scale, k0, cnt in ((10, 0, None), (16, 12345, 100000), (26, (16 << 26) - 5000, 5000)):
        hs, hd = inputs.generate(scale, k0=k0, count=cnt)
        ds, dd = inputs.generate_device(scale, k0=k0, count=cnt)
        torch.cuda.synchronize()
        assert np.array_equal(ds.cpu().view(torch.int64).numpy().view(np.uint64), hs)
        assert np.array_equal(dd.cpu().view(torch.int64).numpy().view(np.uint64), hd)


# ---------------------------------------------------------------- the kernel variants the bench runs
K_HOT_MIN_EDGES = 1 << 22  # kernels.cu kHotMinEdges: P2 levels below it skip the shared-memory hot copy


@pytest.mark.parametrize("scale,grid", [(22, (1, 2)), (23, (2, 2))])
def test_multi_column_hot_path(bfs, scale, grid):
    """C > 1 grids at sizes whose peak levels exceed kHotMinEdges per rank, so K1 runs the
    multi-segment hot-copy lookup (probe_segs) that the N > 1 bench configurations time; the
    first root runs the host-driven level loop, later roots the CUDA-graph loop.  Bit-exact
    level[] / parent[] / m_comp against the oracle."""
    s, d = inputs.generate(scale)
    n = 1 << scale
    og = oracle.Graph(n, s, d)
    g = make_graph(bfs, s, d, n, *grid)
    roots = inputs.sample_roots(n, 4, inputs.nonisolated_mask(n, s, d))
    for r in roots:
        check_root(g, og, r, n)
    # the per-rank peak level of this graph is above the hot-copy threshold (loopback level
    # records sum the R*C local ranks)
    g.set_opts(bfs.make_opts(edges_per_thread=4, phase_timing=True))
    g.run(roots[0])
    peak = max(x.edges for x in g.level_times())
    assert peak / (grid[0] * grid[1]) > 2 * K_HOT_MIN_EDGES, peak


@pytest.mark.parametrize("grid", [(1, 1), (1, 2), (2, 2)])
def test_pos64_variant(bfs, grid):
    """The 64-bit staged-position K1 variant (used when a rank holds >= 2^32 CSC entries),
    forced on a small graph with the test-only BFS_DEBUG_POS64 flag: bit-exact."""
    scale = 16
    s, d = inputs.generate(scale)
    n = 1 << scale
    og = oracle.Graph(n, s, d)
    g = make_graph(bfs, s, d, n, *grid)
    g.set_opts(bfs.make_opts(edges_per_thread=4, debug_flags=bfs.DEBUG_POS64))
    for r in inputs.sample_roots(n, 6, inputs.nonisolated_mask(n, s, d)):
        check_root(g, og, r, n)


def test_deeper_than_level_records(bfs):
    """A path of 5000 vertices: 5000 levels, more than the 4096 per-level records kept; the
    BFS runs to the end (graph loop and host loop) and stats cover every level."""
    n = 5000
    t = np.stack([np.arange(n - 1, dtype=np.uint64), np.arange(1, n, dtype=np.uint64)], 1)
    og = oracle.Graph(n, t[:, 0], t[:, 1])
    g = make_graph(bfs, t[:, 0], t[:, 1], n, 1, 2)
    for r in (0, 0, n - 1):  # first run host loop, then the CUDA-graph loop
        check_root(g, og, r, n)
    st = g.run(0)
    assert st.nlevels == n and st.edges_scanned == 2 * (n - 1)  # n - 1 discovering levels + the empty one
    g.set_opts(bfs.make_opts(edges_per_thread=4, phase_timing=True))
    check_root(g, og, 0, n)
    assert len(g.level_times(max_levels=8192)) == 4096


def test_gather_loopback(bfs):
    scale = 12
    s, d = inputs.generate(scale)
    n = 1 << scale
    g = make_graph(bfs, s, d, n, 2, 2)
    r = inputs.sample_roots(n, 1, inputs.nonisolated_mask(n, s, d))[0]
    lv, pa = g.bfs(r)
    la = np.full(g.info.npad, 7, dtype=np.int32)
    pad = torch.full((g.info.npad,), 7, dtype=torch.int64, device="cuda")
    g.gather(pa, lv, pad, la)
    assert np.array_equal(la, lv) and np.array_equal(pad.cpu().numpy(), pa)


# ---------------------------------------------------------------- real-world graph files (NEXT-4)
SNAP_GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "snap_small.txt")


@pytest.mark.parametrize("grid", [(1, 1), (2, 2), (1, 3)])
def test_snap_file_parity(bfs, grid):
    """A SNAP-format file (tests/golden/snap_small.txt: sparse ids, duplicates, self-loops, two
    components) through bfs_load_edges -> bfs_graph_create (nverts = max id + 1, padded): every
    vertex of the file as root, bit-exact against the oracle on the same tuples."""
    src, dst, n = bfs.load_edges(SNAP_GOLDEN)
    og = oracle.Graph(n, src, dst)
    g = make_graph(bfs, src, dst, n, *grid, on_device=False)
    for r in np.unique(np.concatenate([src, dst])).tolist() + [0, n - 1]:
        check_root(g, og, int(r), n)


def test_snap_kronecker_roundtrip(bfs, tmp_path):
    """The s14 Kronecker tuples written as a SNAP text file and as binary pairs, loaded back and
    searched: identical to the oracle on the generator's own tuples."""
    scale = 14
    s, d = inputs.generate(scale)
    n = 1 << scale
    txt = tmp_path / "kron.txt"
    with open(txt, "w") as f:
        f.write("# Directed graph: kron s14\n# FromNodeId\tToNodeId\n")
        f.write("".join(f"{a}\t{b}\n" for a, b in zip(s.tolist(), d.tolist())))
    binp = tmp_path / "kron.bin"
    binp.write_bytes(np.stack([s, d], 1).astype("<u8").tobytes())
    roots = inputs.sample_roots(n, 4, inputs.nonisolated_mask(n, s, d))
    for path, fmt in ((txt, "snap-text"), (binp, "binary-pairs")):
        ls, ld, nv = bfs.load_edges(str(path), fmt)
        assert np.array_equal(ls, s) and np.array_equal(ld, d) and nv == int(max(s.max(), d.max())) + 1
        og = oracle.Graph(nv, s, d)
        g = make_graph(bfs, ls, ld, nv, 2, 2)
        for r in roots:
            check_root(g, og, r, nv)
        g.close()


# ---------------------------------------------------------------- full size (bench config)
def test_s26_bench_config_graph500_valid(bfs):
    """s26 1x1 (configs[2], the bench workload): device-generated graph, bench launch options,
    three roots (the first runs the host-driven level loop, the others the CUDA-graph loop the
    bench times).  The oracle's streaming Graph500 validator regenerates the tuples from the
    seed chunk by chunk and checks V1-V6 (equivalent to bit-exact equality with the oracle,
    SURVEY.md §8(c)) and m_comp."""
    scale = 26
    n = 1 << scale
    M = inputs.num_tuples(scale)
    ds, dd = inputs.generate_device(scale)
    g = bfs.Graph(ds, dd, n, 1, 1, opts=bfs.make_opts(edges_per_thread=4))
    del ds, dd
    torch.cuda.empty_cache()
    roots = []
    t = 0
    while len(roots) < 3:
        v = inputs.root_candidate(inputs.ROOT_SEED, t, n)
        t += 1
        if v not in roots and g.degree(v) > 0:
            roots.append(v)
    step = 1 << 26
    for r in roots:
        lv, pa = g.bfs(r)
        mc = g.mcomp()
        chunks = (inputs.generate(scale, k0=k, count=min(step, M - k)) for k in range(0, M, step))
        mask, omc = oracle.validate_stream(n, r, lv[:n], pa[:n], chunks)
        assert mask == 0, oracle.failed_names(mask)
        assert mc == omc


def test_unaligned_device_outputs(bfs):
    """Device output buffers that are not 16-byte aligned take the staging path."""
    scale = 12
    s, d = inputs.generate(scale)
    n = 1 << scale
    og = oracle.Graph(n, s, d)
    g = make_graph(bfs, s, d, n)
    r = inputs.sample_roots(n, 1, inputs.nonisolated_mask(n, s, d))[0]
    ol, op = og.bfs(r)
    pbuf = torch.empty(g.info.nout + 1, dtype=torch.int64, device="cuda")
    lbuf = torch.empty(g.info.nout + 1, dtype=torch.int32, device="cuda")
    pd, ld = pbuf[1:], lbuf[1:]  # 8- and 4-byte offsets
    g.run(r, pd, ld)
    assert np.array_equal(ld.cpu().numpy()[:n], ol) and np.array_equal(pd.cpu().numpy()[:n], op)


@pytest.mark.parametrize("grid", [(1, 1), (2, 2)])
def test_run_batch(bfs, grid):
    """bfs_run_batch: every root's outputs equal the oracle's, for pinned and pageable host buffers
    (the copies of root k overlap root k+1's search), device buffers, a host buffer reused by
    several roots (it ends with the last one), a NULL entry, and per-root stats."""
    scale = 14
    s, d = inputs.generate(scale)
    n = 1 << scale
    og = oracle.Graph(n, s, d)
    g = make_graph(bfs, s, d, n, *grid)
    roots = [int(r) for r in inputs.sample_roots(n, 5, inputs.nonisolated_mask(n, s, d))]
    exp = [og.bfs(r) for r in roots]
    nout = g.info.nout
    pin = [torch.empty(nout, dtype=torch.int64).pin_memory() for _ in roots]
    lpin = [torch.empty(nout, dtype=torch.int32).pin_memory() for _ in roots]
    page = [np.empty(nout, dtype=np.int64) for _ in roots]
    dev = [torch.empty(nout, dtype=torch.int64, device="cuda") for _ in roots]
    for bufs, lbufs in ((pin, lpin), (page, None), (dev, None)):
        st = g.run_batch(roots, bufs, lbufs, want_stats=True)
        for k, (ol, op) in enumerate(exp):
            pa = bufs[k].cpu().numpy() if hasattr(bufs[k], "cpu") else bufs[k]
            assert np.array_equal(pa[:n], op), f"parent mismatch root {roots[k]}"
            assert (pa[n:] == -1).all()
            if lbufs is not None:
                assert np.array_equal(lbufs[k].numpy()[:n], ol), f"level mismatch root {roots[k]}"
            assert st[k].nlevels == int(ol.max()) + 1
    # one host buffer for every root: it holds the last root's tree; a NULL entry skips a root's output
    shared = torch.empty(nout, dtype=torch.int64).pin_memory()
    g.run_batch(roots, [shared] * len(roots))
    assert np.array_equal(shared.numpy()[:n], exp[-1][1])
    page2 = [np.full(nout, 7, dtype=np.int64) for _ in roots]
    bufs = list(page2)
    bufs[1] = None
    g.run_batch(roots, bufs)
    assert (page2[1] == 7).all() and np.array_equal(page2[2][:n], exp[2][1])
    # a single bfs_run after a batch still sees its own staging
    ph = torch.empty(nout, dtype=torch.int64).pin_memory()
    g.run(roots[0], ph)
    assert np.array_equal(ph.numpy()[:n], exp[0][1])
    with pytest.raises(bfs.BfsError) as e:
        g.run_batch([roots[0], 1 << 40])
    assert e.value.status == bfs.BFS_ERANGE
