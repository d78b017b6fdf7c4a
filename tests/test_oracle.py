"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

* brute force: Floyd-Warshall distances + definitional min parent on tiny graphs (every root);
* closed forms: path, cycle, star, complete, complete bipartite, grid, binary tree;
* library routine: scipy.sparse.csgraph BFS distances on Kronecker graphs;
* worked examples: tests/golden/worked_examples.json (SPEC.md / SURVEY.md citations inside);
* the Graph500 validator (V1-V6) with fault injection, and m_comp by direct count.
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_1408_1605_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")


# ---------------------------------------------------------------- brute-force helpers (tests only)
def floyd_warshall(n, tuples):
    INF = 10**9
    D = np.full((n, n), INF, dtype=np.int64)
    np.fill_diagonal(D, 0)
    A = np.zeros((n, n), dtype=bool)
    for a, b in tuples:
        if a != b:
            A[a, b] = A[b, a] = True
    D[A] = 1
    for k in range(n):
        D = np.minimum(D, D[:, k:k + 1] + D[k:k + 1, :])
    return D, A, INF


def brute(n, tuples, r):
    D, A, INF = floyd_warshall(n, tuples)
    level = np.where(D[r] >= INF, -1, D[r]).astype(np.int32)
    parent = np.full(n, -1, dtype=np.int64)
    for v in range(n):
        if level[v] > 0:
            cands = [u for u in range(n) if A[u, v] and level[u] == level[v] - 1]
            parent[v] = min(cands)
    parent[r] = r
    return level, parent


def run_oracle(n, tuples, r):
    t = np.asarray(tuples, dtype=np.uint64).reshape(-1, 2)
    g = oracle.Graph(n, t[:, 0], t[:, 1])
    level, parent = g.bfs(r)
    return level, parent, g.mcomp(level), g


def random_gnp(n, p, rng):
    tuples = [(a, b) for a in range(n) for b in range(n) if a < b and rng.random() < p]
    # sprinkle duplicates, reversed duplicates and self-loops: they must not change the result
    extra = []
    for (a, b) in tuples[: len(tuples) // 4]:
        extra.append((b, a))
    for v in rng.choice(n, size=max(1, n // 8), replace=False):
        extra.append((int(v), int(v)))
    allt = tuples + extra
    rng.shuffle(allt)
    return allt


# ---------------------------------------------------------------- brute force
@pytest.mark.parametrize("seed", range(6))
def test_oracle_vs_floyd_warshall_gnp(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 65))
    p = float(rng.choice([0.03, 0.08, 0.2, 0.5]))
    tuples = random_gnp(n, p, rng)
    if not tuples:
        tuples = [(0, 0)]
    for r in range(n):
        lv, pa, mc, _ = run_oracle(n, tuples, r)
        bl, bp = brute(n, tuples, r)
        np.testing.assert_array_equal(lv, bl)
        np.testing.assert_array_equal(pa, bp)
        assert mc == sum(1 for (a, b) in tuples if bl[a] >= 0)


@pytest.mark.parametrize("scale", [3, 4, 5, 6])
def test_oracle_vs_floyd_warshall_kronecker(scale):
    s, d = inputs.generate(scale)
    n = 1 << scale
    tuples = list(zip(s.tolist(), d.tolist()))
    for r in range(n):
        lv, pa, mc, _ = run_oracle(n, tuples, r)
        bl, bp = brute(n, tuples, r)
        np.testing.assert_array_equal(lv, bl)
        np.testing.assert_array_equal(pa, bp)
        assert mc == int(np.sum(bl[s.astype(np.int64)] >= 0))


# ---------------------------------------------------------------- closed forms
def test_path_closed_form():
    n = 37
    tuples = [(i, i + 1) for i in range(n - 1)]
    for r in (0, 5, 36):
        lv, pa, _, _ = run_oracle(n, tuples, r)
        v = np.arange(n)
        np.testing.assert_array_equal(lv, np.abs(v - r))
        exp = np.where(v < r, v + 1, v - 1)
        exp[r] = r
        np.testing.assert_array_equal(pa, exp)


@pytest.mark.parametrize("n", [10, 11])
def test_cycle_closed_form(n):
    tuples = [(i, (i + 1) % n) for i in range(n)]
    r = 3
    lv, pa, _, _ = run_oracle(n, tuples, r)
    for v in range(n):
        dist = min(abs(v - r), n - abs(v - r))
        assert lv[v] == dist
        if v == r:
            assert pa[v] == r
        else:
            nb = [(v - 1) % n, (v + 1) % n]
            assert pa[v] == min(u for u in nb if min(abs(u - r), n - abs(u - r)) == dist - 1)
    if n % 2 == 0:  # antipode has both neighbours one level up -> the smaller one
        anti = (r + n // 2) % n
        assert pa[anti] == min((anti - 1) % n, (anti + 1) % n)


def test_star_and_complete():
    n = 20
    star = [(0, i) for i in range(1, n)]
    lv, pa, _, _ = run_oracle(n, star, 0)
    assert lv[0] == 0 and (lv[1:] == 1).all() and (pa == 0).all()
    lv, pa, _, _ = run_oracle(n, star, 7)  # leaf root: centre at 1, other leaves at 2 via centre
    assert lv[7] == 0 and lv[0] == 1 and pa[0] == 7
    others = [i for i in range(1, n) if i != 7]
    assert (lv[others] == 2).all() and (pa[others] == 0).all()
    kn = [(a, b) for a in range(n) for b in range(a + 1, n)]
    lv, pa, _, _ = run_oracle(n, kn, 13)
    assert (pa == 13).all() and lv[13] == 0 and (np.delete(lv, 13) == 1).all()


def test_complete_bipartite():
    a, b = 5, 7  # parts {0..4}, {5..11}
    tuples = [(i, a + j) for i in range(a) for j in range(b)]
    lv, pa, _, _ = run_oracle(a + b, tuples, 2)
    assert list(lv[:a]) == [2, 2, 0, 2, 2] and (lv[a:] == 1).all()
    assert (pa[a:] == 2).all()
    assert pa[0] == a and pa[1] == a and pa[3] == a and pa[4] == a  # smallest vertex of the other side


def test_grid_graph_manhattan():
    R, C = 6, 9
    vid = lambda i, j: i * C + j
    tuples = []
    for i in range(R):
        for j in range(C):
            if i + 1 < R:
                tuples.append((vid(i, j), vid(i + 1, j)))
            if j + 1 < C:
                tuples.append((vid(i, j), vid(i, j + 1)))
    ri, rj = 2, 4
    lv, pa, _, _ = run_oracle(R * C, tuples, vid(ri, rj))
    for i in range(R):
        for j in range(C):
            assert lv[vid(i, j)] == abs(i - ri) + abs(j - rj)
            if (i, j) != (ri, rj):
                nb = [(i + di, j + dj) for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1))
                      if 0 <= i + di < R and 0 <= j + dj < C]
                up = [vid(x, y) for x, y in nb if abs(x - ri) + abs(y - rj) == lv[vid(i, j)] - 1]
                assert pa[vid(i, j)] == min(up)


def test_binary_tree():
    n = 127
    tuples = [(v, (v - 1) // 2) for v in range(1, n)]
    lv, pa, _, _ = run_oracle(n, tuples, 0)
    v = np.arange(n)
    np.testing.assert_array_equal(lv, np.floor(np.log2(v + 1)).astype(int))
    exp = (v - 1) // 2
    exp[0] = 0
    np.testing.assert_array_equal(pa, exp)


# ---------------------------------------------------------------- worked examples (golden)
def _golden():
    with open(GOLDEN) as f:
        return json.load(f)["examples"]


@pytest.mark.parametrize("ex", _golden(), ids=lambda e: e["name"])
def test_worked_examples(ex):
    lv, pa, mc, _ = run_oracle(ex["n"], ex["tuples"], ex["root"])
    assert lv.tolist() == ex["level"]
    assert pa.tolist() == ex["parent"]
    assert mc == ex["m_comp"]
    t = np.asarray(ex["tuples"], dtype=np.uint64)
    assert oracle.validate(ex["n"], t[:, 0], t[:, 1], ex["root"], lv, pa) == 0


# ---------------------------------------------------------------- library routine (scipy)
@pytest.mark.parametrize("scale", [10, 12])
def test_oracle_vs_scipy_kronecker(scale):
    sp = pytest.importorskip("scipy.sparse")
    csgraph = pytest.importorskip("scipy.sparse.csgraph")
    s, d = inputs.generate(scale)
    n = 1 << scale
    keep = s != d
    A = sp.coo_matrix((np.ones(int(keep.sum())), (s[keep].astype(np.int64), d[keep].astype(np.int64))),
                      shape=(n, n)).tocsr()
    A = ((A + A.T) > 0).astype(np.int8).tocsr()
    g = oracle.Graph(n, s, d)
    elig = inputs.nonisolated_mask(n, s, d)
    roots = inputs.sample_roots(n, 8, elig)
    dist = csgraph.shortest_path(A, unweighted=True, indices=roots)
    for ri, r in enumerate(roots):
        lv, pa = g.bfs(r)
        exp = np.where(np.isinf(dist[ri]), -1, dist[ri]).astype(np.int32)
        np.testing.assert_array_equal(lv, exp)
        # parents: min over the scipy adjacency row of neighbours one level up
        for v in np.flatnonzero(lv > 0)[:: max(1, n // 400)]:
            nb = A.indices[A.indptr[v]:A.indptr[v + 1]]
            assert pa[v] == nb[lv[nb] == lv[v] - 1].min()
        assert pa[r] == r and (pa[lv < 0] == -1).all()
        assert g.mcomp(lv) == int(np.sum(exp[s.astype(np.int64)] >= 0))


# ---------------------------------------------------------------- validator with fault injection
def _kron_case(scale=9):
    s, d = inputs.generate(scale)
    n = 1 << scale
    g = oracle.Graph(n, s, d)
    r = inputs.sample_roots(n, 1, inputs.nonisolated_mask(n, s, d))[0]
    lv, pa = g.bfs(r)
    return n, s, d, r, lv, pa


def test_validator_accepts_oracle():
    n, s, d, r, lv, pa = _kron_case()
    assert oracle.validate(n, s, d, r, lv, pa) == 0


def _fault_cases():
    """(label, level, parent, check) for each invariant: check(mask) says what must fail."""
    n, s, d, r, lv, pa = _kron_case()
    bit = lambda name: 1 << oracle.V_NAMES.index(name)
    cases = []
    # V1: root parent wrong
    p2 = pa.copy(); p2[r] = (r + 1) % n
    cases.append(("V1", lv, p2, lambda m: m & bit("V1 root")))
    # V6: a non-minimal but valid parent (pick a vertex with >= 2 candidates): ONLY V6 fails
    keep = s != d
    a = np.concatenate([s[keep], d[keep]]).astype(np.int64)
    b = np.concatenate([d[keep], s[keep]]).astype(np.int64)
    up = (lv[a] >= 0) & (lv[b] == lv[a] + 1)
    cand_a, cand_b = a[up], b[up]
    for v in np.unique(cand_b):
        cs = np.unique(cand_a[cand_b == v])
        if cs.size >= 2:
            p3 = pa.copy(); p3[v] = cs[-1]
            cases.append(("V6", lv, p3, lambda m: m == bit("V6 min-rule")))
            break
    else:
        raise AssertionError("no vertex with two candidate parents")
    # V3: level off by one on a leaf-ish reached vertex
    v = int(np.flatnonzero(lv == lv.max())[0])
    l3 = lv.copy(); l3[v] += 1
    cases.append(("V3", l3, pa, lambda m: m & bit("V3 level+1")))
    # V2: parent that is not a neighbour but sits one level up: ONLY V2 fails
    # (a level-1 non-neighbour BELOW the true minimum parent, so the min rule V6 still holds)
    l1 = np.flatnonzero(lv == 1)
    v = max(np.flatnonzero(lv == 2).tolist(), key=lambda x: pa[x])
    nbrs = set(b[a == v].tolist())
    fake = [u for u in l1 if u not in nbrs and u < pa[v]]
    p4 = pa.copy(); p4[v] = fake[0]
    cases.append(("V2", lv, p4, lambda m: m == bit("V2 tree-edge")))
    # V5 alone (1): an unreached vertex whose parent is not -1 -- no other invariant looks at it
    v = int(np.flatnonzero(lv < 0)[0])
    p5 = pa.copy(); p5[v] = r
    cases.append(("V5-unreached", lv, p5, lambda m: m == bit("V5 component")))
    # V5 alone (2): a reached vertex whose parent id is out of range
    v = int(np.flatnonzero(lv == 1)[0])
    p5b = pa.copy(); p5b[v] = n
    cases.append(("V5-range", lv, p5b, lambda m: m == bit("V5 component")))
    # dropping a reached vertex breaks the component (V5) and the edge span (V4) together: the
    # component half of V5 alone cannot fail (V1-V4 imply it: V4 closes the reached set under
    # tuples, V1-V3 connect it to the root), so it is pinned together with V4
    v = int(np.flatnonzero(lv == lv.max())[0])
    l5 = lv.copy(); p5c = pa.copy(); l5[v] = -1; p5c[v] = -1
    cases.append(("V5+V4", l5, p5c, lambda m: (m & bit("V5 component")) and (m & bit("V4 edge-span"))))
    # V4: a tuple spanning two levels
    l6 = lv.copy()
    v = int(np.flatnonzero(lv == 1)[0])
    l6[v] = 3
    cases.append(("V4", l6, pa, lambda m: m & bit("V4 edge-span")))
    return n, s, d, r, cases


def test_validator_fault_injection():
    n, s, d, r, cases = _fault_cases()
    for label, lv, pa, check in cases:
        m = oracle.validate(n, s, d, r, lv, pa)
        assert check(m), (label, oracle.failed_names(m))


@pytest.mark.parametrize("chunk", [7, 1000, None])
def test_stream_validator_matches_oneshot(chunk):
    """The streaming validator (oracle.c step 6, written separately) gives the same mask as
    oracle_validate on every fault case and on valid trees, for any chunking of the tuples."""
    n, s, d, r, cases = _fault_cases()
    m_all = s.size
    step = chunk or m_all
    for label, lv, pa, check in cases + [("valid", *_kron_case()[4:], lambda m: m == 0)]:
        one = oracle.validate(n, s, d, r, lv, pa)
        assert check(one), label
        mask, mc = oracle.validate_stream(n, r, lv, pa, ((s[k:k + step], d[k:k + step]) for k in range(0, m_all, step)))
        assert mask == one, (label, oracle.failed_names(mask), oracle.failed_names(one))
        if not mask & (1 << oracle.V_NAMES.index("V5 component")):  # else parent[] is unusable: no pass
            assert mc == int(np.count_nonzero(lv[s] >= 0))


@pytest.mark.parametrize("scale", [10, 13, 16])
def test_stream_validator_regenerated_chunks(scale):
    """Chunks regenerated from the seed (what the full-size GPU checks do) validate the oracle's
    own trees, and m_comp matches the oracle's count."""
    s, d = inputs.generate(scale)
    n = 1 << scale
    g = oracle.Graph(n, s, d)
    M = inputs.num_tuples(scale)
    step = M // 5 + 3
    for r in inputs.sample_roots(n, 3, inputs.nonisolated_mask(n, s, d)):
        lv, pa = g.bfs(r)
        chunks = (inputs.generate(scale, k0=k, count=min(step, M - k)) for k in range(0, M, step))
        mask, mc = oracle.validate_stream(n, r, lv, pa, chunks)
        assert mask == 0, oracle.failed_names(mask)
        assert mc == g.mcomp(lv)


def test_isolated_and_out_of_range_root():
    g = oracle.Graph(8, [0, 1], [1, 2])
    lv, pa = g.bfs(5)
    assert lv.tolist() == [-1] * 5 + [0] + [-1] * 2
    with pytest.raises(IndexError):
        g.bfs(8)
    with pytest.raises(ValueError):
        oracle.Graph(4, [0, 9], [1, 2])


def test_empty_graph():
    g = oracle.Graph(4, np.zeros(0, np.uint64), np.zeros(0, np.uint64))
    lv, pa = g.bfs(0)
    assert lv.tolist() == [0, -1, -1, -1] and pa.tolist() == [0, -1, -1, -1]
    assert g.mcomp(lv) == 0
