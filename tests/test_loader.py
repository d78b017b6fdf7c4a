"""bfs_load_edges (NEXT-4, SNAP real-world graph ingestion): the C-ABI loader on
the CPU -- the SPEC's own examples, the committed SNAP-format fixture checked against an
independent line parser written here, text/binary round trips, and every error status."""
import os
import tempfile

import numpy as np
import pytest

from paper_1408_1605_b200 import _build, bfs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "snap_small.txt")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    _build.build_bfs()
    bfs.lib()


def write(tmp, name, data, mode="w"):
    p = os.path.join(tmp, name)
    with open(p, mode) as f:
        f.write(data)
    return p


def test_spec_examples():
    with tempfile.TemporaryDirectory() as t:
        # S:62 file "# comment\n0 1\n1 2\n" -> (0,1),(1,2), num_vertices from 3
        s, d, n = bfs.load_edges(write(t, "a.txt", "# comment\n0 1\n1 2\n"))
        assert s.tolist() == [0, 1] and d.tolist() == [1, 2] and n == 3
        # S:63 empty file -> 0 tuples
        s, d, n = bfs.load_edges(write(t, "e.txt", ""))
        assert s.size == 0 and d.size == 0 and n == 0
        # S:64 binary (0,1),(1,0), 32 bytes
        raw = np.array([0, 1, 1, 0], dtype="<u8").tobytes()
        assert len(raw) == 32
        s, d, n = bfs.load_edges(write(t, "b.bin", raw, "wb"), "binary-pairs")
        assert s.tolist() == [0, 1] and d.tolist() == [1, 0] and n == 2


def independent_parse(path):
    src, dst = [], []
    with open(path, newline="") as f:
        for line in f.read().split("\n"):
            line = line.strip()
            if not line or line[0] in "#%":
                continue
            a, b = line.split()[:2]
            src.append(int(a))
            dst.append(int(b))
    return np.array(src, np.uint64), np.array(dst, np.uint64)


def test_golden_snap_fixture():
    s, d, n = bfs.load_edges(GOLDEN)
    es, ed = independent_parse(GOLDEN)
    assert np.array_equal(s, es) and np.array_equal(d, ed)  # file order kept
    assert s.size == 368 and n == int(max(es.max(), ed.max())) + 1
    assert np.any(s == d)  # self-loops are kept (they count for m_comp)


@pytest.mark.parametrize("seed", [0, 1])
def test_text_binary_roundtrip(seed):
    rng = np.random.default_rng(seed)
    m = 5000
    a = rng.integers(0, 1 << 40, size=m, dtype=np.uint64)
    b = rng.integers(0, 1 << 20, size=m, dtype=np.uint64)
    with tempfile.TemporaryDirectory() as t:
        txt = "# header\n" + "".join(f"{x}\t{y}\t{k}\n" for k, (x, y) in enumerate(zip(a, b)))  # 3rd field ignored
        s, d, n = bfs.load_edges(write(t, "r.txt", txt))
        assert np.array_equal(s, a) and np.array_equal(d, b) and n == int(max(a.max(), b.max())) + 1
        raw = np.stack([a, b], 1).astype("<u8").tobytes()
        s2, d2, n2 = bfs.load_edges(write(t, "r.bin", raw, "wb"), "binary-pairs")
        assert np.array_equal(s2, a) and np.array_equal(d2, b) and n2 == n


def test_large_text_crosses_read_buffer():
    """Lines straddling the loader's 4 MiB read buffer are reassembled."""
    m = 400_000
    a = np.arange(m, dtype=np.uint64) * 7919 % 1_000_003
    b = (a * 31 + 5) % 1_000_003
    with tempfile.TemporaryDirectory() as t:
        s, d, _ = bfs.load_edges(write(t, "big.txt", "".join(f"{x} {y}\n" for x, y in zip(a, b))))
        assert np.array_equal(s, a) and np.array_equal(d, b)


def test_errors():
    L = bfs.lib()
    with tempfile.TemporaryDirectory() as t:
        with pytest.raises(bfs.BfsError) as e:
            bfs.load_edges(write(t, "m.txt", "# c\n0 1\n2 x\n"))
        assert e.value.status == bfs.BFS_EPARSE and "m.txt:3" in str(e.value)  # names the line
        with pytest.raises(bfs.BfsError) as e:
            bfs.load_edges(write(t, "one.txt", "0 1\n5\n"))
        assert e.value.status == bfs.BFS_EPARSE and ":2" in str(e.value)
        with pytest.raises(bfs.BfsError) as e:
            bfs.load_edges(write(t, "big.txt", f"0 {1 << 48}\n"))
        assert e.value.status == bfs.BFS_ERANGE  # S:61 id >= 2^48
        bfs.load_edges(write(t, "ok.txt", f"0 {(1 << 48) - 1}\n"))  # the largest supported id
        with pytest.raises(bfs.BfsError) as e:
            bfs.load_edges(write(t, "t.bin", b"\x00" * 20, "wb"), "binary-pairs")
        assert e.value.status == bfs.BFS_EPARSE
        with pytest.raises(bfs.BfsError) as e:
            bfs.load_edges(write(t, "r.bin", np.array([1 << 50, 0], "<u8").tobytes(), "wb"), "binary-pairs")
        assert e.value.status == bfs.BFS_ERANGE
        with pytest.raises(bfs.BfsError) as e:
            bfs.load_edges(os.path.join(t, "missing.txt"))
        assert e.value.status == bfs.BFS_EINVAL
        with pytest.raises(bfs.BfsError) as e:
            bfs.load_edges(GOLDEN, 7)
        assert e.value.status == bfs.BFS_EINVAL
    assert L.bfs_strerror(bfs.BFS_EPARSE) == b"edge-list parse error"
