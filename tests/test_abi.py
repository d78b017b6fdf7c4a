"""CPU checks of the C-ABI boundary: libbfs200.so loads, exports every function include/*.h
declares, and the ctypes mirrors of the structs have the C layout (no GPU compute calls)."""
import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from paper_1408_1605_b200 import _build, bfs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "bfs200.h")


@pytest.fixture(scope="module")
def L():
    _build.build_bfs()
    return bfs.lib()


def declared_functions():
    text = open(HDR).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bfs_[a-z_0-9]+)\s*\(", text)))


def test_exports_every_declared_symbol(L):
    names = declared_functions()
    assert "bfs_graph_create" in names and "bfs_run" in names and "bfs_destroy" in names
    for n in names:
        assert hasattr(L, n), f"{n} declared in bfs200.h but not exported"
    assert set(names) == set(bfs.EXPORTS)


def test_struct_layout_matches_header(L):
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "bfs200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu\n", sizeof(bfs_comm), sizeof(bfs_opts), sizeof(bfs_info), sizeof(bfs_stats),
         sizeof(bfs_level_record));
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", offsetof(bfs_info, nout), offsetof(bfs_stats, bytes_exchanged),
         offsetof(bfs_level_record, edges), offsetof(bfs_opts, exchange), offsetof(bfs_stats, list_messages),
         offsetof(bfs_stats, kernel_launches), offsetof(bfs_opts, peer_exchange), offsetof(bfs_opts, debug_flags));
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        exe = os.path.join(d, "t")
        open(c, "w").write(src)
        subprocess.check_call(["gcc", "-I", os.path.dirname(HDR), c, "-o", exe])
        out = subprocess.check_output([exe]).decode().split()
    sizes = [int(x) for x in out]
    assert sizes[:5] == [ctypes.sizeof(bfs.Comm), ctypes.sizeof(bfs.Opts), ctypes.sizeof(bfs.Info),
                         ctypes.sizeof(bfs.Stats), ctypes.sizeof(bfs.LevelRecord)]
    assert sizes[5:] == [bfs.Info.nout.offset, bfs.Stats.bytes_exchanged.offset, bfs.LevelRecord.edges.offset,
                         bfs.Opts.exchange.offset, bfs.Stats.list_messages.offset, bfs.Stats.kernel_launches.offset,
                         bfs.Opts.peer_exchange.offset, bfs.Opts.debug_flags.offset]


def test_strerror_and_null_args(L):
    assert L.bfs_strerror(0) == b"ok"
    assert L.bfs_strerror(-2) == b"vertex id out of range"
    # null graph handles are rejected before touching the GPU
    assert L.bfs_run(None, 0, None, None, None) == bfs.BFS_EINVAL
    assert L.bfs_run_batch(None, None, 0, None, None, None) == bfs.BFS_EINVAL
    assert L.bfs_mcomp(None, None) == bfs.BFS_EINVAL
    assert L.bfs_graph_create(None, None, 0, 0, 1, 1, None, None, None) == bfs.BFS_EINVAL
    L.bfs_destroy(None)  # NULL-safe
    out = ctypes.c_void_p()
    # bad shapes are rejected by argument checks (before any CUDA call)
    assert L.bfs_graph_create(None, None, 0, 0, 1, 1, None, None, ctypes.byref(out)) == bfs.BFS_EINVAL
    assert L.bfs_graph_create(None, None, 0, 8, 0, 1, None, None, ctypes.byref(out)) == bfs.BFS_EINVAL
    o = bfs.make_opts(edges_per_thread=3)
    assert L.bfs_graph_create(None, None, 0, 8, 1, 1, None, ctypes.byref(o), ctypes.byref(out)) == bfs.BFS_EINVAL
    assert b"edges_per_thread" in L.bfs_last_error()
    o = bfs.make_opts(debug_flags=2)  # unknown debug flag
    assert L.bfs_graph_create(None, None, 0, 8, 1, 1, None, ctypes.byref(o), ctypes.byref(out)) == bfs.BFS_EINVAL
    assert L.bfs_gather(None, None, None, None, None) == bfs.BFS_EINVAL


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1408_1605_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                text = open(os.path.join(dp, f)).read()
                assert "import oracle" not in text and "from oracle" not in text and "oracle.c" not in text, f
