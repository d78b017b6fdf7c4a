"""CPU oracle for the BFS of arXiv 1408.1605 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_1408_1605_b200``) never imports it, and it imports nothing from the product path.

The arithmetic lives in ``oracle.c`` (plain serial C; see its header for the definition it
follows and the PAPER.md passages it cites).  This module is ctypes marshalling only.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

V_NAMES = ["V1 root", "V2 tree-edge", "V3 level+1", "V4 edge-span", "V5 component", "V6 min-rule",
           "range"]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (plain -O2, no vectorisation tricks needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u64, p = ctypes.c_uint64, ctypes.c_void_p
        L.oracle_build.argtypes = [u64, u64, p, p]
        L.oracle_build.restype = p
        L.oracle_free.argtypes = [p]
        L.oracle_free.restype = None
        L.oracle_num_adjacency.argtypes = [p]
        L.oracle_num_adjacency.restype = u64
        L.oracle_degree.argtypes = [p, u64]
        L.oracle_degree.restype = u64
        L.oracle_bfs.argtypes = [p, u64, p, p]
        L.oracle_bfs.restype = ctypes.c_int
        L.oracle_mcomp.argtypes = [p, p]
        L.oracle_mcomp.restype = u64
        L.oracle_validate.argtypes = [u64, u64, p, p, u64, p, p]
        L.oracle_validate.restype = ctypes.c_int
        L.oracle_vstream_begin.argtypes = [u64, u64, p, p]
        L.oracle_vstream_begin.restype = p
        L.oracle_vstream_feed.argtypes = [p, u64, p, p]
        L.oracle_vstream_feed.restype = None
        L.oracle_vstream_mcomp.argtypes = [p]
        L.oracle_vstream_mcomp.restype = u64
        L.oracle_vstream_end.argtypes = [p]
        L.oracle_vstream_end.restype = ctypes.c_int
        _lib = L
    return _lib


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


class Graph:
    """Undirected adjacency of a tuple list (oracle step 1).  Holds references to the arrays."""

    def __init__(self, n: int, src, dst):
        self.n = int(n)
        self.src = _u64(src)
        self.dst = _u64(dst)
        if self.src.shape != self.dst.shape:
            raise ValueError("src/dst length mismatch")
        self.m = int(self.src.size)
        h = lib().oracle_build(self.n, self.m, self.src.ctypes.data, self.dst.ctypes.data)
        if not h:
            raise ValueError("oracle_build failed (endpoint >= n or out of memory)")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().oracle_free(h)
            self._h = None

    def degree(self, v: int) -> int:
        return int(lib().oracle_degree(self._h, int(v)))

    def bfs(self, root: int):
        """(level int32[n], parent int64[n]) for root (oracle steps 2-3)."""
        level = np.empty(self.n, dtype=np.int32)
        parent = np.empty(self.n, dtype=np.int64)
        rc = lib().oracle_bfs(self._h, int(root), level.ctypes.data, parent.ctypes.data)
        if rc == -2:
            raise IndexError("root out of range")
        if rc != 0:
            raise MemoryError("oracle_bfs failed")
        return level, parent

    def mcomp(self, level) -> int:
        level = np.ascontiguousarray(level, dtype=np.int32)
        return int(lib().oracle_mcomp(self._h, level.ctypes.data))


def validate(n: int, src, dst, root: int, level, parent) -> int:
    """Bitmask of failed Graph500 invariants V1..V6 (0 == valid); see oracle.c."""
    src, dst = _u64(src), _u64(dst)
    level = np.ascontiguousarray(level, dtype=np.int32)
    parent = np.ascontiguousarray(parent, dtype=np.int64)
    return int(lib().oracle_validate(int(n), int(src.size), src.ctypes.data, dst.ctypes.data, int(root),
                                     level.ctypes.data, parent.ctypes.data))


def failed_names(mask: int):
    return [V_NAMES[i] for i in range(len(V_NAMES)) if mask >> i & 1]


def validate_stream(n: int, root: int, level, parent, chunks):
    """Streaming V1..V6 (oracle.c step 6): `chunks` yields (src, dst) tuple arrays, e.g. the
    tuple list regenerated from its seed chunk by chunk.  Returns (mask, m_comp)."""
    level = np.ascontiguousarray(level, dtype=np.int32)
    parent = np.ascontiguousarray(parent, dtype=np.int64)
    if level.size < n or parent.size < n:
        raise ValueError("level/parent shorter than n")
    L = lib()
    st = L.oracle_vstream_begin(int(n), int(root), level.ctypes.data, parent.ctypes.data)
    if not st:
        raise MemoryError("oracle_vstream_begin failed")
    try:
        for s, d in chunks:
            s, d = _u64(s), _u64(d)
            L.oracle_vstream_feed(st, int(s.size), s.ctypes.data, d.ctypes.data)
        mc = int(L.oracle_vstream_mcomp(st))
    finally:
        mask = int(L.oracle_vstream_end(st))
    return mask, mc
