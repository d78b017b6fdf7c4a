"""Thin ctypes binding of libbfs200.so (include/bfs200.h).  Argument marshalling only.

Every step of the BFS runs in the CUDA library; there is no CPU fallback.  If the library is
missing or no GPU is present, the calls raise.

Buffers may be numpy arrays (host) or torch tensors (host or CUDA); the library classifies
pointers itself (cudaPointerGetAttributes).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

_LIB = os.environ.get("BFS200_LIB") or _build.LIB  # BFS200_LIB: an alternative build of the same ABI (A/B runs)

BFS_OK, BFS_EINVAL, BFS_ERANGE, BFS_ENOMEM, BFS_ECUDA, BFS_ENCCL, BFS_ESTATE, BFS_EPARSE = 0, -1, -2, -3, -4, -5, -6, -7
FMT = {"snap-text": 0, "binary-pairs": 1}


class BfsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{msg} (status {status})")
        self.status = status


class Comm(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("device", ctypes.c_int),
                ("loopback", ctypes.c_int), ("nccl_id", ctypes.c_ubyte * 128)]


class Opts(ctypes.Structure):
    _fields_ = [("edges_per_thread", ctypes.c_int), ("phase_timing", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("exchange", ctypes.c_int), ("peer_exchange", ctypes.c_int), ("debug_flags", ctypes.c_int)]


class Info(ctypes.Structure):
    _fields_ = [("nverts", ctypes.c_uint64), ("npad", ctypes.c_uint64), ("block", ctypes.c_uint64),
                ("R", ctypes.c_int), ("C", ctypes.c_int), ("rank", ctypes.c_int), ("nlocal", ctypes.c_int),
                ("first_vertex", ctypes.c_uint64), ("nout", ctypes.c_uint64), ("nnz_local", ctypes.c_uint64),
                ("ntuples", ctypes.c_uint64), ("device_bytes", ctypes.c_uint64)]


class Stats(ctypes.Structure):
    _fields_ = [("nlevels", ctypes.c_int), ("edges_scanned", ctypes.c_uint64),
                ("frontier_columns", ctypes.c_uint64), ("reached", ctypes.c_uint64),
                ("bytes_exchanged", ctypes.c_uint64), ("list_messages", ctypes.c_uint64),
                ("kernel_launches", ctypes.c_uint64),
                ("finalize_ms", ctypes.c_double), ("resolve_ms", ctypes.c_double)]


class LevelRecord(ctypes.Structure):
    _fields_ = [("expand_comm", ctypes.c_double), ("scan", ctypes.c_double), ("expand", ctypes.c_double),
                ("parent", ctypes.c_double), ("fold_comm", ctypes.c_double), ("update", ctypes.c_double), ("allreduce", ctypes.c_double),
                ("frontier", ctypes.c_uint64), ("edges", ctypes.c_uint64)]


EXPORTS = ["bfs_nccl_unique_id", "bfs_graph_create", "bfs_graph_info", "bfs_set_opts", "bfs_degree", "bfs_run",
           "bfs_run_batch",
           "bfs_mcomp", "bfs_level_times", "bfs_gather", "bfs_load_edges", "bfs_free_edges", "bfs_destroy",
           "bfs_strerror", "bfs_last_error"]
DEBUG_POS64 = 1

_lib = None


def lib(build: bool = False):
    """Load libbfs200.so (building it first if `build`); raises if it cannot be loaded."""
    global _lib
    if _lib is None:
        if build:
            _build.build_bfs()
        if not os.path.exists(_LIB):
            raise RuntimeError(f"{_LIB} not built: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(_LIB)
        p, u64, i = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
        L.bfs_nccl_unique_id.argtypes = [p]
        L.bfs_graph_create.argtypes = [p, p, u64, u64, i, i, ctypes.POINTER(Comm), ctypes.POINTER(Opts),
                                       ctypes.POINTER(p)]
        L.bfs_graph_info.argtypes = [p, ctypes.POINTER(Info)]
        L.bfs_set_opts.argtypes = [p, ctypes.POINTER(Opts)]
        L.bfs_degree.argtypes = [p, u64, ctypes.POINTER(u64)]
        L.bfs_run.argtypes = [p, u64, p, p, ctypes.POINTER(Stats)]
        L.bfs_run_batch.argtypes = [p, ctypes.POINTER(u64), i, ctypes.POINTER(p), ctypes.POINTER(p),
                                    ctypes.POINTER(Stats)]
        L.bfs_mcomp.argtypes = [p, ctypes.POINTER(u64)]
        L.bfs_level_times.argtypes = [p, ctypes.POINTER(LevelRecord), i, ctypes.POINTER(i)]
        L.bfs_gather.argtypes = [p, p, p, p, p]
        pu64 = ctypes.POINTER(ctypes.c_uint64)
        L.bfs_load_edges.argtypes = [ctypes.c_char_p, i, ctypes.POINTER(pu64), ctypes.POINTER(pu64),
                                     ctypes.POINTER(u64), ctypes.POINTER(u64)]
        L.bfs_free_edges.argtypes = [pu64, pu64]
        L.bfs_free_edges.restype = None
        L.bfs_destroy.argtypes = [p]
        L.bfs_destroy.restype = None
        L.bfs_strerror.argtypes = [i]
        L.bfs_strerror.restype = ctypes.c_char_p
        L.bfs_last_error.argtypes = []
        L.bfs_last_error.restype = ctypes.c_char_p
        for name in EXPORTS:
            if name not in ("bfs_destroy", "bfs_free_edges", "bfs_strerror", "bfs_last_error"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(rc):
    if rc != BFS_OK:
        L = lib()
        raise BfsError(rc, f"{L.bfs_strerror(rc).decode()}: {L.bfs_last_error().decode()}")


def _ptr(x):
    """Raw address of a numpy array / torch tensor (contiguous) or None."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be contiguous")
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    raise TypeError(f"unsupported buffer type {type(x)}")


def load_edges(path: str, fmt: str = "snap-text"):
    """bfs_load_edges: (src uint64[m], dst uint64[m], nverts) of a SNAP text / binary-pairs file
    (host numpy arrays, copied out of the library's buffers)."""
    L = lib()
    pu64 = ctypes.POINTER(ctypes.c_uint64)
    s, d = pu64(), pu64()
    m, nv = ctypes.c_uint64(), ctypes.c_uint64()
    _check(L.bfs_load_edges(os.fsencode(path), FMT[fmt] if isinstance(fmt, str) else int(fmt), ctypes.byref(s),
                            ctypes.byref(d), ctypes.byref(m), ctypes.byref(nv)))
    try:
        n = int(m.value)
        src = np.ctypeslib.as_array(s, shape=(n,)).copy() if n else np.zeros(0, np.uint64)
        dst = np.ctypeslib.as_array(d, shape=(n,)).copy() if n else np.zeros(0, np.uint64)
    finally:
        L.bfs_free_edges(s, d)
    return src.astype(np.uint64, copy=False), dst.astype(np.uint64, copy=False), int(nv.value)


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _check(lib().bfs_nccl_unique_id(buf))
    return bytes(buf)


def make_comm(rank=0, nranks=1, device=0, loopback=True, nccl_id: bytes | None = None) -> Comm:
    c = Comm()
    c.rank, c.nranks, c.device, c.loopback = rank, nranks, device, 1 if loopback else 0
    if nccl_id is not None:
        ctypes.memmove(c.nccl_id, nccl_id, 128)
    return c


XCHG_BITMAP, XCHG_LIST, XCHG_AUTO = 0, 1, 2
XCHG = {"bitmap": XCHG_BITMAP, "list": XCHG_LIST, "auto": XCHG_AUTO}


def make_opts(edges_per_thread=4, phase_timing=False, stream=None, exchange="bitmap", peer_exchange=False,
              debug_flags=0) -> Opts:
    o = Opts()
    o.debug_flags = int(debug_flags)
    o.peer_exchange = 1 if peer_exchange else 0
    o.edges_per_thread = int(edges_per_thread)
    o.phase_timing = 1 if phase_timing else 0
    o.exchange = XCHG[exchange] if isinstance(exchange, str) else int(exchange)
    if stream is not None:
        o.stream = stream if isinstance(stream, int) else getattr(stream, "cuda_stream", None)
    return o


class Graph:
    """A partitioned graph resident on the GPU (bfs_graph_create .. bfs_destroy)."""

    def __init__(self, src, dst, nverts, R=1, C=1, comm: Comm | None = None, opts: Opts | None = None):
        L = lib()
        n = int(len(src))
        if int(len(dst)) != n:
            raise ValueError("src/dst length mismatch")
        for a in (src, dst):
            dt = getattr(a, "dtype", None)
            if str(dt) not in ("uint64", "torch.uint64", "int64", "torch.int64"):
                raise TypeError(f"edge arrays must be 64-bit integers, got {dt}")
        h = ctypes.c_void_p()
        _check(L.bfs_graph_create(_ptr(src), _ptr(dst), n, int(nverts), int(R), int(C),
                                  ctypes.byref(comm) if comm is not None else None,
                                  ctypes.byref(opts) if opts is not None else None, ctypes.byref(h)))
        self._h = h
        self.info = self.get_info()

    def get_info(self) -> Info:
        inf = Info()
        _check(lib().bfs_graph_info(self._h, ctypes.byref(inf)))
        return inf

    def set_opts(self, opts: Opts):
        _check(lib().bfs_set_opts(self._h, ctypes.byref(opts)))

    def degree(self, v: int) -> int:
        out = ctypes.c_uint64()
        _check(lib().bfs_degree(self._h, int(v), ctypes.byref(out)))
        return int(out.value)

    def run(self, root: int, parent=None, level=None, want_stats=True):
        """BFS from root into the given buffers (numpy/torch, host or device). Returns Stats."""
        st = Stats()
        _check(lib().bfs_run(self._h, int(root), _ptr(parent), _ptr(level),
                             ctypes.byref(st) if want_stats else None))
        return st

    def run_batch(self, roots, parents=None, levels=None, want_stats=False):
        """bfs_run_batch: one BFS per root, outputs into parents[k] / levels[k] (lists of buffers, host
        or device; None to skip). Host copies of root k overlap root k+1's search (pinned buffers).
        Returns the per-root Stats when want_stats."""
        n = len(roots)
        r = (ctypes.c_uint64 * max(n, 1))(*[int(x) for x in roots])

        def ptrs(bufs):
            if bufs is None:
                return None
            if len(bufs) != n:
                raise ValueError("one output buffer (or None) per root")
            return (ctypes.c_void_p * max(n, 1))(*[_ptr(b) for b in bufs])

        st = (Stats * max(n, 1))() if want_stats else None
        _check(lib().bfs_run_batch(self._h, r, n, ptrs(parents), ptrs(levels), st))
        return [st[k] for k in range(n)] if want_stats else None

    def bfs(self, root: int):
        """Convenience: (level int32[nout], parent int64[nout]) as host numpy arrays."""
        parent = np.empty(self.info.nout, dtype=np.int64)
        level = np.empty(self.info.nout, dtype=np.int32)
        self.run(root, parent, level)
        return level, parent

    def gather(self, parent=None, level=None, parent_all=None, level_all=None):
        """bfs_gather: this process's outputs -> every rank's outputs on world rank 0 (collective)."""
        _check(lib().bfs_gather(self._h, _ptr(parent), _ptr(level), _ptr(parent_all), _ptr(level_all)))

    def mcomp(self) -> int:
        out = ctypes.c_uint64()
        _check(lib().bfs_mcomp(self._h, ctypes.byref(out)))
        return int(out.value)

    def level_times(self, max_levels=256):
        recs = (LevelRecord * max_levels)()
        n = ctypes.c_int()
        _check(lib().bfs_level_times(self._h, recs, max_levels, ctypes.byref(n)))
        return [recs[i] for i in range(min(n.value, max_levels))]

    def close(self):
        if getattr(self, "_h", None):
            lib().bfs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
