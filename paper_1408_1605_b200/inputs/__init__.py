"""Seeded synthetic inputs (Graph500-style Kronecker tuples + root sampling).

This module is the ONE piece shared by the CUDA path's harness and the CPU oracle's tests: it
generates inputs and holds none of the BFS method's arithmetic.  The generator itself is
defined once in ``kron_gen.h``; this file loads its host build (``libkron_host.so``).  The
device build (``kron_dev.cu`` -> ``libkron_dev.so``) includes the same header, so both produce identical tuples.

Workload recipe: scale S, edge factor 16, A,B,C,D = .57,.19,.19,.05, graph
seed 1, root seed 2, 64 distinct roots uniform over vertices of degree >= 1 (self-loops
excluded), in candidate order of the counter-based root stream.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kron_host.c")
_HDR = os.path.join(_HERE, "kron_gen.h")
_LIB = os.path.join(_HERE, "libkron_host.so")

EDGE_FACTOR = 16
GRAPH_SEED = 1
ROOT_SEED = 2


def build(force: bool = False) -> str:
    stale = (not os.path.exists(_LIB) or
             os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
    if force or stale:
        subprocess.check_call(["gcc", "-O3", "-std=c99", "-fopenmp", "-shared", "-fPIC", "-I", _HERE,
                               "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u64, p, i = ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
        L.kron_host_generate.argtypes = [i, u64, u64, u64, p, p]
        L.kron_host_generate.restype = None
        L.kron_host_generate_u32.argtypes = [i, u64, u64, u64, p, p]
        L.kron_host_generate_u32.restype = None
        L.kron_host_scramble.argtypes = [i, u64, u64]
        L.kron_host_scramble.restype = u64
        L.kron_host_root_candidate.argtypes = [u64, u64, u64]
        L.kron_host_root_candidate.restype = u64
        L.kron_host_thresholds.argtypes = [p]
        L.kron_host_thresholds.restype = None
        _lib = L
    return _lib


def num_tuples(scale: int, edgefactor: int = EDGE_FACTOR) -> int:
    return int(edgefactor) << int(scale)


def generate(scale: int, edgefactor: int = EDGE_FACTOR, seed: int = GRAPH_SEED, k0: int = 0, count=None,
             dtype=np.uint64):
    """Tuples [k0, k0+count) of the Kronecker graph (default: all M = ef * 2^scale)."""
    if not 0 <= scale <= 32:
        raise ValueError("scale must be in [0, 32]")
    if count is None:
        count = num_tuples(scale, edgefactor) - k0
    count = int(count)
    if dtype == np.uint32:
        s = np.empty(count, dtype=np.uint32)
        d = np.empty(count, dtype=np.uint32)
        lib().kron_host_generate_u32(scale, seed, k0, count, s.ctypes.data, d.ctypes.data)
    else:
        s = np.empty(count, dtype=np.uint64)
        d = np.empty(count, dtype=np.uint64)
        lib().kron_host_generate(scale, seed, k0, count, s.ctypes.data, d.ctypes.data)
    return s, d


def scramble(scale: int, seed: int, x: int) -> int:
    return int(lib().kron_host_scramble(scale, seed, x))


def thresholds():
    out = np.zeros(3, dtype=np.uint32)
    lib().kron_host_thresholds(out.ctypes.data)
    return out


def root_candidate(root_seed: int, t: int, nverts: int) -> int:
    return int(lib().kron_host_root_candidate(root_seed, t, nverts))


def nonisolated_mask(n: int, src, dst) -> np.ndarray:
    """True for vertices with at least one non-self-loop tuple (the root eligibility rule)."""
    src = np.asarray(src)
    dst = np.asarray(dst)
    keep = src != dst
    mask = np.zeros(int(n), dtype=bool)
    mask[src[keep]] = True
    mask[dst[keep]] = True
    return mask


def sample_roots(nverts: int, nroots: int, eligible, root_seed: int = ROOT_SEED, max_draws: int = 1 << 24):
    """First `nroots` distinct candidates v of the root stream with eligible(v) True.

    `eligible` is a bool array indexed by vertex or a callable v -> bool.  Fewer roots are
    returned if the stream runs out (e.g. a graph with fewer eligible vertices)."""
    check = (lambda v: bool(eligible[v])) if not callable(eligible) else eligible
    roots, seen = [], set()
    for t in range(max_draws):
        v = root_candidate(root_seed, t, nverts)
        if v in seen:
            continue
        seen.add(v)
        if check(v):
            roots.append(v)
            if len(roots) == nroots:
                break
    return roots


# ---------------------------------------------------------------- device twin (libkron_dev.so)
_DEV_LIB = os.path.join(_HERE, "libkron_dev.so")
_dlib = None


def dev_lib():
    global _dlib
    if _dlib is None:
        if not os.path.exists(_DEV_LIB):
            raise RuntimeError(f"{_DEV_LIB} not built: run __graft_entry__.build()")
        L = ctypes.CDLL(_DEV_LIB)
        L.kron_device_generate.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.kron_device_generate.restype = ctypes.c_int
        _dlib = L
    return _dlib


def generate_device(scale: int, edgefactor: int = EDGE_FACTOR, seed: int = GRAPH_SEED, k0: int = 0, count=None,
                    device="cuda"):
    """Tuples [k0, k0+count) generated directly in HBM: two torch uint64 CUDA tensors."""
    import torch
    if count is None:
        count = num_tuples(scale, edgefactor) - k0
    s = torch.empty(int(count), dtype=torch.uint64, device=device)
    d = torch.empty(int(count), dtype=torch.uint64, device=device)
    stream = torch.cuda.current_stream(s.device).cuda_stream
    rc = dev_lib().kron_device_generate(int(scale), int(seed), int(k0), int(count), s.data_ptr(), d.data_ptr(),
                                        stream)
    if rc != 0:
        raise RuntimeError(f"kron_device_generate failed: cudaError {rc}")
    return s, d
