"""Build the sm_100a CUDA libraries in-tree with nvcc (no JIT, no torch extension cache).

  libbfs200.so           csrc/*.cu   -- the product: C-ABI BFS library (include/bfs200.h)
  inputs/libkron_dev.so  inputs/kron_dev.cu -- device twin of the input generator

Both are rebuilt only when a source or header is newer than the library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libbfs200.so")
KRON_DEV_LIB = os.path.join(PKG, "inputs", "libkron_dev.so")
BUILD_DIR = os.path.join(PKG, "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
              "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def nccl_dirs():
    cands = []
    try:
        import nvidia.nccl  # type: ignore
        cands.extend(list(nvidia.nccl.__path__))
    except Exception:
        pass
    sp = sysconfig.get_paths().get("purelib", "")
    cands.append(os.path.join(sp, "nvidia", "nccl"))
    for base in cands:
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    raise RuntimeError("NCCL headers/library not found (expected the nvidia-nccl wheel bundled with torch)")


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths), default=0.0)


def _stale(target, deps):
    return not os.path.exists(target) or os.path.getmtime(target) < _newest(deps)


def _run(cmd, log):
    p = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
    if p.returncode != 0:
        sys.stderr.write(p.stdout + p.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ... (see {log})")


def build_bfs(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(INCLUDE, "*.h")))
    if not force and not _stale(LIB, srcs + hdrs):
        return LIB
    os.makedirs(BUILD_DIR, exist_ok=True)
    inc, lib = nccl_dirs()
    objs = []
    jobs = []
    for s in srcs:
        o = os.path.join(BUILD_DIR, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append(([nvcc(), *ARCH, *NVCC_FLAGS, "-I", INCLUDE, "-I", inc, "-c", s, "-o", o], o + ".log"))
    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(lambda a: _run(*a), jobs))
    tmp = LIB + ".tmp"
    _run([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-L", lib, "-l:libnccl.so.2",
          "-Xlinker", f"-rpath={lib}", "-lcudart"], os.path.join(BUILD_DIR, "link.log"))
    os.replace(tmp, LIB)
    if verbose:
        for o in objs:
            print(open(o + ".log").read()[-2000:])
    return LIB


def build_variant(name: str, defines, force: bool = False, csrc: str = CSRC, include: str = INCLUDE) -> str:
    """An experiment build of the library with extra -D flags, or of another source tree (e.g. a
    git revision exported by tools/build_rev.py), for A/B runs through BFS200_LIB;
    build/variants/lib<name>.so.  Never loaded unless BFS200_LIB points at it."""
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(csrc, "*.h")) + glob.glob(os.path.join(csrc, "*.cuh")) +
                  glob.glob(os.path.join(include, "*.h")))
    vdir = os.path.join(BUILD_DIR, "variants", name)
    out = os.path.join(BUILD_DIR, "variants", f"lib{name}.so")
    if not force and not _stale(out, srcs + hdrs):
        return out
    os.makedirs(vdir, exist_ok=True)
    inc, lib = nccl_dirs()
    dflags = [f"-D{d}" for d in defines]
    objs, jobs = [], []
    for s in srcs:
        o = os.path.join(vdir, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        jobs.append(([nvcc(), *ARCH, *NVCC_FLAGS, *dflags, "-I", include, "-I", inc, "-c", s, "-o", o], o + ".log"))
    with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
        list(ex.map(lambda a: _run(*a), jobs))
    _run([nvcc(), *ARCH, "-shared", "-o", out, *objs, "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}",
          "-lcudart"], os.path.join(vdir, "link.log"))
    return out


def build_kron_dev(force: bool = False) -> str:
    src = os.path.join(PKG, "inputs", "kron_dev.cu")
    hdr = os.path.join(PKG, "inputs", "kron_gen.h")
    if not force and not _stale(KRON_DEV_LIB, [src, hdr]):
        return KRON_DEV_LIB
    os.makedirs(BUILD_DIR, exist_ok=True)
    tmp = KRON_DEV_LIB + ".tmp"
    _run([nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-o", tmp, src],
         os.path.join(BUILD_DIR, "kron_dev.log"))
    os.replace(tmp, KRON_DEV_LIB)
    return KRON_DEV_LIB


def build_all(force: bool = False) -> None:
    from . import inputs
    inputs.build(force)
    build_kron_dev(force)
    build_bfs(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print(LIB)
