"""Build the sm_100a extension: csrc/*.cu + csrc/*.cpp -> libshouji_b200.so (in-tree).

Every translation unit is compiled by nvcc for ``-gencode arch=compute_100a,code=sm_100a``
with ``-lineinfo`` (so ncu's source page maps back), in parallel, then linked into one
shared library with a plain C ABI (include/shouji_b200.h). No torch types cross the
boundary; the Python package loads it with ctypes.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libshouji_b200.so")
CLI = os.path.join(PKG, "shouji-b200")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
          "-I" + os.path.join(ROOT, "include")]


def _sources():
    out = []
    for f in sorted(os.listdir(CSRC)):
        if f.endswith((".cu", ".cpp")):
            out.append(os.path.join(CSRC, f))
    return out


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "shouji_b200.h"))
    return hs


def _obj_for(src):
    return os.path.join(OBJ, os.path.basename(src) + ".o")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose=False):
    obj = _obj_for(src)
    if not _stale(obj, [src] + _headers()):
        return obj, None
    cmd = [NVCC] + ARCH + COMMON + ["-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC] + COMMON + ["-x", "c++", "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False, jobs: int | None = None) -> str:
    """Compile (incrementally) and link; returns the path of the shared library."""
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    jobs = jobs or max(1, min(len(srcs), os.cpu_count() or 1))
    logs = []
    with cf.ThreadPoolExecutor(jobs) as ex:
        for obj, log in ex.map(lambda s: _compile(s, verbose), srcs):
            if log:
                logs.append(log)
    objs = [_obj_for(s) for s in srcs]
    if _stale(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    # command-line caller (tools/shouji_cli.cpp), linked against the library
    cli_src = os.path.join(PKG, "tools", "shouji_cli.cpp")
    if _stale(CLI, [cli_src, LIB, os.path.join(ROOT, "include", "shouji_b200.h")]):
        cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"), cli_src,
               "-o", CLI, "-L" + PKG, "-lshouji_b200", "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"CLI build failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        for lg in logs:
            sys.stderr.write(lg)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
