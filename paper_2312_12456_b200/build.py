"""Builds libpi.so in-tree with nvcc for sm_100a (no JIT cache, so the .so travels with the repo).

Every translation unit under csrc/ (the ABI layer, one unit per kernel instantiation group, the
host placement code) compiles to an object in parallel; the objects link into one shared library."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libpi.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include")]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))) + \
        [os.path.join(ROOT, "include", "pi.h")]


def _obj(src: str) -> str:
    return os.path.join(OBJ, os.path.basename(src) + ".o")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build_lib(force: bool = False, verbose: bool = False, jobs: int = 0) -> str:
    srcs = sources()
    hdrs = headers()
    os.makedirs(OBJ, exist_ok=True)
    todo = [s for s in srcs if force or _stale(_obj(s), [s] + hdrs)]

    def compile_one(src):
        cmd = [NVCC, *FLAGS, "-c", src, "-o", _obj(src) + ".tmp"]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {os.path.basename(src)}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        os.replace(_obj(src) + ".tmp", _obj(src))

    if todo:
        n = jobs or min(len(todo), os.cpu_count() or 4)
        with ThreadPoolExecutor(max_workers=n) as ex:
            list(ex.map(compile_one, todo))
    objs = [_obj(s) for s in srcs]
    if todo or force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", *objs, "-o", LIB + ".tmp", "-cudart", "static"]
        subprocess.run(cmd, check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build_lib(force="--force" in sys.argv, verbose="-v" in sys.argv))
