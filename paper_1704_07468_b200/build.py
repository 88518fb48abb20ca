"""Build libgakco.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_1704_07468_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libgakco.so")
# bounds-checked variant (device asserts, GK_CHECK): compute-sanitizer is closed on the
# GPU pool, so the test suite runs against this one instead (GAKCO_LIB=...)
OBJ_CHECKED = os.path.join(ROOT, "build", "obj_checked")
LIB_CHECKED = os.path.join(PKG, "libgakco_checked.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + \
        [os.path.join(ROOT, "include", "gakco.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, extra):
    obj = os.path.join(extra.get("obj", OBJ), os.path.basename(src) + ".o")
    if _stale(obj, [src] + _deps()) or extra.get("force"):
        cmd = [NVCC] + ARCH + FLAGS + extra.get("flags", []) + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if extra.get("verbose") and r.stderr.strip():
            print(r.stderr, file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, flags=None, checked: bool = False) -> str:
    obj_dir, lib = (OBJ_CHECKED, LIB_CHECKED) if checked else (OBJ, LIB)
    os.makedirs(obj_dir, exist_ok=True)
    srcs = sources()
    extra = {"force": force, "verbose": verbose, "obj": obj_dir,
             "flags": list(flags or []) + (["-DGAKCO_CHECKS"] if checked else [])}
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, extra), srcs))
    if force or _stale(lib, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-lcudart", "-ldl"]
        subprocess.check_call(cmd)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                flags=["-Xptxas", "-v"] if "--ptxas" in sys.argv else None,
                checked="--checked" in sys.argv))
