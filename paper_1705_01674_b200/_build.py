"""In-tree build of the native library (sm_100a only).

``build_native()`` compiles every ``csrc/*.cu`` with
``nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` in parallel into
``build/obj`` and links ``paper_1705_01674_b200/libsgwls_b200.so`` (git-ignored,
shipped to the GPU box with the snapshot).  Rebuilds only what changed.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libsgwls_b200.so")
INCLUDE = os.path.join(ROOT, "include")
CLI = os.path.join(PKG, "bin", "sgwls_b200")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
              "--expt-relaxed-constexpr", "-I" + INCLUDE]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise FileNotFoundError("nvcc not found")


def _deps() -> list[str]:
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + [os.path.join(INCLUDE, "sgwls_b200.h")])


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources if os.path.exists(s))


def _compile(src: str, extra: list[str], obj_dir: str = OBJ) -> str:
    obj = os.path.join(obj_dir, os.path.basename(src).replace(".cu", ".o"))
    if _stale(obj, [src] + _deps()):
        cmd = [nvcc()] + ARCH + NVCC_FLAGS + extra + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build_native(verbose: bool = False, extra: list[str] | None = None, variant: str | None = None) -> str:
    """variant: build a tuning variant (extra nvcc flags) into variants/lib_<variant>.so
    (load it with SGWLS_B200_LIB=...); the default build is libsgwls_b200.so."""
    obj_dir = OBJ if variant is None else os.path.join(ROOT, "build", "obj_" + variant)
    lib = LIB if variant is None else os.path.join(PKG, "variants", f"lib_{variant}.so")
    os.makedirs(obj_dir, exist_ok=True)
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    extra = list(extra or [])
    with cf.ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda s: _compile(s, extra, obj_dir), srcs))
    if _stale(lib, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", lib] + objs + ["-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if variant is None:
        build_cli()
    if verbose:
        print("built", lib)
    return lib


def build_cli() -> str:
    """The command-line tool (csrc/tools/sgwls_b200_main.cpp, the drop-in for the
    reference's proj/tools/sgwls_main.cpp): plain C++ on the C ABI, linked against
    the in-tree library with an $ORIGIN-relative rpath."""
    src = os.path.join(CSRC, "tools", "sgwls_b200_main.cpp")
    if _stale(CLI, [src, LIB, os.path.join(INCLUDE, "sgwls_b200.h")]):
        os.makedirs(os.path.dirname(CLI), exist_ok=True)
        cmd = ["g++", "-O2", "-std=c++17", "-Wall", "-Wextra", "-I" + INCLUDE, src, "-o", CLI, "-L" + PKG,
               "-lsgwls_b200", "-Wl,-rpath,$ORIGIN/.."]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"g++ failed for {src}:\n{r.stdout}\n{r.stderr}")
    return CLI


if __name__ == "__main__":
    import sys

    args = sys.argv[1:]
    var = None
    if args and args[0] == "--variant":
        var, args = args[1], args[2:]
    build_native(verbose=True, extra=args, variant=var)
