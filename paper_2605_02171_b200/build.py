"""Build libqvg.so (sm_100a CUDA + host C++) in-tree with nvcc.

``python paper_2605_02171_b200/build.py`` or ``__graft_entry__.build()``.
Objects go to build/, the shared library next to this file so it travels to
the GPU box with the repo snapshot.  ptxas register/smem reports are kept in
build/ptxas.log.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libqvg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-Wall",
                "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]


def _deps():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))


def _stale(obj, src):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in [src] + _deps())


def _compile(src, obj_dir=OBJ, defines=()):
    obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
    if not _stale(obj, src):
        return obj, ""
    cmd = [NVCC] + FLAGS + list(defines) + ["-c", src, "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{p.stdout}\n{p.stderr}")
    return obj, p.stderr


def build(verbose: bool = False, variant: str = "", defines=()) -> str:
    """Build libqvg.so.  A named `variant` (e.g. instrumented with
    -DQVG_PHASES) goes to build/<variant>/libqvg.so, selected at run time with
    QVG_LIB; the product library is never built with extra defines."""
    obj_dir, lib = OBJ, LIB
    if variant:
        obj_dir = os.path.join(ROOT, "build", "obj_" + variant)
        lib = os.path.join(ROOT, "build", variant, "libqvg.so")
        os.makedirs(os.path.dirname(lib), exist_ok=True)
    os.makedirs(obj_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s_: _compile(s_, obj_dir, defines), srcs))
    objs = [o for o, _ in results]
    logs = "".join(l for _, l in results if l)
    if logs and not variant:
        with open(os.path.join(ROOT, "build", "ptxas.log"), "w") as f:
            f.write(logs)
    if (not os.path.exists(lib)) or any(os.path.getmtime(o) > os.path.getmtime(lib) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{p.stdout}\n{p.stderr}")
    if verbose:
        print(lib)
    return lib


if __name__ == "__main__":
    # python paper_2605_02171_b200/build.py [--variant NAME -DMACRO ...]
    args = sys.argv[1:]
    var = ""
    if args[:1] == ["--variant"]:
        var, args = args[1], args[2:]
    build(verbose=True, variant=var, defines=[a for a in args if a.startswith("-D")])
    sys.exit(0)
