"""Builds libgut.so (the C-ABI library, include/gut.h) in-tree for sm_100a.

    python -m paper_2412_12507_b200.build [--force]

nvcc cross-compiles here without a GPU; the .so travels to the B200 box with
the gpurun snapshot.  Only compute_100a / sm_100a code is generated: there is
no other architecture and no CPU fallback.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libgut.so")
OBJ = os.path.join(HERE, "build")
SOURCES = ["k1_project.cu", "k3_sort.cu", "k2_emit.cu", "k5_blend.cu", "k6_backward.cu", "gut_abi.cu"]
HEADERS = ["gut_internal.cuh", "launch.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include")]
# tuning experiments only: extra -D flags and an alternative output (see gut.py GUT_LIB)
FLAGS += os.environ.get("GUT_EXTRA_FLAGS", "").split()
if os.environ.get("GUT_LIB_OUT"):
    OUT = os.environ["GUT_LIB_OUT"]
    OBJ = OUT + ".objs"


def _newest_input() -> float:
    paths = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "gut.h")]
    return max(os.path.getmtime(p) for p in paths)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= _newest_input():
        return OUT
    os.makedirs(OBJ, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        cmd = [NVCC] + FLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        with open(os.path.join(OBJ, src + ".ptxas.txt"), "w") as f:
            f.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", "-o", OUT] + objs
    subprocess.check_call(cmd)
    if verbose:
        for s in SOURCES:
            print(open(os.path.join(OBJ, s + ".ptxas.txt")).read())
    return OUT


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)
