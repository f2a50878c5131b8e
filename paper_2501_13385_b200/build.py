"""Build libprgd.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2501_13385_b200.build [--force]

The shared library exports exactly the C-ABI declared in include/prgd.h.  CUDA
runtime is linked statically so the .so has no dependency on the toolkit's
libcudart at run time (PyTorch ships its own)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libprgd.so")
SOURCES = ["api.cu", "sort.cu", "plan.cu", "adaptive.cu", "spectral.cu", "tables.cu", "levels.cu", "passes.cu", "passes_flat.cu", "chains.cu", "dense.cu"]
INCLUDES = ["round_cs.inc"]
HEADERS = ["prgd_internal.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-fvisibility=hidden",
    "-Xptxas", "-v",
    "--cudart", "static",
    "-shared",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS + INCLUDES]
    deps.append(os.path.join(ROOT, "include", "prgd.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"] + os.environ.get("PRGD_EXTRA_NVCC", "").split()
    inc = ["-I", os.path.join(ROOT, "include")]

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *cflags, *inc, "-c", os.path.join(CSRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, res

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log = os.path.join(HERE, "build.log")
    failed = False
    with open(log, "w") as f:
        for src, obj, cmd, res in results:
            f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            failed |= res.returncode != 0
        if not failed:
            cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "--cudart", "static",
                   "-shared", "-o", LIB + ".tmp"] + [r[1] for r in results]
            res = subprocess.run(cmd, capture_output=True, text=True)
            f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            failed = res.returncode != 0
    if failed:
        sys.stderr.write(open(log).read()[-20000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(open(log).read())
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
