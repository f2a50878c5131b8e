"""Build an experimental variant of libprgd.so with extra nvcc flags (measurement only):

    python tools/build_variant.py NAME "-DFLAG=1 ..."   -> paper_2501_13385_b200/libprgd_NAME.so

Run it with PRGD_LIB_PATH=paper_2501_13385_b200/libprgd_NAME.so (the product path always loads
libprgd.so built by __graft_entry__.build())."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_13385_b200 import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2].split()
objdir = os.path.join(B.HERE, "build_" + name)
os.makedirs(objdir, exist_ok=True)
cflags = [f for f in B.FLAGS if f not in ("-shared", "-Xptxas", "-v")] + extra
inc = ["-I", os.path.join(ROOT, "include")]


def one(src):
    obj = os.path.join(objdir, src.replace(".cu", ".o"))
    r = subprocess.run([B.NVCC, *cflags, *inc, "-c", os.path.join(B.CSRC, src), "-o", obj],
                       capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stderr)
        raise SystemExit(1)
    return obj


with ThreadPoolExecutor(len(B.SOURCES)) as ex:
    objs = list(ex.map(one, B.SOURCES))
out = os.path.join(B.HERE, f"libprgd_{name}.so")
subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "--cudart", "static", "-shared",
                "-o", out] + objs, check=True)
print(out)
