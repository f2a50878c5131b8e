"""Write the oracle reference iterates used by the long GPU parity tests.

    python tools/make_golden.py CASE [CASE ...]      (CASE in tests/_golden.py CASES)

Calls ONLY `synth` (seeded inputs) and `oracle` (the CPU fp64 PRGD of Alg. 2,
PAPER.md:208-222): no CUDA path is imported.  Each case stores, in tests/golden/<case>.npz,
the oracle iterate after the saved steps, the residual-norm trajectory, and a fingerprint of
the inputs (SHA-256 of the synth arrays idx / noise / init, plus sum and sum of squares of y)
so a test refuses a stale file.  The GPU tests (tests/test_gpu_parity_long.py) re-derive the
same inputs from synth + oracle.eval_at and compare the library's iterates with these files
at BASELINE.json's tolerances (1e-11 after one step, 1e-8 after 50).  They exist because the
full-size oracle runs take minutes to hours of CPU (config 5 at 3e7 samples: ~5 min per step
on 2 threads)."""
from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from tests import _golden as G  # noqa: E402


def _ckpt(case: str) -> str:
    # resumable runs (config 5 at full size: hours of CPU); scratch, not a golden file
    return os.path.join(ROOT, "gpurun_out", "golden_ckpt", case + ".npz")


# cases still being generated (moved into tests/_golden.py CASES once their file exists)
PENDING = {
    # full config 5, 50 steps (BASELINE.json:11 "50 iterations"; north star: 1e-8 after 50)
    "cfg5_full_50steps": (5, None, 1.0, 50, (1, 10, 50)),
}


def make(case: str) -> str:
    cfg, m, step, steps, keep = {**G.CASES, **PENDING}[case]
    t0 = time.time()
    pr = G.problem(cfg, m)
    y = G.observations(pr)
    sha = G.input_sha(pr)
    T = pr.init
    res, out = [], {}
    start = 1
    ck = _ckpt(case)
    if os.path.exists(ck):
        z = np.load(ck)
        if str(z["sha"]) == sha:
            start = int(z["it"]) + 1
            T = [z[f"T{k}"] for k in range(len(pr.n))]
            res = [float(v) for v in z["res"]]
            out = {k: z[k] for k in z.files if k.startswith("s") and "_c" in k}   # saved iterates s<it>_c<k>
            print(f"{case}: resuming after step {start - 1}", flush=True)
    for it in range(start, steps + 1):
        T, info = oracle.prgd_step(T, pr.idx, y, pr.n, pr.r, step, return_info=True)
        res.append(math.sqrt(info["sumsq"]))        # residual of the iterate the step started from
        if it in keep:
            for k, c in enumerate(T):
                out[f"s{it}_c{k}"] = c
        print(f"{case}: step {it}/{steps} residual {res[-1]:.6e} ({time.time() - t0:.0f} s)", flush=True)
        if steps > 1:
            os.makedirs(os.path.dirname(ck), exist_ok=True)
            np.savez(ck + ".tmp.npz", it=it, sha=sha, res=np.array(res),
                     **{f"T{k}": c for k, c in enumerate(T)}, **out)
            os.replace(ck + ".tmp.npz", ck)
    res.append(float(np.linalg.norm(oracle.residual(T, pr.idx, y))))
    os.makedirs(G.GOLDEN_DIR, exist_ok=True)
    p = G.path(case)
    np.savez_compressed(p, cfg=cfg, m=-1 if m is None else m, step_size=step, steps=steps,
                        keep=np.array(keep), d=len(pr.n), res=np.array(res), sha=sha,
                        ysum=float(np.sum(y)), ysq=float(np.dot(y, y)), mm=pr.m, **out)
    return p


if __name__ == "__main__":
    for c in sys.argv[1:]:
        print(make(c))
