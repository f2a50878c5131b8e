"""CPU oracle timings: median of 3 oracle PRGD steps per config on this host,
with the BLAS limited to 1 thread and with all affinity cores; CPU model and BLAS reported.

    python tools/cpu_oracle.py [cfgs...]      (default 1 2 3; config 4/5 at a bounded sample)"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from threadpoolctl import threadpool_info, threadpool_limits  # noqa: E402

import bench  # noqa: E402  (host_info only)
import oracle  # noqa: E402
import synth  # noqa: E402

cfgs = [int(c) for c in sys.argv[1:]] or [1, 2, 3]
out = {"host": bench.host_info(), "configs": {}}
ncores = len(os.sched_getaffinity(0))
for cfg in cfgs:
    m = {4: 300_000, 5: 1_000_000}.get(cfg)
    pr = synth.make_problem(cfg, m=m)
    y = pr.observations(oracle.eval_at(pr.truth, pr.idx))
    T0 = pr.init if pr.init is not None else oracle.spectral_init(pr.idx, y, pr.n, pr.r)
    row = {"m": pr.m, "m_full": synth.make_problem(cfg).m if cfg not in (5,) else 29999562}
    for threads in (1, ncores):
        with threadpool_limits(limits=threads, user_api="blas"):
            ts = []
            T = T0
            for _ in range(3):
                t0 = time.perf_counter()
                T = oracle.prgd_step(T, pr.idx, y, pr.n, pr.r, 0.5 if cfg == 3 else 1.0)
                ts.append(time.perf_counter() - t0)
        med = statistics.median(ts)
        row[f"threads_{threads}"] = {"step_s": round(med, 4), "iter_per_s": round(1 / med, 4),
                                     "entries_per_s": round(pr.m / med, 1)}
    out["configs"][cfg] = row
    print(cfg, json.dumps(row), flush=True)
print(json.dumps(out))
