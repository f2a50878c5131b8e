"""Benchmark of the PRGD hot path (arXiv 2501.13385) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 5]

Workload (BASELINE.json configs[4], the metric's config): d=10, n_k=16, TT ranks 16,
3e7 uniform draws of the multi-index with duplicates removed, noise 1e-4 * RMS,
synthetic (synth.make_problem(5)).  A "step" is one PRGD iteration (Alg. 2 loop
body: pass A, weights, orthogonalisation, pass B, projection, TT-rounding) over all
of Omega.  value = iterations per second (whole job = sum over ranks), inputs
resident in HBM; e2e = the same metric through the C-ABI from pinned host buffers
(observations uploaded + bucketed, cores in, K steps with a residual read per step,
cores out).  Prints one JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "PRGD iter/s (observed entries/s = M x iter/s) at d=10, n=16, r=16, |Omega|~3e7, fp64"
FP64_DMMA_TFS = 37.1   # measured DMMA fp64 peak (tools/fp64_peak.cu), DESIGN.md 8
UNIT = "iter/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "src": "measured", "sm_max_mhz": d.get("sm_max_mhz")}
    return {"hbm_gbs": 6650.0, "src": "fallback", "sm_max_mhz": 1965.0}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 8:
                for nm, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def algorithmic_bytes(group, m, KL, NL, NR, ld, nvrows_L, nvrows_R):
    """Compulsory DRAM bytes of one launch of a pass kernel: streamed
    per-sample arrays + each table row read once + outputs written once + plan."""
    tab = lambda N: N * ld * 8  # noqa: E731
    plan = lambda nv: nv * 20   # noqa: E731
    if group == "passA_prefix":
        return m * (4 + 8 + 8) + tab(NL) + tab(NR) + NL * 8 + plan(nvrows_L)
    if group == "passA_suffix":
        return m * (4 + 8 + 8) + NR * 8 + plan(nvrows_R)      # pos_suf, g gathered, g_suf written
    if group == "passB_prefix":
        return m * (4 + 8) + tab(NR) + tab(NL) + NL * 8 + plan(nvrows_L)
    if group == "passB_suffix":
        return m * (4 + 4 + 8) + tab(NL) + tab(NR) + NR * 8 + plan(nvrows_R)
    return None


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1:
        return 0, 1, None
    import torch
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    backend = "nccl" if args.impl == "ours" else "gloo"
    if args.impl == "ours":
        torch.cuda.set_device(local)
    dist.init_process_group(backend=backend)
    return rank, ws, dist


def run_ours(args, rank, ws, dist):
    import torch
    import synth
    import paper_2501_13385_b200 as pkg

    dev = torch.cuda.current_device()
    t0 = time.perf_counter()
    if ws > 1:
        # sharded Omega: same truth and init on every rank, disjoint samples
        pr = synth.make_problem(args.config, m=args.m, rank=rank, world=ws)
    else:
        pr = synth.make_problem(args.config, m=args.m)
    t_gen = time.perf_counter() - t0
    m_global = pr.m
    if dist is not None:
        t = torch.tensor([float(pr.m)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        m_global = int(round(float(t.item())))
    ar = pkg.torch_allreduce() if dist is not None else None
    # observations: T*(Omega) through the library (tt_eval_at), plus seeded noise
    tctx = pkg.TTContext(pr.n, pr.r)
    tctx.set_cores(pr.truth)
    clean = tctx.eval_at(pr.idx)
    tctx.close()
    y = pr.observations(clean)
    init = pr.init
    if init is None:
        # config 1 prescribes the spectral init (BASELINE.json): the library's own GPU TT-SVD
        # of p^-1 P_Omega(y) (tt_spectral_init), computed once here, outside the timed region
        sctx = pkg.TTContext(pr.n, pr.r)
        sctx.set_observations(pr.idx, y)
        sctx.spectral_init()
        init = sctx.get_cores()
        sctx.close()
    KL, NL, NR = pkg.plan(pr.n, pr.r)

    ctx = pkg.TTContext(pr.n, pr.r)
    if args.step_rule != "theory":
        ctx.set_metric("vee", 0.0, args.step_rule)
    if ar is not None:
        ctx.set_allreduce(ar, m_global)
    stream = ctx.stream
    t1 = time.perf_counter()
    ctx.set_observations(pr.idx, y)
    t_setobs = time.perf_counter() - t1
    ctx.set_cores(init)
    res0 = ctx.residual_norm()
    for _ in range(args.warmup):
        ctx.step(args.step_size)
    ctx.sync()
    st0 = ctx.stats()

    sampler = ClockSampler(dev)
    sampler.start()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        ctx.step(args.step_size)
    ev1.record(stream)
    ev1.synchronize()
    ctx.sync()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    st1 = ctx.stats()
    res1 = ctx.residual_norm()
    launches = st1["launches"] - st0["launches"]
    ms_max = ms
    if dist is not None:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())

    # dense-sweep diagnostics over one extra step: Jacobi sweeps, QR paths
    e0 = ctx.debug("eps")
    ctx.step(args.step_size)
    e1 = ctx.debug("eps")
    dd = e1 - e0
    dense_diag = {"jacobi_sweeps": int(dd[4]), "cholqr2_ok": int(dd[11]), "cholqr2_fail_first": int(dd[12])}
    # per-kernel-group durations (CUDA events on the library stream), profile mode
    ctx.set_profiling(True)
    for _ in range(args.profile_steps):
        ctx.step(args.step_size)
    prof = ctx.get_profile()
    ctx.set_profiling(False)
    ctx.close()

    out = dict(pr=pr, y=y, init=init, KL=KL, NL=NL, NR=NR, ms=ms_max, launches=launches,
               m_global=m_global,
               clocks=clocks, prof=prof, t_gen=t_gen, t_setobs=t_setobs, res0=res0, res1=res1,
               dense_diag=dense_diag)
    if not args.no_e2e:
        # three end-to-end repetitions (fresh context each), the median reported: a single
        # 20-step run is dominated by the one-time upload / bucketing and varies run to run
        reps = [run_e2e(args, pr, y, init, ar, m_global, dist) for _ in range(3)]
        reps.sort(key=lambda e: e["value"])
        out["e2e"] = dict(reps[1], reps=[round(e["value"], 3) for e in reps])
    return out


def run_e2e(args, pr, y, init, ar=None, m_global=None, dist=None):
    """Same metric through the public API from pinned host buffers: upload + bucket
    Omega, set cores, K steps each followed by a residual read (D2H), cores out."""
    import torch
    import paper_2501_13385_b200 as pkg
    idx_p = torch.from_numpy(np.ascontiguousarray(pr.idx)).pin_memory()
    y_p = torch.from_numpy(np.ascontiguousarray(y)).pin_memory()
    cores_p = [torch.from_numpy(np.ascontiguousarray(c)).pin_memory() for c in init]
    K = args.steps
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    ctx = pkg.TTContext(pr.n, pr.r)
    if args.step_rule != "theory":
        ctx.set_metric("vee", 0.0, args.step_rule)
    if ar is not None:
        ctx.set_allreduce(ar, m_global)
    ctx.set_observations(idx_p.numpy(), y_p.numpy())
    for k, c in enumerate(cores_p):
        ctx.set_core(k, c.numpy())
    for _ in range(K):
        ctx.step(args.step_size)
        ctx.residual_norm()
    cores = ctx.get_cores()
    t1 = time.perf_counter()
    ctx.close()
    if dist is not None:   # whole-job time = slowest rank
        t = torch.tensor([t1 - t0], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t0, t1 = 0.0, float(t.item())
    core_bytes = sum(c.nbytes for c in cores)
    h2d = idx_p.numel() * 4 + y_p.numel() * 8 + core_bytes
    d2h = K * 8 + core_bytes
    ws = dist.get_world_size() if dist is not None else 1
    return {"value": ws * K / (t1 - t0), "unit": UNIT, "h2d_bytes_per_step": int(h2d / K),
            "d2h_bytes_per_step": int(d2h / K), "wall_s": t1 - t0}


def oracle_sample(pr, y, init, m_sample, steps=1, warmup=0):
    """Time the oracle (as it stands) on the first m_sample entries of Omega."""
    import oracle
    idx = pr.idx[:m_sample]
    ys = y[:m_sample]
    T = [c.copy() for c in init]
    for _ in range(warmup):
        T = oracle.prgd_step(T, idx, ys, pr.n, pr.r, 1.0)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        T = oracle.prgd_step(T, idx, ys, pr.n, pr.r, 1.0)
        times.append(time.perf_counter() - t0)
    return times


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        th = [i.get("num_threads") for i in threadpool_info() if i.get("user_api") == "blas"]
        if th:
            return int(max(th))
    except Exception:
        pass
    return len(os.sched_getaffinity(0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--m", type=int, default=None, help="override |Omega| draws (debug only)")
    ap.add_argument("--step-size", type=float, default=1.0)
    ap.add_argument("--step-rule", choices=["theory", "adaptive"], default="theory",
                    help="A12 rule: theory (Thm 4.1 form, the default) or adaptive (steepest step, "
                         "PAPER.md:236-238; one more pass over Omega per step)")
    ap.add_argument("--profile-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1_000_000)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, ws, dist = dist_setup(args)

    if args.impl == "reference":
        run_reference(args, rank, ws)
        return

    r = run_ours(args, rank, ws, dist)
    if rank != 0:
        return
    pr = r["pr"]
    m = pr.m
    ms_step = r["ms"] / args.steps
    value = ws * args.steps / (r["ms"] / 1e3)
    pk = peaks()
    prof = r["prof"]
    nsteps = max(prof["steps"], 1)
    per = {k: v / nsteps for k, v in prof["ms"].items()}
    tot = sum(per.values())
    import paper_2501_13385_b200 as pkg  # noqa: F401
    ld = 2
    while ld < pr.r[r["KL"]]:
        ld *= 2
    pass_groups = ["passA_prefix", "passA_suffix", "passB_prefix", "passB_suffix"]
    dom = max(per, key=per.get)
    dom_pass = max(pass_groups, key=lambda g: per.get(g, 0.0))
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        with open(tf) as f:
            traffic = json.load(f).get(dom_pass)
    alg = algorithmic_bytes(dom_pass, m, r["KL"], r["NL"], r["NR"], ld, r["NL"], r["NR"])
    t_dom = per[dom_pass] / 1e3
    achieved = alg / t_dom / 1e9 if t_dom > 0 else 0.0
    roof = {"bound": "hbm", "kernel": dom_pass, "achieved": round(achieved, 1),
            "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
            "traffic": traffic, "peak_src": pk["src"],
            # the kernel's measured DRAM traffic (ncu, profiles/traffic.json) over its live time:
            # the gathers re-read table rows, so this exceeds the algorithmic bytes
            "dram_gbs": round(traffic / t_dom / 1e9, 1) if traffic and t_dom > 0 else None,
            "dram_frac": round(traffic / t_dom / 1e9 / pk["hbm_gbs"], 4) if traffic and t_dom > 0 else None,
            "share_of_step": round(per[dom_pass] / tot, 4) if tot else None,
            "group_ms": {k: round(v, 4) for k, v in per.items()},
            "dominant_group": dom}
    # FP64 side (SURVEY 8(d) "FP64 util vs peak"): the backward recursions are the path's dense
    # contraction (A9 as DMMA GEMMs over the table levels); algorithmic flops per level k =
    # 4 r_k n_k r_{k+1} per parent row (the O and Z products), parents = prod of the other modes
    # on that side.  Peak: DMMA measured with tools/fp64_peak.cu on this pool.
    fl = 0.0
    for k in range(pr.d):
        parents = math.prod(pr.n[:k]) if k < r["KL"] else math.prod(pr.n[k + 1:])
        fl += 4.0 * pr.r[k] * pr.n[k] * pr.r[k + 1] * parents
    t_back = per.get("backward_Y", 0.0) / 1e3
    fp64 = {"kernel": "backward_Y", "bound": "tensor (DMMA fp64)", "flops": fl,
            "achieved": round(fl / t_back / 1e12, 2) if t_back > 0 else None, "peak": FP64_DMMA_TFS,
            "unit": "TFLOP/s", "frac": round(fl / t_back / 1e12 / FP64_DMMA_TFS, 4) if t_back > 0 else None,
            "peak_src": "tools/fp64_peak.cu (mma.sync m8n8k4 f64, measured on the pool's B200)"}
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        ms_ = min(args.cpu_sample, m)
        times = oracle_sample(pr, r["y"], r["init"], ms_, steps=1)
        t = times[0]
        cpu = {"value": round((ms_ / m) / t, 6), "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
               "sample": f"one oracle PRGD step on the first {ms_} of {m} observed entries; "
                         f"value = (sample/M)/t_step (linear in |Omega|); entries/s = {ms_ / t:.3e}",
               "step_s": round(t, 3)}
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (synth.make_problem(5): Gaussian TT cores, uniform Omega, seeded)",
        "config": {"workload": f"cfg{args.config}: d={pr.d}, n={pr.n[0]}, r={max(pr.r)}, "
                               f"|Omega|={m}, noise {pr.noise_sigma} {pr.noise_kind}",
                   "d": pr.d, "n": list(pr.n), "r": list(pr.r), "m": m, "K_L": r["KL"],
                   "l2": "inputs larger than L2 (Omega arrays + tables > 126 MB); no flush",
                   "m_global": r["m_global"], "step_rule": args.step_rule,
                   "parallelism": (f"sharded Omega over {ws} GPUs (h and Y all-reduced, NCCL); "
                                   "value = N x iter/s of the N-times-larger problem") if ws > 1
                                  else "single"},
        "entries_per_s": round(r["m_global"] * args.steps / (r["ms"] / 1e3), 1),
        "roofline": roof,
        "fp64": fp64,
        "cpu_baseline": cpu,
        "e2e": r.get("e2e"),
        "gpu_launches": int(r["launches"]),
        "clocks": r["clocks"],
        "setup_s": {"generate": round(r["t_gen"], 2), "set_observations": round(r["t_setobs"], 3)},
        "residual": {"before": r["res0"], "after": r["res1"]},
        "dense_diag": r["dense_diag"],
    }
    print(json.dumps(line), flush=True)


def run_reference(args, rank, ws):
    """--impl reference: the CPU oracle (as it stands) on the box's host cores, same
    config / metric / unit; each step a bounded sample of Omega."""
    if rank != 0:
        return
    import synth
    import oracle
    pr = synth.make_problem(args.config, m=args.m)
    clean = oracle.eval_at(pr.truth, pr.idx[: args.cpu_sample])
    m_s = clean.shape[0]
    y = np.zeros(pr.m)
    y[:m_s] = pr.observations(np.concatenate([clean, np.zeros(pr.m - m_s)]))[:m_s]
    steps = max(1, min(args.steps, 3))
    times = oracle_sample(pr, y, pr.init, m_s, steps=steps, warmup=1 if args.warmup else 0)
    t = statistics.median(times)
    v = (m_s / pr.m) / t
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": UNIT,
            "n_gpus": ws, "steps": steps, "warmup": 1, "ms_per_step": round(1e3 * t * pr.m / m_s, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"cfg{args.config}", "m": pr.m},
            "cpu_baseline": {"value": round(v, 6), "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
                             "sample": f"{steps} oracle steps on the first {m_s} of {pr.m} entries, median"},
            "e2e": {"value": round(v, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
