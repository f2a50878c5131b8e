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
UNIT = "iter/s"
# FP64 peak (MEASURED_PEAKS.json has none): 148 SMs x 64 FP64 FMA lanes x 2 flop x 1.965 GHz =
# 37.2 TF/s (the guide's SM count and max clock); the mma.sync m8n8k4 f64 (DMMA) loop of
# tools/fp64_peak.cu measured 37.1 TF/s at 1965 MHz (profiles/r02_fp64_peak.md) -> 37.1 is used.
FP64_PEAK_TFS = 37.1
FP64_PEAK_SRC = "measured DMMA loop (tools/fp64_peak.cu, profiles/r02_fp64_peak.md); derived 37.2"
NCU_KERNELS = os.path.join(ROOT, "profiles", "r02_ncu_kernels.json")


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


def chain_models(pr):
    """Per-step FP64 work of the chain path's groups (SURVEY §8(d) per-sample flop model, App. X.4):
    pass A = sum_{k>=2} 2 r_{k-1} r_k + 1 per sample (the left chain), interfaces = both chains,
    contraction = sum_k 2 r_{k-1} r_k per sample; h = d adds per sample."""
    m, d, r = pr.m, pr.d, pr.r
    chain = sum(2.0 * r[k - 1] * r[k] for k in range(2, d + 1))
    contr = sum(2.0 * r[k] * r[k + 1] for k in range(d))
    return {"passA_prefix": ("fp64", m * (chain + 1), "flop"), "marginals": ("fp64", m * d, "flop"),
            "passB_prefix": ("fp64", m * 2 * chain, "flop"), "backward_Y": ("fp64", m * contr, "flop"),
            "dense_orth": group_models(pr, 1, 1, 1)["dense_orth"], "dense_round": group_models(pr, 1, 1, 1)["dense_round"]}


def group_models(pr, KL, NL, NR):
    """Algorithmic work of one launch of each kernel group per step: compulsory
    DRAM bytes for the HBM-bound groups (streamed per-sample arrays + each table row read once +
    each output written once), FP64 flops for the arithmetic groups.  Returns
    {group: (bound, units, unit_name)}."""
    m, d, n, r = pr.m, pr.d, pr.n, pr.r
    ld = lambda k: 2 if r[k] <= 2 else 1 << (r[k] - 1).bit_length()   # noqa: E731  pad(r)
    tab = lambda rows, k: rows * ld(k) * 8                             # noqa: E731
    rows_L = [math.prod(n[:k]) for k in range(KL + 1)]
    rows_R = [math.prod(n[k:]) for k in range(d + 1)]
    tables = sum(tab(rows_L[k], k) for k in range(1, KL + 1)) + sum(tab(rows_R[k], k) for k in range(KL, d))
    out = {
        "tables_C": ("hbm", tables, "B"), "tables_U": ("hbm", tables, "B"),
        "passA_prefix": ("hbm", m * (4 + 8 + 8) + tab(NL, KL) + tab(NR, KL) + NL * 8, "B"),
        "passA_suffix": ("hbm", m * (4 + 8 + 8) + NR * 8, "B"),
        "passB_prefix": ("hbm", m * (4 + 8) + tab(NR, KL) + tab(NL, KL) + NL * 8, "B"),
        "passB_suffix": ("hbm", m * (4 + 4 + 8) + tab(NL, KL) + tab(NR, KL) + NR * 8, "B"),
        "marginals": ("hbm", (NL + NR) * 8, "B"), "weights_psi": ("hbm", (NL + NR) * 8, "B"),
    }
    # backward recursions (A9 as DMMA GEMMs over the table levels): per level 4 r_k n_k r_{k+1}
    # flops per parent row (the O and Z products)
    fl = 0.0
    for k in range(d):
        parents = math.prod(n[:k]) if k < KL else math.prod(n[k + 1:])
        fl += 4.0 * r[k] * n[k] * r[k + 1] * parents
    out["backward_Y"] = ("fp64", fl, "flop")
    # dense sweeps: CholeskyQR2 of each unfolding (2 Grams + 2 triangular applies, 8 rows cols^2)
    # plus the neighbour push (2 R^2 rows); A4-A6 on r-sized cores, A10-A14 on 2r-sized blocks
    orth = 0.0
    for k in range(d - 1):
        rows, cols = r[k] * n[k], r[k + 1]
        orth += 8.0 * rows * cols ** 2 + 2.0 * cols * cols * n[k + 1] * r[k + 2] + 4.0 * rows * cols ** 2
    out["dense_orth"] = ("fp64", orth, "flop")
    rnd = 0.0
    for k in range(d):
        R0 = 1 if k == 0 else 2 * r[k]
        R1 = 1 if k == d - 1 else 2 * r[k + 1]
        rnd += 6.0 * r[k] * n[k] * r[k + 1] ** 2          # projection (solve, U^T Z, U W)
        if k > 0:
            rnd += 8.0 * n[k] * R1 * R0 ** 2 + 2.0 * R0 * R0 * n[k - 1] * (2 * r[k - 1] or 1)   # r2l QR + push
        if k < d - 1:
            rnd += 8.0 * r[k] * n[k] * R1 ** 2 + 2.0 * r[k + 1] * R1 * n[k + 1] * 2 * r[k + 2] \
                + 4.0 * R1 ** 3                                                              # l2r QR, push, Jacobi
    out["dense_round"] = ("fp64", rnd, "flop")
    return out


def stage_latency(pr, ms):
    """Latency model of the dense sweeps: 2(d-1) dependent QR / truncation stages (A14) or
    d-1 (A4-A5) + d-2 Gram steps (A6); per-stage time = group time / stages."""
    d = pr.d
    return {"dense_round": {"stages": 2 * (d - 1), "us_per_stage": round(1e3 * ms.get("dense_round", 0) / (2 * (d - 1)), 2)},
            "dense_orth": {"stages": 2 * d - 3, "us_per_stage": round(1e3 * ms.get("dense_orth", 0) / max(2 * d - 3, 1), 2)}}


def ncu_kernels():
    """Per-kernel ncu counters captured at this build (profiles/r02_ncu_kernels.json, written by
    tools/ncu_table.py from one ncu run of bench.py --profile-steps 1)."""
    if not os.path.exists(NCU_KERNELS):
        return None
    with open(NCU_KERNELS) as f:
        return json.load(f)


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
        nov = tuple(int(x) for x in args.n_override.split(",")) if args.n_override else None
        rov = ((1,) + (args.rank,) * (len(nov) - 1) + (1,)) if (nov and args.rank) else None
        pr = synth.make_problem(args.config, m=args.m, n=nov, r=rov)
    if args.rank and not args.n_override:
        # diagnostic only: the same Omega with every interior TT rank set to
        # args.rank (truth and init truncated), e.g. r = 1 for the HBM-bound shape of the passes
        pr.r = (1,) + (args.rank,) * (pr.d - 1) + (1,)
        pr.truth = [c[:pr.r[k], :, :pr.r[k + 1]].copy() for k, c in enumerate(pr.truth)]
        pr.init = [c[:pr.r[k], :, :pr.r[k + 1]].copy() for k, c in enumerate(pr.init)]
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

    ctx = pkg.TTContext(pr.n, pr.r, path=args.path)
    if args.step_rule != "theory":
        ctx.set_metric("vee", 0.0, args.step_rule)
    if ar is not None:
        ctx.set_allreduce(ar, m_global)
    stream = ctx.stream
    path = ctx.path
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

    out = dict(pr=pr, y=y, init=init, KL=KL, NL=NL, NR=NR, ms=ms_max, launches=launches, path=path,
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
    # multi-indices as bytes when every mode size allows it (tt_set_observations_u8: a quarter of
    # the int32 upload), int32 otherwise
    idt = np.uint8 if max(pr.n) <= 256 else np.int32
    idx_p = torch.from_numpy(np.ascontiguousarray(pr.idx, dtype=idt)).pin_memory()
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
    h2d = idx_p.numel() * idx_p.element_size() + y_p.numel() * 8 + core_bytes
    d2h = K * 8 + core_bytes
    ws = dist.get_world_size() if dist is not None else 1
    return {"value": ws * K / (t1 - t0), "unit": UNIT, "h2d_bytes_per_step": int(h2d / K),
            "d2h_bytes_per_step": int(d2h / K), "wall_s": t1 - t0,
            "idx_dtype": "u8" if idt is np.uint8 else "i32"}


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


def host_info():
    """CPU model, BLAS vendor / version and threads of the oracle's numpy."""
    out = {"cpu_model": None, "blas": None, "affinity_cores": len(os.sched_getaffinity(0))}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    out["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    try:
        from threadpoolctl import threadpool_info
        b = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if b:
            out["blas"] = f"{b[0].get('internal_api')} {b[0].get('version')} ({b[0].get('num_threads')} threads)"
    except Exception:
        pass
    return out


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
    ap.add_argument("--path", choices=["auto", "tables", "chains"], default="auto",
                    help="path over Omega (tt_set_path); auto = tables when they fit")
    ap.add_argument("--n-override", type=str, default=None,
                    help="diagnostic: comma-separated mode sizes with --config 5 (e.g. 16x15 as '16,...')")
    ap.add_argument("--rank", type=int, default=0,
                    help="diagnostic: override every interior TT rank (e.g. 1: HBM-bound passes)")
    ap.add_argument("--step-size", type=float, default=1.0)
    ap.add_argument("--step-rule", choices=["theory", "adaptive"], default="theory",
                    help="A12 rule: theory (Thm 4.1 form, the default) or adaptive (steepest step, "
                         "PAPER.md:236-238; one more pass over Omega per step)")
    ap.add_argument("--profile-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=2_000_000)
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
    models = chain_models(pr) if r["path"] == "chains" else group_models(pr, r["KL"], r["NL"], r["NR"])
    ncu = ncu_kernels()
    ncu_groups = (ncu or {}).get("groups", {})
    table = {}
    for g, t in per.items():
        if t <= 0 or g not in models:
            continue
        bound, units, uname = models[g]
        if bound == "hbm":
            ach, peak, unit = units / (t / 1e3) / 1e9, pk["hbm_gbs"], "GB/s"
        else:
            ach, peak, unit = units / (t / 1e3) / 1e12, FP64_PEAK_TFS, "TFLOP/s"
        ng = ncu_groups.get(g, {})
        table[g] = {"ms": round(t, 4), "share": round(t / tot, 4), "bound": bound,
                    "algorithmic": units, "algorithmic_unit": uname, "achieved": round(ach, 3),
                    "peak": peak, "unit": unit, "frac": round(ach / peak, 5),
                    "ncu_dram_bytes": ng.get("dram_bytes"), "ncu_dmma_pct": ng.get("dmma_pct"),
                    "ncu_fp64_pct": ng.get("fp64_pct")}
    dom = max(table, key=lambda g: table[g]["ms"])
    td = table[dom]
    bound = "alu" if td["bound"] == "fp64" else "hbm"
    roof = {"bound": bound, "kernel": dom, "achieved": td["achieved"], "peak": td["peak"],
            "unit": td["unit"], "frac": td["frac"], "traffic": td["ncu_dram_bytes"],
            "peak_src": (pk["src"] + " MEASURED_PEAKS.json hbm_gbs") if bound == "hbm" else FP64_PEAK_SRC,
            "share_of_step": td["share"],
            "note": ("latency-bound dependent sweeps (one 8-CTA cluster); see latency_model"
                     if dom in ("dense_round", "dense_orth") else ""),
            "latency_model": stage_latency(pr, per),
            "traffic_src": (f"{os.path.relpath(NCU_KERNELS, ROOT)} (commit {ncu.get('commit')})"
                            if ncu else None),
            "kernels": table}
    # FP64 side (SURVEY 8(d) "FP64 util vs peak"): the backward recursions (the DMMA contraction)
    bY = table.get("backward_Y", {})
    fp64 = {"kernel": "backward_Y", "bound": "tensor (DMMA fp64)", "flops": bY.get("algorithmic"),
            "achieved": bY.get("achieved"), "peak": FP64_PEAK_TFS, "unit": "TFLOP/s",
            "frac": bY.get("frac"), "ncu_dmma_pipe_pct": bY.get("ncu_dmma_pct"), "peak_src": FP64_PEAK_SRC}
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        ms_ = min(args.cpu_sample, m)
        times = oracle_sample(pr, r["y"], r["init"], ms_, steps=1)
        t = times[0]
        cpu = {"value": round((ms_ / m) / t, 6), "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
               "sample": f"one oracle PRGD step on the first {ms_} of {m} observed entries; "
                         f"value = (sample/M)/t_step (linear in |Omega|); entries/s = {ms_ / t:.3e}",
               "step_s": round(t, 3), **host_info()}
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
                   "diagnostic_rank_override": args.rank or None, "path": args.path,
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
