"""Copy a measurement lease's results (tools/gpu_measure.sh -> gpurun_out/) into profiles/ and
print the markdown tables of profiles/r02_configs.md and profiles/r02_ncu_step.md.

    python tools/profiles_refresh.py            (after tools/ncu_table.py wrote r02_ncu_kernels.json)
"""
import json
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def line(name):
    path = os.path.join(G, name)
    if not os.path.exists(path):
        return None
    for ln in open(path):
        if ln.startswith("{"):
            return json.loads(ln)
    return None


for src, dst in (("bench.log", "r02_bench_cfg5.json"), ("bench_r1.log", "r02_bench_r1_diag.json")):
    j = line(src)
    if j:
        json.dump(j, open(os.path.join(P, dst), "w"), indent=1)
for src, dst in (("fp64_peak.log", "r02_fp64_peak.log"), ("fp64_clocks.csv", "r02_fp64_clocks.csv"),
                 ("launches.csv", "r02_launches.csv")):
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))

print("| config | |Omega| | iter/s | ms/step | observed entries/s | three largest groups (ms) |")
print("|---|---|---|---|---|---|")
rows = [("1", "bench_cfg1.log"), ("1 adaptive", "bench_cfg1_ad.log"), ("2", "bench_cfg2.log"),
        ("2 adaptive", "bench_cfg2_ad.log"), ("3 (step 0.5)", "bench_cfg3.log"), ("3 adaptive", "bench_cfg3_ad.log"),
        ("4", "bench_cfg4.log"), ("4 adaptive", "bench_cfg4_ad.log"), ("5", "bench.log"),
        ("5 adaptive", "bench_cfg5_ad.log"), ("6 (QST shape)", "bench_cfg6.log"), ("6 adaptive", "bench_cfg6_ad.log"),
        ("5, r = 1 (HBM diagnostic)", "bench_r1.log")]
for name, f in rows:
    j = line(f)
    if not j:
        continue
    k = j["roofline"]["kernels"]
    top = sorted(k.items(), key=lambda kv: -kv[1]["ms"])[:3]
    m = j["config"]["m"]
    print(f"| {name} | {m:,} | {j['value']:.1f} | {j['ms_per_step']:.3f} | {j['value'] * m:.3g} | "
          + ", ".join(f"{n} {v['ms']:.3f}" for n, v in top) + " |")
print()
nk = json.load(open(os.path.join(P, "r02_ncu_kernels.json")))
print("| group | launches | ncu time (us) | DRAM MB | DMMA pipe % | FP64 pipe % |")
print("|---|---|---|---|---|---|")
for g, a in nk["groups"].items():
    print(f"| {g} | {a['launches']} | {a['time_ns'] / 1e3:.1f} | {a['dram_bytes'] / 1e6:.1f} | "
          f"{a['dmma_pct']:.1f} | {a['fp64_pct']:.1f} |")
