"""Per-kernel ncu counters of one profiled PRGD step -> profiles/<out>.json.

    python tools/ncu_table.py gpurun_out/ncu_step.csv profiles/r02_ncu_kernels.json [commit]

Input: `ncu --csv --page raw` (or --metrics ... --csv) output of tools/ncu_step.py.  Kernels are
assigned to bench.py's groups by launch order within the step (update graph first, then the
evaluate graph of the new iterate: api.cu)."""
import csv
import json
import sys
from collections import OrderedDict

METRICS = {"gpu__time_duration.sum": "time_ns", "dram__bytes_read.sum": "dram_read",
           "dram__bytes_write.sum": "dram_write",
           "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed": "dmma_pct",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed": "fp64_pct",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.sum": "dmma_inst",
           "lts__t_sector_hit_rate.pct": "l2_hit_pct",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct"}


def load(path):
    rows = OrderedDict()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for row in rd:
        if row.get("Metric Name"):          # --metrics long format
            key = (row["ID"], row["Kernel Name"])
            ent = rows.setdefault(key, {"kernel": row["Kernel Name"]})
            name = METRICS.get(row["Metric Name"])
            if name:
                unit = row.get("Metric Unit", "")
                v = float(row["Metric Value"].replace(",", ""))
                if unit in ("Kbyte", "KB"):
                    v *= 1e3
                elif unit in ("Mbyte", "MB"):
                    v *= 1e6
                elif unit in ("Gbyte", "GB"):
                    v *= 1e9
                elif unit == "usecond":
                    v *= 1e3
                elif unit == "msecond":
                    v *= 1e6
                ent[name] = v
    return list(rows.values())


def group_of(seq):
    """Launch-order state machine over one step (api.cu: update graph, then evaluate graph)."""
    out, phase, nseg = [], "pre", 0
    for ent in seq:
        k = ent["kernel"]
        if "k_orth_cs" in k or "k_dense_orth" in k:
            phase, g = "orth", "dense_orth"
        elif phase in ("pre",) and ("k_weights" in k or "k_psi" in k or "k_set_step" in k):
            g = "weights_psi"
        elif "k_tab" in k or "k_table" in k:
            g = "tables_U" if phase in ("orth", "tabU") else "tables_C"
            phase = "tabU" if phase in ("orth", "tabU") else "tabC"
        elif "k_flat_gsq" in k or "k_sum_slices" in k or ("k_flat_fix" in k and phase == "passA_sfx"):
            phase, g = "passA_sfx", "passA_suffix"   # sliced pass A suffix (gather, fix-up, slice sum)
        elif "k_flat" in k:                        # pass A prefix (flat SDDMM + fix-up)
            phase, nseg, g = "passA", 1, "passA_prefix"
        elif "k_seg" in k or "k_spmm_pipe" in k:
            if phase == "tabU" or phase == "passB":
                if "k_seg_fix" not in k:
                    nseg += 1
                g = "passB_prefix" if nseg <= 1 else "passB_suffix"
                phase = "passB"
            else:
                if phase != "passA":
                    nseg = 0
                phase = "passA"
                if "k_seg_fix" not in k:
                    nseg += 1
                g = "passA_prefix" if nseg <= 1 else "passA_suffix"
        elif any(x in k for x in ("k_back", "k_zreduce", "k_Y", "k_E_down", "k_F_up", "k_jsplit")):
            phase, g = "back", "backward_Y"
        elif "k_project" in k or "k_round" in k or "k_dense_round" in k or "k_unweight" in k:
            phase, g = "round", "dense_round"
        elif "k_marg" in k or "k_gather_sq" in k or "k_sumsq" in k:
            g = "marginals"
        elif "k_chain" in k or "k_piece" in k:
            g = "chains"
        elif "k_stack" in k or "k_concat" in k or "k_vsum" in k or "k_adapt" in k:
            g = "adaptive_step"
        else:
            g = "other"
        out.append(g)
    return out


def main():
    src, dst = sys.argv[1], sys.argv[2]
    commit = sys.argv[3] if len(sys.argv) > 3 else None
    seq = load(src)
    groups = group_of(seq)
    agg = OrderedDict()
    for ent, g in zip(seq, groups):
        ent["group"] = g
        a = agg.setdefault(g, {"launches": 0, "time_ns": 0.0, "dram_bytes": 0.0, "dmma_inst": 0.0,
                               "_w": 0.0, "_dm": 0.0, "_fp": 0.0})
        a["launches"] += 1
        t = ent.get("time_ns", 0.0)
        a["time_ns"] += t
        a["dram_bytes"] += ent.get("dram_read", 0.0) + ent.get("dram_write", 0.0)
        a["dmma_inst"] += ent.get("dmma_inst", 0.0)
        a["_w"] += t
        a["_dm"] += t * ent.get("dmma_pct", 0.0)
        a["_fp"] += t * ent.get("fp64_pct", 0.0)
    for a in agg.values():
        w = a.pop("_w") or 1.0
        a["dmma_pct"] = round(a.pop("_dm") / w, 3)      # time-weighted over the group's launches
        a["fp64_pct"] = round(a.pop("_fp") / w, 3)
    json.dump({"commit": commit, "source": src, "kernels": seq, "groups": agg}, open(dst, "w"), indent=1)
    for g, a in agg.items():
        print(f"{g:14s} launches {a['launches']:3d}  {a['time_ns'] / 1e3:9.1f} us  "
              f"DRAM {a['dram_bytes'] / 1e6:9.1f} MB  DMMA {a['dmma_pct']:5.1f}%  FP64 {a['fp64_pct']:5.1f}%")


if __name__ == "__main__":
    main()
