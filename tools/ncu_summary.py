"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and a
`--set full` report exported with `ncu -i X.ncu-rep --page raw --csv` into markdown.

    python tools/ncu_summary.py launches.csv raw.csv > profiles/rNN_ncu.md
"""
import collections
import csv
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
        name = d["Kernel Name"].split("(")[0].replace("unnamed>::", "").replace("void ", "")
        agg.setdefault((name, d["Grid Size"]), []).append(v)
    return agg


def full(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    cols = ["Kernel Name", "launch__grid_size", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]
    ix = [hdr.index(c) if c in hdr else None for c in cols]
    out = []
    for r in rows[2:]:
        out.append([(r[i] + (" " + units[i] if units[i] else "")) if i is not None else "-" for i in ix])
    return cols, out


def main():
    lp = sys.argv[1]
    agg = launches(lp)
    print("## Launch list (ncu gpu__time_duration.sum, cold-cache, serialised)\n")
    print("| kernel | grid | launches | mean us | total us |")
    print("|---|---|---|---|---|")
    for (k, g), v in agg.items():
        print(f"| {k} | {g} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} |")
    if len(sys.argv) > 2:
        cols, out = full(sys.argv[2])
        print("\n## `--set full` captures\n")
        print("| " + " | ".join(c.replace("sm__", "").replace(".avg.pct_of_peak_sustained", "%")
                                for c in cols) + " |")
        print("|" + "---|" * len(cols))
        for r in out:
            r[0] = r[0].split("(")[0].replace("unnamed>::", "").replace("void ", "")
            print("| " + " | ".join(r) + " |")


if __name__ == "__main__":
    main()
