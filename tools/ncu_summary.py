"""Summarise ncu outputs brought back in gpurun_out/ into a markdown table.

  python tools/ncu_summary.py launches.csv [prof.ncu-rep]  > profiles/ncu_rNN.md
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0].replace("tgs::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total ms | avg us | share |", "|---|---|---|---|---|"]
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {k[:70]} | {n} | {v / 1e6:.3f} | {v / n / 1e3:.1f} | {100 * v / tot:.1f}% |")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "smsp__inst_executed.sum"]


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    idx = [(w, h.index(w)) for w in WANT if w in h]
    ki = h.index("Kernel Name")
    out = ["| kernel | " + " | ".join(f"{w} [{units[i]}]" for w, i in idx) + " |",
           "|---|" + "---|" * len(idx)]
    for r in data:
        out.append(f"| {r[ki].split('(')[0].replace('tgs::<unnamed>::', '')} | " +
                   " | ".join(r[i] for _, i in idx) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    print("## Launch list (ncu gpu__time_duration.sum, serialised, cold cache)\n")
    print(launches(sys.argv[1]))
    if len(sys.argv) > 2:
        print("\n## Full captures (ncu --set full)\n")
        print(full(sys.argv[2]))
