"""Summaries for profiles/: aggregate an ncu launch list per kernel, and key metrics of a --set full report.

    python scripts/summarize_ncu.py launches <launches.csv> "<header line>"
    python scripts/summarize_ncu.py full <report.ncu-rep>
"""
import csv, io, subprocess, sys
from collections import defaultdict


def launches(path, header):
    rows = [l for l in open(path) if l.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(rows)))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r["Metric Unit"], 1.0)
        name = r["Kernel Name"].split("(")[0]
        tot[name] += v * scale
        cnt[name] += 1
    T = sum(tot.values())
    print(f"# {header}")
    print("# gpu__time_duration.sum, --clock-control none (cold-cache, serialised; compare shares)")
    print(f"# total kernel time {T:.3f} ms over {sum(cnt.values())} launches")
    print("kernel,launches,total_ms,share")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k},{cnt[k]},{tot[k]:.3f},{tot[k] / T:.4f}")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
           "launch__block_size", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rd = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rd[0], rd[1], rd[2:]
    idx = [hdr.index(m) for m in METRICS if m in hdr]
    print("# columns: " + ", ".join(f"{hdr[i]} [{units[i]}]" for i in idx))
    for row in data:
        print(row[hdr.index("Kernel Name")] + "," + ",".join(row[i] for i in idx))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2])
