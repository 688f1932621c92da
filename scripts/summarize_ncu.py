"""Summaries for profiles/: aggregate an ncu launch list per kernel, and key metrics of a --set full report.

    python scripts/summarize_ncu.py launches <launches.csv> "<header line>"
    python scripts/summarize_ncu.py full <report.ncu-rep>
    python scripts/summarize_ncu.py json <report.ncu-rep> "<source note>"   # bench.py's roofline.traffic input
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


def as_json(path, note):
    import json
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rd = list(csv.reader(io.StringIO(out)))
    hdr, units, row = rd[0], rd[1], rd[2]

    def val(name, scale_units):
        i = hdr.index(name)
        return float(row[i].replace(",", "")) * scale_units.get(units[i], 1.0)

    byte_u = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    time_u = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    dram = val("dram__bytes_read.sum", byte_u) + val("dram__bytes_write.sum", byte_u)
    ms = val("gpu__time_duration.sum", time_u)
    print(json.dumps({
        "kernel": row[hdr.index("Kernel Name")],
        "dram_bytes": dram, "duration_ms": ms, "dram_gbs": dram / (ms * 1e-3) / 1e9,
        "fp64_pipe_pct": val("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", {}),
        "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active", {}),
        "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active", {}),
        "source": note}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "json":
        as_json(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2])
