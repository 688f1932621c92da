"""Per-source-line warp-stall samples and executed instructions of an ncu report
(--set full --import-source on, kernels built with -lineinfo).

    python scripts/ncu_source_lines.py <report.ncu-rep> [top_n]
"""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname, hdr = "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        i_s, i_i = hdr.index("# Samples"), hdr.index("Instructions Executed")
        i_bar, i_wait = hdr.index("stall_barrier"), hdr.index("stall_wait")
        continue
    if hdr is None or not r[0].isdigit() or len(r) <= i_wait or not r[i_s].isdigit():
        continue
    rows.append((fname, r[0], r[1].strip(), int(r[i_s]), int(r[i_i] or 0), int(r[i_bar] or 0),
                 int(r[i_wait] or 0)))
tot_s = sum(r[3] for r in rows)
tot_i = sum(r[4] for r in rows)
byf = defaultdict(lambda: [0, 0])
for f, _, _, s, i, _, _ in rows:
    byf[f][0] += s
    byf[f][1] += i
for f, (s, i) in sorted(byf.items(), key=lambda kv: -kv[1][0]):
    print(f"{f:40s} samples {100 * s / tot_s:5.1f}% inst {100 * i / max(tot_i, 1):5.1f}%")
print("--- top lines by samples")
for f, ln, src, s, i, b, w in sorted(rows, key=lambda r: -r[3])[:top]:
    print(f"{f[:10]:10s}:{ln:>5s} S {100 * s / tot_s:5.1f}% I {100 * i / max(tot_i, 1):5.1f}% "
          f"bar {100 * b / tot_s:4.1f} wait {100 * w / tot_s:4.1f} | {src[:90]}")
