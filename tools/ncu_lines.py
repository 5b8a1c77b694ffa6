"""Per-source-line share of executed warp instructions and stall samples of one
.ncu-rep (captured with --import-source on and -lineinfo builds).
    python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
cur = None
hdr = None
agg = collections.defaultdict(lambda: [0, 0, ""])
for r in csv.reader(io.StringIO(raw)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        try:
            n = int(r[hdr.index("Instructions Executed")])
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        k = (cur, int(r[0]))
        agg[k][0] += n
        agg[k][1] += s
        agg[k][2] = r[1].strip()[:90]
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"# {rep}: {tot} warp instructions, {ts} stall samples")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / tot * 100:5.1f}% {v[1] / ts * 100:5.1f}% {k[0]}:{k[1]} {v[2]}")
