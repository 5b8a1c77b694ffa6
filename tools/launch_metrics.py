"""Per-launch time and DRAM bytes of one step from an ncu CSV taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum.

    python tools/launch_metrics.py launches.csv [step index = 3] [n launches = 24]
"""
import collections
import csv
import sys

rows = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
which = int(sys.argv[2]) if len(sys.argv) > 2 else 3
count = int(sys.argv[3]) if len(sys.argv) > 3 else 24
d = collections.OrderedDict()
for r in csv.DictReader(rows):
    d.setdefault((r["ID"], r["Kernel Name"][:60]), {})[r["Metric Name"]] = r["Metric Value"]
items = list(d.items())
starts = [i for i, (k, _) in enumerate(items) if "preprocess_fwd" in k[1]]
for (_, name), m in items[starts[which]:starts[which] + count]:
    t = float(m.get("gpu__time_duration.sum", 0)) / 1e3
    rd = float(m.get("dram__bytes_read.sum", 0)) / 1e6
    wr = float(m.get("dram__bytes_write.sum", 0)) / 1e6
    print(f"{name:60s} {t:8.1f} us  read {rd:7.1f} MB  write {wr:7.1f} MB")
