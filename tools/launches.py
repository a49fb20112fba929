"""Per-kernel summary of an ncu --csv launch list (gpu__time_duration, dram bytes).
usage: python tools/launches.py <launches.csv>"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if not h or len(r) < len(h):
        continue
    name = r[h.index("Kernel Name")][:64]
    met = r[h.index("Metric Name")]
    val = float(r[h.index("Metric Value")].replace(",", ""))
    agg.setdefault(name, collections.defaultdict(list))[met].append(val)
for k, v in agg.items():
    t = v.get("gpu__time_duration.sum", [0])
    n = len(t)
    print(f"{k:64s} n={n:3d} avg_us={sum(t) / n / 1e3:9.1f} rdMB={sum(v.get('dram__bytes_read.sum', [0])) / n / 1e6:8.1f} "
          f"wrMB={sum(v.get('dram__bytes_write.sum', [0])) / n / 1e6:8.1f}")
