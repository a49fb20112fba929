"""Per-instruction SASS listing (address, executions, stall samples, top stall reason) of one
kernel from an ncu report, in address order, for instructions executed >= MIN times.

usage: python tools/sass_hot.py REPORT.ncu-rep kernel-substring [MIN]"""
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
mn = int(sys.argv[3]) if len(sys.argv) > 3 else 100000
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
for b in out.split('"Kernel Name"')[1:]:
    rows = list(csv.reader(io.StringIO('"Kernel Name"' + b)))
    if pat not in rows[0][1]:
        continue
    h = rows[1]
    iex, ist = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    tot = 0
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        n = int(r[iex] or 0)
        if n < mn:
            continue
        tot += n
        s = int(r[ist] or 0)
        top = max(((int(r[h.index(k)] or 0), k[6:]) for k in reasons))
        print(f"{r[0][-5:]} {n:9d} {s:6d} {top[1] if s else '':14s} {r[1].strip()}")
    print("sum executed", tot)
    break
