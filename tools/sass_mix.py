"""Dynamic SASS instruction mix and stall samples of one kernel from an ncu report (source page).

usage: python tools/sass_mix.py REPORT.ncu-rep [kernel-substring] [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
for b in blocks[1:]:
    rows = list(csv.reader(io.StringIO('"Kernel Name"' + b)))
    name = rows[0][1]
    if pat not in name:
        continue
    h = rows[1]
    ia, isrc, iex, ist = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), \
        h.index("Warp Stall Sampling (All Samples)")
    mix = collections.Counter()
    stall = collections.Counter()
    lines = []
    tot = 0
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        op = r[isrc].split()[0] if r[isrc].split() else "?"
        if op.startswith("@"):
            op = r[isrc].split()[1]
        op = op.split(".")[0]
        n = int(r[iex] or 0)
        s = int(r[ist] or 0)
        mix[op] += n
        stall[op] += s
        tot += n
        lines.append((s, n, r[ia], r[isrc].strip()))
    print(name)
    print(f"total warp instructions {tot}")
    for op, n in mix.most_common(top):
        print(f"  {op:10s} {n:12d} {100 * n / tot:5.1f}%  stall-samples {stall[op]}")
    reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    tot_r = collections.Counter()
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        for k in reasons:
            tot_r[k] += int(r[h.index(k)] or 0)
    print("stall reasons (all samples):", ", ".join(f"{k[6:]} {v}" for k, v in tot_r.most_common(8)))
    print("hottest instructions by stall samples (top reasons):")
    byaddr = {r[ia]: r for r in rows[2:] if len(r) > iex}
    for s, n, a, src in sorted(lines, reverse=True)[:25]:
        r = byaddr[a]
        why = sorted(((int(r[h.index(k)] or 0), k[6:]) for k in reasons), reverse=True)[:2]
        print(f"  {s:7d} {n:10d} {a[-5:]} {src[:60]:60s} {why}")
