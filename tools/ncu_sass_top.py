"""Top SASS instructions of an ncu source-page CSV by warp-stall samples (with stall breakdown).
usage: python tools/ncu_sass_top.py <source.csv> [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
data = rows[2:]
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
iexe = hdr.index("Instructions Executed")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[isamp] or 0) for r in data)
print(f"total samples {tot:.0f}; instructions {len(data)}")
for r in sorted(data, key=lambda r: -float(r[isamp] or 0))[:n]:
    s = float(r[isamp] or 0)
    top = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stalls), reverse=True)[:3]
    print(f"{r[ia]:>6} {100*s/tot:5.1f}% exe={r[iexe]:>10} {r[isrc][:60]:60s} " +
          " ".join(f"{k}={v:.0f}" for v, k in top if v > 0))
# opcode histogram weighted by samples
agg = {}
for r in data:
    op = r[isrc].split()[0] if r[isrc].split() else "?"
    if op.startswith("@"):
        op = r[isrc].split()[1]
    op = op.split(".")[0]
    a = agg.setdefault(op, [0.0, 0.0])
    a[0] += float(r[isamp] or 0)
    a[1] += float(r[iexe] or 0)
print("\nby opcode: samples% / executed")
for op, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"  {op:10s} {100*s/tot:5.1f}%  {e:14.0f}")
