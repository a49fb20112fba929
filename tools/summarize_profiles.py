"""Copy bench lines and summarise ncu captures from gpurun_out/ into profiles/ (tag = round/version).

usage: python tools/summarize_profiles.py TAG
expects gpurun_out/TAG_bench.json, TAG_bench_cfg{3,4,5}.json, TAG_launches.csv,
        TAG_gather_cfg2.ncu-rep, TAG_gather_cfg4.ncu-rep (any may be missing)."""
import csv
import json
import os
import shutil
import subprocess
import sys

tag = sys.argv[1]
src, dst = "gpurun_out", "profiles"


def last_json_line(path):
    for line in reversed(open(path).read().strip().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    return None


for name in ["bench", "bench_reference"] + [f"bench_cfg{c}" for c in (3, 4, 5)]:
    p = os.path.join(src, f"{tag}_{name}.json")
    if os.path.exists(p):
        d = last_json_line(p)
        json.dump(d, open(os.path.join(dst, f"{tag}_{name}.json"), "w"), indent=1)

p = os.path.join(src, f"{tag}_launches.csv")
if os.path.exists(p):
    shutil.copy(p, os.path.join(dst, f"{tag}_launches_cfg2.csv"))
    rows = list(csv.reader(open(p)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[h], rows[h + 1:]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    K = {}
    for r in data:
        K.setdefault(r[ii], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    agg = {}
    for v in K.values():
        n = v["name"].split("(")[0].replace("void ", "")
        a = agg.setdefault(n, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += v.get("gpu__time_duration.sum", 0)
        a[2] += v.get("dram__bytes_read.sum", 0)
        a[3] += v.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    lines = ["ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none (cold-cache, serialised launches; compare shares)",
             "command: python bench.py --steps 2 --warmup 1 --no-variants --no-cpu --no-e2e (cfg2 sinh c64)",
             f"{'kernel':60s} {'n':>3s} {'time_us':>10s} {'share':>6s} {'dram_rd_MB':>10s} {'dram_wr_MB':>10s}"]
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{n[:60]:60s} {a[0]:3d} {a[1] / 1e3:10.1f} {100 * a[1] / tot:5.1f}% "
                     f"{a[2] / 1e6:10.1f} {a[3] / 1e6:10.1f}")
    open(os.path.join(dst, f"{tag}_launches_cfg2_summary.txt"), "w").write("\n".join(lines) + "\n")

want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for cfg, algo in (("cfg2", 21 * 16777216), ("cfg4", 52 * (1 << 26))):
    p = os.path.join(src, f"{tag}_gather_{cfg}.ncu-rep")
    if not os.path.exists(p):
        continue
    out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hh, units, v = r[0], r[1], r[2]
    res = {"kernel": v[hh.index("Kernel Name")], "source": f"ncu --set full --clock-control none ({p})"}
    scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
    for k in want:
        if k in hh:
            val = float(v[hh.index(k)].replace(",", ""))
            u = units[hh.index(k)]
            res[k] = val * scale.get(u, 1.0) if "bytes" in k else val
            res[k + ".unit"] = "byte" if "bytes" in k else u
    res["dram_bytes_per_launch"] = res.get("dram__bytes_read.sum", 0) + res.get("dram__bytes_write.sum", 0)
    res["algorithmic_bytes_per_launch"] = algo
    json.dump(res, open(os.path.join(dst, f"{tag}_ncu_gather_{cfg}.json"), "w"), indent=1)
    if cfg == "cfg2":
        json.dump(res, open(os.path.join(dst, "ncu_gather_cfg2_sinh_c64.json"), "w"), indent=1)
    if cfg == "cfg4":
        json.dump(res, open(os.path.join(dst, "ncu_gather_cfg4_sinh_c64.json"), "w"), indent=1)
print("ok", tag)
