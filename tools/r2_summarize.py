"""Copy a round-2 capture (tools/r2_capture.sh TAG) from gpurun_out/ into profiles/: bench lines,
launch lists with per-kernel summaries, and key ncu metrics of the captured kernels.
usage: python tools/r2_summarize.py TAG"""
import collections
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


for name in ("bench", "bench_reference"):
    p = os.path.join(src, f"{tag}_{name}.json")
    if os.path.exists(p) and last_json_line(p):
        json.dump(last_json_line(p), open(os.path.join(dst, f"{tag}_{name}.json"), "w"), indent=1)
for f in ("tests.log", "smi.txt"):
    p = os.path.join(src, f"{tag}_{f}")
    if os.path.exists(p):
        shutil.copy(p, os.path.join(dst, f"{tag}_{f}"))

for cfg in ("cfg4", "cfg2"):
    p = os.path.join(src, f"{tag}_launches_{cfg}.csv")
    if not os.path.exists(p):
        continue
    shutil.copy(p, os.path.join(dst, f"{tag}_launches_{cfg}.csv"))
    rows = list(csv.reader(open(p)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[h], rows[h + 1:]
    ki, mi, vi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value"))
    agg = collections.OrderedDict()
    for r in data:
        if len(r) < len(hdr):
            continue
        agg.setdefault(r[ki][:90], collections.defaultdict(list))[r[mi]].append(float(r[vi].replace(",", "")))
    lines = [f"{'kernel':90s} {'n':>3s} {'avg_us':>9s} {'rd_MB':>9s} {'wr_MB':>9s}"]
    for k, v in agg.items():
        t = v.get("gpu__time_duration.sum", [0])
        n = len(t)
        lines.append(f"{k:90s} {n:3d} {sum(t) / n / 1e3:9.1f} {sum(v.get('dram__bytes_read.sum', [0])) / n / 1e6:9.1f} "
                     f"{sum(v.get('dram__bytes_write.sum', [0])) / n / 1e6:9.1f}")
    open(os.path.join(dst, f"{tag}_launches_{cfg}_summary.txt"), "w").write("\n".join(lines) + "\n")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
for name in ("gather_cfg4", "sort_cfg4", "gather_cfg2", "gather_cfg3"):
    rep = os.path.join(src, f"{tag}_{name}.ncu-rep")
    if not os.path.exists(rep):
        continue
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        continue
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")], "metrics": {}}
    for k in KEYS:
        if k in hdr:
            d["metrics"][k] = vals[hdr.index(k)] + " " + units[hdr.index(k)]
    json.dump(d, open(os.path.join(dst, f"{tag}_ncu_{name}.json"), "w"), indent=1)
    print(name, json.dumps(d)[:400])
