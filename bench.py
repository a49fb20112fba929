#!/usr/bin/env python
"""Benchmark of the bnfft hot path (Algorithm 2 of arXiv 2502.07155) on B200.

One step = one pass of the whole hot path over one batch of synthetic input, in the C ABI:
  bnfft_precompute   step 0(a)  psi^ table                     (row a2)
  bnfft_set_nodes    row a1     validate + stable bin sort + sorted node copy
  bnfft_execute      rows a3, a4, a6: deconvolution/zero-pad, cuFFT iFFT, gather
Inputs (nodes, spectrum) are resident in HBM when the timed region starts; the working set
(~0.7 GiB for cfg2) exceeds the 126 MB L2, so no explicit flush is done between steps.

Workload (N=1): BASELINE.json configs[1] = cfg2, d=1, M=2^20, sigma=2 (L=2^21), m=8, N=2^24
uniform nodes, complex-normal spectrum; default sinh window, complex64 (--prec/--window select
the other runs of that config).  N>1 (torchrun): every rank runs the same per-GPU workload on
its own node shard (weak scaling, no data-path collective: "replicas only").

`--impl reference` times the CPU oracle (oracle/, float64 numpy) on the same workload: steps
0(a)-2 at full size plus step 3 on a bounded node sample, extrapolated to N (see "sample").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402



def gather_kernel_name(bn, info):
    """The gather kernel the library dispatches for this plan (bnfft_info.gather_kernel)."""
    return bn.GATHER_KERNELS.get(int(info.gather_kernel), "unknown")


FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback (only if MEASURED_PEAKS.json is absent)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="bnfft", choices=["bnfft", "reference"])
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--prec", default=None, choices=[None, "c64", "c128"])
    ap.add_argument("--window", default=None, choices=[None, "sinh", "gauss", "ckb"])
    ap.add_argument("--N", type=int, default=None, help="override node count (testing only)")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        mp = json.load(open(path))
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", mp
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)", {}


def workload(args):
    cfg = synth.CONFIGS[args.cfg]
    prec = args.prec or ("c64" if "c64" in cfg.precs else cfg.precs[0])
    window = args.window or cfg.windows[0]
    if args.N:
        cfg = cfg.scaled(N=args.N)
    return cfg, prec, window


def describe(cfg, prec, window):
    L = 2 * math.ceil(math.ceil(cfg.sigma * cfg.M) / 2)
    return {
        "workload": f"cfg{cfg.cfg_id} (BASELINE configs[{cfg.cfg_id - 1}]): d={cfg.d} M={cfg.M} "
                    f"sigma={cfg.sigma:g} (L={L}) m={cfg.m} N={cfg.N} batch={cfg.batch} "
                    f"{window} {prec}, nodes {cfg.nodes}",
        "d": cfg.d, "M": cfg.M, "sigma": cfg.sigma, "L": L, "m": cfg.m, "N": cfg.N,
        "batch": cfg.batch, "window": window, "prec": prec, "nodes": cfg.nodes,
        "l2": "no flush: per-step working set (nodes 8dN B, sort buffers 16N B, sorted nodes, "
              "outputs, grids) exceeds the 126 MB L2",
    }


# ----------------------------------------------------------------------------- clocks (NVML)
class ClockSampler:
    def __init__(self, device_index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU oracle arm
def oracle_step(cfg, prec, window, x, fh, sample):
    """Oracle steps 0(a)-2 at full size, step 3 on `sample` nodes; returns (t02, t3)."""
    import oracle as O
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):
        L = O.grid_length(cfg.M, cfg.sigma)
        shape = O.default_shape(window, cfg.m, cfg.M, L)
        t0 = time.perf_counter()
        tab = O.psihat_table(window, cfg.M, cfg.m, L, shape)
        th_hat = O.step1_deconvolve_pad(fh.astype(np.complex128), O.psihat_multi(tab, cfg.d), L)
        theta = O.step2_inverse_fft(th_hat)
        t1 = time.perf_counter()
        O.step3_short_sums(theta, x[:sample], window, cfg.m, shape)
        t2 = time.perf_counter()
    return t1 - t0, t2 - t1


def cpu_sample_size(cfg):
    per_node_taps = (2 * cfg.m + 1) ** cfg.d * cfg.batch
    return int(max(1024, min(cfg.N, 4.5e6 // per_node_taps)))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg, prec, window = workload(args)
    x = synth.make_nodes(cfg)
    fh = synth.make_spectrum(cfg, prec=prec)
    S = cpu_sample_size(cfg)
    vals, times = [], []
    for it in range(args.warmup + args.steps):
        t02, t3 = oracle_step(cfg, prec, window, x, fh, S)
        est = t02 + t3 * cfg.N / S
        if it >= args.warmup:
            vals.append(cfg.N * cfg.batch / est)
            times.append(est)
    v = statistics.mean(vals)
    sample = (f"oracle (numpy float64, 1 thread) steps 0(a)-2 at full size, step 3 on the first "
              f"{S} of {cfg.N} nodes; per-step time extrapolated as t_0-2 + t_3*N/{S}")
    line = {
        "impl": "reference", "metric": "nonequispaced evaluations/sec (nodes/s)", "value": v,
        "unit": "nodes/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth/)",
        "config": describe(cfg, prec, window),
        "cpu_baseline": {"value": v, "unit": "nodes/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "nodes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
def gather_bytes_per_node(cfg, prec):
    """Algorithmic HBM bytes of one gather launch per node: sorted node
    (8d B), permutation (4 B), output (batch x 8|16 B), and the theta grid read once
    (batch L^d x 8|16 B / N)."""
    cs = 16 if prec == "c128" else 8
    L = 2 * math.ceil(math.ceil(cfg.sigma * cfg.M) / 2)
    return 8 * cfg.d + 4 + cfg.batch * cs + cfg.batch * (L ** cfg.d) * cs / cfg.N


def time_variant(torch, bn, cfg, prec, window, x_dev, fh_dev, steps, warmup, stream, device):
    plan = bn.Plan(cfg.d, cfg.M, cfg.sigma, cfg.m, window, prec, batch=cfg.batch, timing=True,
                   device=device, stream=stream.cuda_stream)
    out = torch.empty((cfg.batch, cfg.N), dtype=plan.cdtype, device=x_dev.device)

    def step():
        plan.precompute()
        plan.set_nodes(x_dev)
        plan.execute(fh_dev, out)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    plan.reset_timing()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    return plan, out, step, e0, e1


def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    from paper_2502_07155_b200 import bnfft as bn
    from paper_2502_07155_b200 import shard

    cfg, prec, window = workload(args)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    x_np = synth.make_nodes(cfg, variant=rank)
    fh_np = synth.make_spectrum(cfg, prec=prec)
    x_dev = torch.from_numpy(x_np).to(dev)
    fh_dev = torch.from_numpy(fh_np).to(dev)

    sampler = ClockSampler(local)
    sampler.start()        # samples from the warm-up on, through the timed region
    plan, out, step, e0, e1 = time_variant(torch, bn, cfg, prec, window, x_dev, fh_dev,
                                           args.steps, args.warmup, stream, local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if world > 1:
        dist.barrier()
    ms_total = shard.max_over_ranks(e0.elapsed_time(e1), device=dev)
    ms_step = ms_total / args.steps
    tm = plan.timing()
    info = plan.info()
    K = args.steps
    stages = {k: getattr(tm, "ms_" + k) / K for k in
              ("psihat", "keys", "sort", "build", "deconv", "fft", "gather")}
    launches = int(tm.kernel_launches)
    value = shard.aggregate_rate(cfg.N * cfg.batch, world, ms_step)

    line = None
    if rank == 0:
        hbm, hbm_src, mp = peaks()
        bpn = gather_bytes_per_node(cfg, prec)
        g_ms = stages["gather"]
        achieved = bpn * cfg.N / (g_ms * 1e-3) / 1e9
        traffic = None
        kname = gather_kernel_name(bn, info)
        tpath = os.path.join(ROOT, "profiles", f"ncu_gather_cfg{cfg.cfg_id}_{window}_{prec}.json")
        if os.path.exists(tpath):
            try:
                tj = json.load(open(tpath))
                # only a capture of the kernel this build dispatches counts
                if kname.split("::")[-1] in tj.get("kernel", ""):
                    traffic = tj.get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        line = {
            "metric": "nonequispaced evaluations/sec (nodes/s)",
            "value": value, "unit": "nodes/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64" if prec == "c128" else "f32",
            "data": "synthetic (seeded, synth/; BASELINE configs recipe)",
            "config": dict(describe(cfg, prec, window), parallelism=f"replicas{world}"),
            "roofline": {"bound": "hbm", "kernel": kname,
                         "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "bytes_per_node": bpn, "peak_source": hbm_src,
                         "gather_ms": g_ms},
            "stages_ms": stages,
            "gather_nodes_per_s": cfg.N * cfg.batch / (g_ms * 1e-3) if g_ms > 0 else None,
            "gpu_launches": launches,
            "clocks": clocks,
            "plan": {"L": info.L, "shape": info.shape, "nbins": info.nbins,
                     "bin_log2": list(info.bin_log2)[: cfg.d], "sort_passes": info.sort_passes,
                     "flatness": info.flatness},
        }

    # ---- e2e through the host-buffer C-ABI call (pinned host memory)
    if not args.no_e2e:
        xh = torch.from_numpy(x_np).pin_memory()
        fhh = torch.from_numpy(fh_np).pin_memory()
        fo = torch.empty((cfg.batch, cfg.N), dtype=plan.cdtype).pin_memory()
        for _ in range(max(1, args.warmup // 2)):
            plan.precompute()
            plan.transform_host(xh, fhh, fo)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(K):
            plan.precompute()
            plan.transform_host(xh, fhh, fo)
        b.record(stream)
        torch.cuda.synchronize()
        ems = shard.max_over_ranks(a.elapsed_time(b) / K, device=dev)
        if rank == 0:
            line["e2e"] = {"value": shard.aggregate_rate(cfg.N * cfg.batch, world, ems), "unit": "nodes/s",
                           "ms_per_step": ems,
                           "h2d_bytes_per_step": int(xh.numel() * 8 + fhh.numel() * fhh.element_size()),
                           "d2h_bytes_per_step": int(fo.numel() * fo.element_size()),
                           "api": "bnfft_transform_host (pinned host buffers)"}
    plan.close()

    # ---- other runs of the same config (context; the headline is the line's own workload)
    if rank == 0 and not args.no_variants and args.cfg == 2 and args.N is None:
        var = {}
        for vp, vw in (("c64", "sinh"), ("c128", "sinh"), ("c64", "gauss"), ("c128", "gauss")):
            if (vp, vw) == (prec, window):
                continue
            fh_v = torch.from_numpy(synth.make_spectrum(cfg, prec=vp)).to(dev)
            p2, _, st2, a2, b2 = time_variant(torch, bn, cfg, vp, vw, x_dev, fh_v, 10, 3, stream, local)
            a2.record(stream)
            for _ in range(10):
                st2()
            b2.record(stream)
            torch.cuda.synchronize()
            t2 = p2.timing()
            var[f"{vw}-{vp}"] = {"nodes_per_s": cfg.N / (a2.elapsed_time(b2) / 10 * 1e-3),
                                 "gather_ms": t2.ms_gather / 10}
            p2.close()
        line["variants"] = var
        # fixed nodes, repeated transforms (paper step 0(b), BNFFT_PRECOMPUTE_PSI): execute-only rates
        rep = {}
        for rp in ("c64", "c128"):
            fh_r = torch.from_numpy(synth.make_spectrum(cfg, prec=rp)).to(dev)
            for name, kw in (("default", {}), ("precompute_psi", {"precompute_psi": True})):
                p3 = bn.Plan(cfg.d, cfg.M, cfg.sigma, cfg.m, window, rp, batch=cfg.batch, timing=True,
                             device=local, stream=stream.cuda_stream, **kw)
                out3 = torch.empty((cfg.batch, cfg.N), dtype=p3.cdtype, device=dev)
                p3.set_nodes(x_dev)
                for _ in range(3):
                    p3.execute(fh_r, out3)
                torch.cuda.synchronize()
                t_set = p3.timing()
                p3.reset_timing()
                a3, b3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a3.record(stream)
                for _ in range(20):
                    p3.execute(fh_r, out3)
                b3.record(stream)
                torch.cuda.synchronize()
                t3 = p3.timing()
                rep[f"{name}-{rp}"] = {"execute_nodes_per_s": cfg.N / (a3.elapsed_time(b3) / 20 * 1e-3),
                                       "gather_ms": t3.ms_gather / 20,
                                       "set_nodes_ms": t_set.ms_keys + t_set.ms_sort + t_set.ms_build}
                p3.close()
                del out3
        line["repeated_execute"] = rep

    # ---- CPU oracle on this box's host cores (rank 0, N=1 only)
    if rank == 0 and world == 1 and not args.no_cpu:
        S = cpu_sample_size(cfg)
        t02, t3 = oracle_step(cfg, prec, window, x_np, fh_np, S)
        est = t02 + t3 * cfg.N / S
        line["cpu_baseline"] = {
            "value": cfg.N * cfg.batch / est, "unit": "nodes/s", "cores": 1, "kind": "oracle",
            "sample": f"oracle (numpy float64, 1 thread): steps 0(a)-2 at full size "
                      f"({t02:.2f} s), step 3 on the first {S} of {cfg.N} nodes ({t3:.2f} s), "
                      f"extrapolated to N"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
