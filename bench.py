"""Throughput benchmark of the B200 concealment path (BASELINE.json metric:
lost 16x16 blocks concealed/sec at 1/2/4/8 B200; % roofline; vs CPU ref).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfgX] [--impl ours|reference]

A step conceals one batch of the workload (BASELINE.json config) resident in
HBM; for N > 1 (torchrun, one process per GPU) the frames are sharded by
contiguous range and the uint8 results gathered to rank 0 over NCCL inside
the timed step.  `value` is device-timed (CUDA events, barrier + synchronize
on both sides, max over ranks); `e2e` is the same metric through the C ABI
entry with host buffers (bm_conceal_host: H2D of pixels + states, D2H of the
uint8 result every step).  `--impl reference` times the CPU reference port
(oracle/, the reference itself is pure Python and cannot travel to the box)
on the host cores.  Inputs are seeded synthetic frames.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2205_11226_b200.synth import CONFIGS, make_config  # noqa: E402

METRIC = "lost 16x16 blocks concealed/sec"
UNIT = "blocks/s"
# FP64 peak: DMMA (mma.sync m8n8k4 f64) and DFMA share the SM's FP64 hardware
# (tools/pipebench.cu: mixing them does not add up); the measured ceiling is
# 36.8 TF/s DMMA, 36.2 DFMA (profiles/peaks_r01.txt) -> the roofline uses 36.8.
FP64_PEAK_TFLOPS = 36.8
FP32_PEAK_TFLOPS = 69.7  # measured FFMA peak (same run)
LAUNCHES_PER_STEP = 12   # k_init_out, k_cell_flags, 2 x CUB scan, k_slots, 2 x k_depth, k_sched_prep,
                         # k_sched_seed, k_conceal (256- and 512-thread builds; the one not serving
                         # the DAG shape returns at once), k_summary (profiles/ launch list)
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_traffic.json")  # ncu --set full dram bytes per launch

WORKLOADS = {
    # name: (cfg, profile, forced_layer)
    "cfg1": (1, "sentinel", None),
    "cfg2": (2, "efficient", None),
    "cfg3": (3, "efficient", None),
    "cfg4": (4, "sentinel", "HQL"),
    "cfg4idl": (4, "sentinel", "IDL"),  # forced IDL: the distance/weight-stage stress
    "cfg5": (5, "efficient", None),
}


def profile_of(name):
    from paper_2205_11226_b200 import Profile

    return Profile.sentinel() if name == "sentinel" else Profile.named(name)


def _gen_frame(args):
    cfg, f = args
    px, st = make_config(cfg, frames=1, first=f)
    return px[0], st[0]


def make_inputs(cfg: int, start: int, stop: int, ranks: int = 1):
    """Frames [start, stop) of config `cfg` (host numpy), generated in parallel
    (the host cores shared by the `ranks` processes of this node)."""
    from multiprocessing import Pool

    idx = list(range(start, stop))
    procs = max(1, min(len(idx), (os.cpu_count() or 1) // max(1, ranks)))
    if len(idx) <= 2 or procs == 1:
        res = [_gen_frame((cfg, f)) for f in idx]
    else:
        with Pool(procs) as pool:
            res = pool.map(_gen_frame, [(cfg, f) for f in idx])
    return np.stack([r[0] for r in res]), np.stack([r[1] for r in res])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def flush_l2(torch, buf):
    buf.add_(1)  # 256 MiB write > 126 MB L2


# ----------------------------------------------------------------- CPU baseline


def _oracle_crop(args):
    px, st, t_phi, t_nu, forced = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import oracle

    t0 = time.perf_counter()
    _, _, status, cells = oracle.conceal(px.astype(np.float64), st, t_phi, t_nu, 10.0, forced)
    return cells, time.perf_counter() - t0


def cpu_jobs(workload: str, crop: int = 384):
    """Bounded CPU sample of the workload: one crop x crop tile (multiple of 16)
    per host core, from the workload's own frames; built outside any timing."""
    cfg, prof_name, forced = WORKLOADS[workload]
    prof = profile_of(prof_name)
    forced_code = -1 if forced is None else {"BRL": 0, "IDL": 1, "HQL": 2}[forced]
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    nb = CONFIGS[cfg][0]
    px_all, st_all = make_inputs(cfg, 0, min(nb, cores))
    h, w = px_all.shape[1:]
    crop = min(crop, h // 16 * 16, w // 16 * 16)
    gy, gx = max(h // crop, 1), max(w // crop, 1)
    jobs = []
    for i in range(cores):
        f = i % px_all.shape[0]
        k = i // px_all.shape[0]
        y0 = (k % gy) * crop
        x0 = ((k // gy) % gx) * crop
        jobs.append((px_all[f, y0 : y0 + crop, x0 : x0 + crop], st_all[f, y0 : y0 + crop, x0 : x0 + crop],
                     prof.t_phi, prof.t_nu, forced_code))
    return jobs, cores, crop


def cpu_baseline(workload: str, jobs=None):
    """Oracle (plain-C FP64 port of the reference path) on all host cores over
    the bounded sample of cpu_jobs (one process per core)."""
    from multiprocessing import Pool

    from oracle import oracle

    oracle.lib()  # build once before forking
    if jobs is None:
        jobs = cpu_jobs(workload)
    jobs, cores, crop = jobs
    t0 = time.perf_counter()
    with Pool(cores) as pool:
        res = pool.map(_oracle_crop, jobs)
    wall = time.perf_counter() - t0
    cells = sum(r[0] for r in res)
    return {
        "value": cells / wall,
        "cells": int(cells),
        "wall_s": wall,
        "unit": UNIT,
        "cores": cores,
        "kind": "port",
        "sample": f"{cores} crops {crop}x{crop} of {workload} frames ({cells} lost cells), one process per core, "
                  f"plain-C FP64 oracle, {wall:.1f}s wall",
    }


def run_reference(args, rank, world):
    if rank != 0:
        return
    jobs = cpu_jobs(args.workload)
    times = []
    cells = []
    last = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        last = cpu_baseline(args.workload, jobs)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
            cells.append(last["cells"])
    value = float(np.sum(cells)) / float(np.sum(times))  # lost cells over the timed steps / their wall time
    last = dict(last, value=value)
    cfg, prof_name, forced = WORKLOADS[args.workload]
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": args.workload, "profile": prof_name, "forced_layer": forced,
                   "baseline_config": CONFIGS[cfg][:3]},
        "cpu_baseline": last,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------- ours


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg5", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = each rank conceals its own batch of the config's size (default; frames are "
                         "independent, SURVEY.md §8(e)); strong = the config's batch sharded by frame range")
    args = ap.parse_args()

    from paper_2205_11226_b200.parallel import dist_env, gather_frames, shard_range

    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_2205_11226_b200 import _native
    from paper_2205_11226_b200.profiles import conceal_batch, make_params

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg, prof_name, forced = WORKLOADS[args.workload]
    prof = profile_of(prof_name)
    n_frames = CONFIGS[cfg][0]
    if n_frames == 1:  # single-image configs: one replica per GPU
        start, stop = 0, n_frames
        scaling = "weak"
        total_frames = n_frames * world
    elif args.scaling == "strong":  # the config's batch sharded by frame range
        start, stop = shard_range(n_frames, rank, world)
        scaling = "strong"
        total_frames = n_frames
    else:  # weak: every rank conceals its own batch of the config's size (frames are independent)
        start, stop = rank * n_frames, (rank + 1) * n_frames
        scaling = "weak"
        total_frames = n_frames * world
    px_np, st_np = make_inputs(cfg, start, stop, world)
    px = torch.from_numpy(px_np).to(dev)
    st = torch.from_numpy(st_np).to(dev)
    out_u8 = torch.empty_like(px)
    l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    in_bytes = px.numel() * 2
    needs_flush = in_bytes < 2 * 126 * 1024 * 1024

    def step():
        res = conceal_batch(px, st, prof, forced_layer=forced, out_u8=out_u8, sync=False, time_kernel=True)
        if world > 1:
            gather_frames(out_u8, total_frames if n_frames > 1 else n_frames, None)  # result gather to rank 0
        return res

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    _native.kernel_times_reset()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    step_ms = []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            if needs_flush:
                flush_l2(torch, l2)
            ev0.record()
            step()
            ev1.record()
            ev1.synchronize()
            step_ms.append(ev0.elapsed_time(ev1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    kms = _native.kernel_times_ms()
    # summary of one (deterministic) step for counts / algorithmic work
    res = conceal_batch(px, st, prof, forced_layer=forced, out_u8=out_u8, sync=True)
    summ = res.summary
    local_ms = float(np.sum(step_ms))
    t = torch.tensor([local_ms], dtype=torch.float64, device=dev)
    cells = torch.tensor([float(summ["lost_cells"])], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(cells, op=dist.ReduceOp.SUM)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = float(cells.item()) / (ms_per_step / 1e3)

    # ---- e2e through the C ABI with host buffers (pinned), every step H2D + D2H
    e2e = None
    if not args.no_e2e:
        import ctypes

        lib = _native.lib()
        params = make_params(px.shape[0], px.shape[1], px.shape[2], 0, prof, 10.0, forced)
        h_px = torch.from_numpy(px_np).pin_memory()
        h_st = torch.from_numpy(st_np).pin_memory()
        h_out = torch.empty_like(h_px).pin_memory()
        summ_h = _native.Summary()
        for _ in range(max(1, args.warmup)):
            _native.check(lib.bm_conceal_host(params, h_px.data_ptr(), h_st.data_ptr(), None, h_out.data_ptr(),
                                              None, None, ctypes.byref(summ_h)))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            _native.check(lib.bm_conceal_host(params, h_px.data_ptr(), h_st.data_ptr(), None, h_out.data_ptr(),
                                              None, None, ctypes.byref(summ_h)))
        e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        e2e = {"value": float(cells.item()) * args.steps / float(e2e_s.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(h_px.numel() + h_st.numel()), "d2h_bytes_per_step": int(h_out.numel())
               + ctypes.sizeof(_native.Summary)}

    if rank == 0:
        kmean = float(np.mean(kms)) if kms else None
        flop64 = summ["flop64"]
        flop32 = summ["flop32"]
        roof = None
        if kmean:
            a64 = flop64 / (kmean * 1e-3) / 1e12
            a32 = flop32 / (kmean * 1e-3) / 1e12
            traffic = None
            try:
                with open(TRAFFIC_FILE) as fh:
                    tr = json.load(fh).get(args.workload)
                if tr and tr.get("frames") == int(px.shape[0]):  # same launch size as profiled
                    traffic = tr["dram_bytes_per_launch"]
            except (OSError, ValueError):
                pass
            roof = {
                "bound": "fp64", "achieved": a64, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": a64 / FP64_PEAK_TFLOPS, "traffic": traffic,
                "traffic_unit": "bytes per k_conceal launch (dram__bytes_read.sum + dram__bytes_write.sum, "
                                "ncu --set full, profiles/ncu_traffic.json)",
                "algorithmic_bytes_per_launch": int(px.numel() * 2 + out_u8.numel()),
                "kernel": "bm::k_conceal", "kernel_ms": kmean, "kernel_share_of_step": kmean / ms_per_step,
                "flop64_per_launch": flop64, "flop32_per_launch": flop32,
                "fp32_gate": {"achieved": a32, "peak": FP32_PEAK_TFLOPS, "frac": a32 / FP32_PEAK_TFLOPS},
                "composite_frac": a64 / FP64_PEAK_TFLOPS + a32 / FP32_PEAK_TFLOPS,
                "peak_source": "measured on this pool's B200: DMMA m8n8k4 f64 36.8 TF/s (DFMA 36.2, same FP64 "
                               "hardware), FFMA 69.7 TF/s (tools/peakbench.cu, tools/pipebench.cu; "
                               "MEASURED_PEAKS.json has HBM and bf16 only)",
            }
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                cpu = cpu_baseline(args.workload)
            except Exception as exc:  # reported, not fatal
                cpu = {"error": repr(exc)}
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "profile": prof_name, "forced_layer": forced,
                       "frames": total_frames, "height": int(px.shape[1]), "width": int(px.shape[2]),
                       "lost_cells_per_step": int(cells.item()), "patches": summ["patches"],
                       "layer_counts": summ["layer_counts"], "dag_depth": summ["max_level"],
                       "l2": "flushed (256 MiB write) between steps" if needs_flush else "inputs larger than L2",
                       "parallelism": (f"frames sharded x{world}" if scaling == "strong" else
                                       f"{n_frames} frames per rank x{world}" if n_frames > 1 else f"replicas x{world}"),
                       "conceal_build": ("512-thread CTAs, 1 cell/SM (narrow DAG)"
                                         if summ["lost_cells"] < (summ["max_level"] + 1) * 2 * torch.cuda.get_device_properties(dev).multi_processor_count
                                         else "256-thread CTAs, 2 cells/SM")},
            "gpu_launches": LAUNCHES_PER_STEP * args.steps,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
