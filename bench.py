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

BUILD_LABEL = {"256": "256-thread CTAs, 2 cells/SM", "512": "512-thread CTAs, 1 cell/SM (narrow DAG)",
               "cluster": "2-CTA clusters of 512 threads per cell (narrow DAG)"}
METRIC = "lost 16x16 blocks concealed/sec"
UNIT = "blocks/s"
# FP64 peak: DMMA (mma.sync m8n8k4 f64) and DFMA share the SM's FP64 hardware
# (tools/pipebench.cu: mixing them does not add up); the measured ceiling is
# 36.8 TF/s DMMA, 36.2 DFMA (profiles/peaks_r01.txt) -> the roofline uses 36.8.
FP64_PEAK_TFLOPS = 36.8
FP32_PEAK_TFLOPS = 69.7  # measured FFMA peak (same run)
LAUNCHES_PER_STEP = 14   # k_init_out, k_cell_flags, 2 x CUB scan, k_slots, 2 x k_depth, k_sched_prep, k_postab,
                         # k_sched_seed, k_conceal x 3 (256-thread, 512-thread and 2-CTA cluster builds; the
                         # two not serving the DAG shape return at once), k_summary (profiles/ launch list)
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


def host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def cpu_jobs(workload: str, crop: int = 384):
    """Bounded CPU sample of the workload: one crop x crop tile (multiple of 16)
    per host core from the workload's own frames, at crop positions spread
    over the whole frame (a seeded draw per core, not only the corner where
    the support areas are clipped); built outside any timing."""
    cfg, prof_name, forced = WORKLOADS[workload]
    prof = profile_of(prof_name)
    forced_code = -1 if forced is None else {"BRL": 0, "IDL": 1, "HQL": 2}[forced]
    cores = host_cores()
    nb = CONFIGS[cfg][0]
    px_all, st_all = make_inputs(cfg, 0, min(nb, cores))
    h, w = px_all.shape[1:]
    crop = min(crop, h // 16 * 16, w // 16 * 16)
    gy, gx = max((h - crop) // 16 + 1, 1), max((w - crop) // 16 + 1, 1)  # 16-aligned crop origins
    rng = np.random.default_rng(20260)
    jobs = []
    for i in range(cores):
        f = i % px_all.shape[0]
        y0 = int(rng.integers(0, gy)) * 16
        x0 = int(rng.integers(0, gx)) * 16
        jobs.append((px_all[f, y0 : y0 + crop, x0 : x0 + crop], st_all[f, y0 : y0 + crop, x0 : x0 + crop],
                     prof.t_phi, prof.t_nu, forced_code))
    return jobs, cores, crop


def cpu_baseline(workload: str, jobs=None, pool=None):
    """Oracle (plain-C FP64 port of the reference path) on all host cores over
    the bounded sample of cpu_jobs (one process per core).  `pool`: a
    multiprocessing Pool created once by the caller (outside the timing)."""
    from multiprocessing import Pool

    from oracle import oracle

    oracle.lib()  # build once before forking
    if jobs is None:
        jobs = cpu_jobs(workload)
    jobs, cores, crop = jobs
    own = pool is None
    if own:
        pool = Pool(cores)
    try:
        t0 = time.perf_counter()
        res = pool.map(_oracle_crop, jobs, chunksize=1)
        wall = time.perf_counter() - t0
    finally:
        if own:
            pool.close()
            pool.join()
    cells = sum(r[0] for r in res)
    return {
        "value": cells / wall,
        "cells": int(cells),
        "wall_s": wall,
        "unit": UNIT,
        "cores": cores,
        "kind": "port",
        "sample": f"{cores} crops {crop}x{crop} at seeded positions over {workload} frames ({cells} lost cells), "
                  f"one process per core, plain-C FP64 oracle, {wall:.1f}s wall",
    }


def run_reference(args, rank, world):
    """Reference arm: the CPU reference path (oracle port) on the host cores;
    rank 0 alone works under torchrun, the other ranks exit without work."""
    if rank != 0:
        return
    from multiprocessing import Pool

    from oracle import oracle

    oracle.lib()
    jobs = cpu_jobs(args.workload)
    times = []
    cells = []
    last = None
    with Pool(jobs[1]) as pool:  # created once, outside the timed steps
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            last = cpu_baseline(args.workload, jobs, pool)
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
                cells.append(last["cells"])
    value = float(np.sum(cells)) / float(np.sum(times))  # lost cells over the timed steps / their wall time
    last = dict(last, value=value)
    cfg, prof_name, forced = WORKLOADS[args.workload]
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True,
        "scaling": default_scaling(args, cfg), "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": args.workload, "profile": prof_name, "forced_layer": forced,
                   "baseline_config": CONFIGS[cfg][:3]},
        "cpu_baseline": last,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------- launcher


def free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-exec under torchrun with N
    ranks (one process per GPU, rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, BM_BENCH_RELAUNCHED="1")
    return subprocess.call(cmd, env=env)


def default_scaling(args, cfg: int) -> str:
    """Batch configs shard the config's own batch (strong); single-image
    configs run one replica per GPU (weak)."""
    if CONFIGS[cfg][0] == 1:
        return "weak"
    return "strong" if args.scaling == "auto" else args.scaling


def blocks8_lost(st_np) -> int:
    """Lost 8x8 blocks (SURVEY.md §8(d) secondary unit of cfg 4)."""
    b, h, w = st_np.shape
    g = (st_np[:, : h // 8 * 8, : w // 8 * 8] == 1).reshape(b, h // 8, 8, w // 8, 8)
    return int(g.any(axis=(2, 4)).sum())


# ----------------------------------------------------------------------- ours


class Timer:
    """Device time of one step: CUDA events on the launching stream (GPU), or
    the host clock for the CPU stub (--stub, launcher tests)."""

    def __init__(self, torch, cuda: bool):
        self.torch, self.cuda = torch, cuda
        if cuda:
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e1 = torch.cuda.Event(enable_timing=True)

    def start(self):
        if self.cuda:
            self.e0.record()
        else:
            self.t0 = time.perf_counter()

    def stop(self) -> float:
        if self.cuda:
            self.e1.record()
            self.e1.synchronize()
            return self.e0.elapsed_time(self.e1)
        return 1e3 * (time.perf_counter() - self.t0)


def measure(args, ctx, frame_range, n_total):
    """W warm-up + K timed steps over frames [start, stop) of the workload on
    this rank, each step = concealment of the rank's frames + the result
    gather to rank 0.  Returns the per-rank timing and counts."""
    torch, dev, world, cuda = ctx["torch"], ctx["dev"], ctx["world"], ctx["cuda"]
    from paper_2205_11226_b200.parallel import FrameGather

    cfg, prof_name, forced = WORKLOADS[args.workload]
    start, stop = frame_range
    if args.stub:  # launcher test: tiny frames, the step is a host copy
        px_np = np.zeros((stop - start, 32, 48), np.uint8)
        for i in range(stop - start):
            px_np[i] = (start + i if CONFIGS[cfg][0] > 1 else ctx["rank"]) % 251
        st_np = np.zeros_like(px_np)
    else:
        px_np, st_np = make_inputs(cfg, start, stop, world)
    px = torch.from_numpy(px_np).to(dev)
    st = torch.from_numpy(st_np).to(dev)
    gather = FrameGather(n_total, px.shape[1], px.shape[2], torch.uint8, dev)
    assert gather.local.shape[0] == px.shape[0]
    l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev) if cuda else None
    needs_flush = cuda and px.numel() * 2 < 2 * 126 * 1024 * 1024
    prof = profile_of(prof_name)
    if not args.stub:
        from paper_2205_11226_b200 import _native
        from paper_2205_11226_b200.profiles import conceal_batch

    def step():
        if args.stub:
            gather.local.copy_(px)
        else:
            conceal_batch(px, st, prof, forced_layer=forced, out_u8=gather.local, sync=False, time_kernel=True,
                          kernel_build=kbuild(args))
        gather.gather()  # the result gather to rank 0 (the path's only collective)

    for _ in range(args.warmup):
        step()
    if cuda:
        torch.cuda.synchronize()
        _native.kernel_times_reset()
    if world > 1:
        ctx["dist"].barrier()
    if cuda:
        torch.cuda.synchronize()
    timer = Timer(torch, cuda)
    step_ms = []
    with ClockSampler(ctx["local_rank"]) if cuda else _Null() as clk:
        for _ in range(args.steps):
            if needs_flush:
                flush_l2(torch, l2)
            timer.start()
            step()
            step_ms.append(timer.stop())
    if cuda:
        torch.cuda.synchronize()
    if world > 1:
        ctx["dist"].barrier()
    kms = _native.kernel_times_ms() if cuda else []
    if args.stub:
        summ = {"lost_cells": int(px.shape[0]), "patches": 0, "layer_counts": {}, "max_level": 0,
                "flop64": 0, "flop32": 0}
    else:  # counts / algorithmic work of one (deterministic) step
        summ = conceal_batch(px, st, prof, forced_layer=forced, out_u8=gather.local, sync=True,
                             kernel_build=kbuild(args)).summary
    frames = gather.frames()
    if frames is not None and ctx["rank"] == 0:
        assert frames.shape[0] == n_total
        if args.stub and stop - start < n_total:  # every rank's frames arrived in order at rank 0
            want = torch.arange(start if world == 1 else 0, (start if world == 1 else 0) + n_total) % 251
            assert torch.equal(frames[:, 0, 0].to(torch.int64), want), "result gather out of order"
    return {"px_np": px_np, "st_np": st_np, "step_ms": step_ms, "kms": kms, "summ": summ,
            "clocks": clk.summary() if cuda else None, "px": px}


def kbuild(args):
    b = args.kernel_build
    return None if b == "auto" else (int(b) if b.isdigit() else b)


def build_flags(args) -> int:
    from paper_2205_11226_b200 import _native

    return {"auto": 0, "256": _native.BM_FLAG_BUILD_256, "512": _native.BM_FLAG_BUILD_512,
            "cluster": _native.BM_FLAG_BUILD_CLUSTER, "narrow512": _native.BM_FLAG_NARROW_512}[args.kernel_build]


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def reduce_max_sum(ctx, local_ms: float, cells: float):
    torch = ctx["torch"]
    t = torch.tensor([local_ms], dtype=torch.float64, device=ctx["dev"])
    c = torch.tensor([cells], dtype=torch.float64, device=ctx["dev"])
    if ctx["world"] > 1:
        ctx["dist"].all_reduce(t, op=ctx["dist"].ReduceOp.MAX)
        ctx["dist"].all_reduce(c, op=ctx["dist"].ReduceOp.SUM)
    return float(t.item()), float(c.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg5", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"],
                    help="auto (default): batch configs shard the config's own batch by frame range over the N "
                         "ranks (strong scaling) and also report weak scaling (every rank its own batch of the "
                         "config's size) in `secondary`; single-image configs run one replica per GPU")
    ap.add_argument("--kernel-build", default="auto", choices=["auto", "256", "512", "cluster", "narrow512"],
                    help="concealment kernel build (default: chosen on the device from the DAG shape)")
    ap.add_argument("--stub", action="store_true", help=argparse.SUPPRESS)  # CPU launcher test (gloo, no GPU)
    args = ap.parse_args()

    from paper_2205_11226_b200.parallel import dist_env, shard_range

    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} runs under a world of {world} ranks")

    import torch
    import torch.distributed as dist

    cuda = not args.stub
    if cuda:
        torch.cuda.set_device(local_rank)
        dev = torch.device("cuda", local_rank)
    else:
        dev = torch.device("cpu")
    if world > 1:
        if cuda:
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
        assert dist.get_world_size() == args.gpus
    ctx = {"torch": torch, "dist": dist, "dev": dev, "world": world, "rank": rank, "local_rank": local_rank,
           "cuda": cuda}
    cfg, prof_name, forced = WORKLOADS[args.workload]
    prof = profile_of(prof_name)
    n_frames = CONFIGS[cfg][0]
    scaling = default_scaling(args, cfg)
    if n_frames == 1:  # single-image configs: one replica per GPU
        rng_main, n_total = (0, 1), 1
    elif scaling == "strong":  # the config's own batch sharded by frame range
        rng_main, n_total = shard_range(n_frames, rank, world), n_frames
    else:  # weak: every rank conceals its own batch of the config's size (frames are independent)
        rng_main, n_total = (rank * n_frames, (rank + 1) * n_frames), n_frames * world
    # replicas gather one frame per rank; batch configs gather the frames
    m = measure(args, ctx, rng_main, n_total if n_frames > 1 else world)
    total_ms, cells = reduce_max_sum(ctx, float(np.sum(m["step_ms"])), float(m["summ"]["lost_cells"]))
    ms_per_step = total_ms / args.steps
    value = cells / (ms_per_step / 1e3)
    summ, px_np, st_np, px = m["summ"], m["px_np"], m["st_np"], m["px"]
    blocks8 = None
    if cfg == 4 and not args.stub:
        _, b8 = reduce_max_sum(ctx, 0.0, float(blocks8_lost(st_np)))
        blocks8 = b8 / (ms_per_step / 1e3)

    # weak scaling as the secondary line of a strong N > 1 run
    secondary = {}
    if world > 1 and n_frames > 1 and scaling == "strong" and args.scaling == "auto":
        wk = measure(args, ctx, (rank * n_frames, (rank + 1) * n_frames), n_frames * world)
        w_ms, w_cells = reduce_max_sum(ctx, float(np.sum(wk["step_ms"])), float(wk["summ"]["lost_cells"]))
        secondary["weak"] = {"value": w_cells / (w_ms / args.steps / 1e3), "unit": UNIT,
                             "ms_per_step": w_ms / args.steps, "frames_per_rank": n_frames,
                             "frames": n_frames * world}
        del wk

    # ---- e2e through the C ABI with host buffers (pinned), every step H2D + D2H
    e2e = None
    if cuda and not args.no_e2e:
        import ctypes

        from paper_2205_11226_b200 import _native
        from paper_2205_11226_b200.profiles import make_params

        lib = _native.lib()
        params = make_params(px.shape[0], px.shape[1], px.shape[2], 0, prof, 10.0, forced)
        params.flags |= build_flags(args)
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
        e2e_ms, _ = reduce_max_sum(ctx, 1e3 * (time.perf_counter() - t0), 0.0)
        e2e = {"value": cells * args.steps / (e2e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h_px.numel() + h_st.numel()),
               "d2h_bytes_per_step": int(h_out.numel()) + ctypes.sizeof(_native.Summary),
               "path": "bm_conceal_host (C ABI, host buffers), per rank"}

    if rank == 0:
        kms = m["kms"]
        kmean = float(np.mean(kms)) if kms else None
        roof = None
        if kmean:
            roof = roofline(args, summ, kmean, ms_per_step, px)
        cpu = None
        if cuda and not args.no_cpu_baseline and world == 1:
            try:
                cpu = cpu_baseline(args.workload)
            except Exception as exc:  # reported, not fatal
                cpu = {"error": repr(exc)}
        sms = torch.cuda.get_device_properties(dev).multi_processor_count if cuda else 148
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic" if not args.stub else "stub",
            "config": {"workload": args.workload, "profile": prof_name, "forced_layer": forced,
                       "frames": n_total, "height": int(px.shape[1]), "width": int(px.shape[2]),
                       "lost_cells_per_step": int(cells), "patches": summ["patches"],
                       "layer_counts": summ["layer_counts"], "dag_depth": summ["max_level"],
                       "l2": "flushed (256 MiB write) between steps" if px.numel() * 2 < 2 * 126 * 1024 * 1024
                             else "inputs larger than L2",
                       "parallelism": (f"frames sharded x{world} (strong)" if scaling == "strong" else
                                       f"{n_frames} frames per rank x{world}" if n_frames > 1 else f"replicas x{world}"),
                       "result_gather": "dist.gather of the u8 frames to rank 0 (NCCL), preallocated buffers",
                       "conceal_build": BUILD_LABEL.get(summ.get("kernel_build"), summ.get("kernel_build"))},
            "gpu_launches": LAUNCHES_PER_STEP * args.steps if cuda else 0,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": m["clocks"],
        }
        if blocks8 is not None:
            secondary["lost_8x8_blocks_per_s"] = blocks8
        if secondary:
            out["secondary"] = secondary
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def roofline(args, summ, kmean, ms_per_step, px):
    flop64 = summ["flop64"]
    flop32 = summ["flop32"]
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
    return {
        "bound": "fp64", "achieved": a64, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
        "frac": a64 / FP64_PEAK_TFLOPS, "traffic": traffic,
        "traffic_unit": "bytes per k_conceal launch (dram__bytes_read.sum + dram__bytes_write.sum, "
                        "ncu --set full, profiles/ncu_traffic.json)",
        "algorithmic_bytes_per_launch": int(px.numel() * 3),
        "kernel": "bm::k_conceal", "kernel_ms": kmean, "kernel_share_of_step": kmean / ms_per_step,
        "flop64_per_launch": flop64, "flop32_per_launch": flop32,
        "fp32_gate": {"achieved": a32, "peak": FP32_PEAK_TFLOPS, "frac": a32 / FP32_PEAK_TFLOPS},
        "composite_frac": a64 / FP64_PEAK_TFLOPS + a32 / FP32_PEAK_TFLOPS,
        "peak_source": "measured on this pool's B200: DMMA m8n8k4 f64 36.8 TF/s (DFMA 36.2, same FP64 "
                       "hardware), FFMA 69.7 TF/s (tools/peakbench.cu, tools/pipebench.cu; "
                       "MEASURED_PEAKS.json has HBM and bf16 only)",
    }


if __name__ == "__main__":
    main()
