"""MPNL detector benchmark (driver contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl mpnl|reference]

A *step* = one pass of the hot path over one batch: `mpnl_plan_batch` (fp64
sorted QR of every RB channel) + `mpnl_detect_hard` (fp32 traversal kernel +
fp64 fix-up) over all the config's received vectors, inputs resident in HBM.
Default workload = BASELINE configs[1] (C2: 12x12, 16-QAM, 64 paths, 273 RBs,
6-point SNR sweep = 275,184 vectors per step).

* value  = vectors/s over all ranks (weak scaling: every rank detects its own
  seeded copy of the workload; no collective on the data path);
* e2e    = same metric through the public API from pinned HOST buffers:
  H2D of H and y, plan + detect, D2H of hard labels + metrics, every step;
* roofline = the traversal kernel (dominant): algorithmic path FLOPs
  P*4N(N+1) per vector / its CUDA-event duration, against the FP32 peak
  (max of a live FFMA probe and the spec 148 SM x 128 x 2 x 1.965 GHz);
* cpu_baseline = the numpy oracle port of the reference path on this host's
  cores, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SPEC_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def _traffic(cfg_name, n_rb, full_rb):
    """DRAM bytes per launch of the traversal kernel from the committed ncu
    capture summary (profiles/traffic.json, written by tools/ncu_summary.py
    traffic); only valid for the full-size workload it was captured on."""
    try:
        t = json.loads((ROOT / "profiles" / "traffic.json").read_text())[cfg_name]
    except Exception:
        return None, None
    if n_rb != full_rb:
        return None, None
    return t["dram_bytes_per_launch"], t["source"]


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    """SM clock + throttle reasons sampled by NVML every ~2 ms while the timed
    region runs (nvidia-smi -lms is too coarse for a ~10 ms region)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._nv = None
        return self

    def _run(self):
        nv = self._nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        while not self._stop.is_set():
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM),
                                     int(get_reasons(self._h))))
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        mask = 0
        for s in self.samples:
            mask |= s[1]
        reasons = sorted(k for k, bit in self.REASONS.items() if mask & bit)
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml"}


# ---------------------------------------------------------------------------
# CPU side (oracle port = the reference algorithm, numpy)
# ---------------------------------------------------------------------------

def cpu_rate(cfg_name, target_s=12.0, seed=2409):
    """Oracle vectors/s on all host cores over a bounded sample of the config."""
    from oracle import mpnl_oracle as orc
    from paper_2409_14355_b200.workloads import CONFIGS, generate

    cfg = CONFIGS[cfg_name]
    cores = len(os.sched_getaffinity(0))
    pilot = generate(cfg_name, seed=seed, n_rb=1)
    t0 = time.perf_counter()
    orc.detect_rb(pilot["h"], pilot["y"], pilot["nv"][0], cfg.n_paths, cfg.order,
                  __import__("paper_2409_14355_b200.core", fromlist=["x"])
                  .constellation_for(cfg.order).points)
    per_rb = time.perf_counter() - t0
    n_rb = int(max(cores, min(cfg.n_rb, round(target_s * cores / max(per_rb, 1e-3)))))
    n_rb = min(n_rb, cfg.n_rb)
    d = generate(cfg_name, seed=seed, n_rb=n_rb)
    t0 = time.perf_counter()
    orc.detect_rb_parallel(d["h"], d["y"], d["nv"][0], cfg.n_paths, cfg.order, workers=cores,
                           rbs_per_task=1)
    dt = time.perf_counter() - t0
    vec = n_rb * cfg.vectors_per_channel
    return {"value": vec / dt, "unit": "vectors/s", "cores": cores, "kind": "port",
            "n_rb": n_rb,
            "sample": f"first {n_rb} of {cfg.n_rb} RBs ({vec} vectors) of {cfg_name}, "
                      f"plan per RB + detect, ProcessPool x{cores}, {dt:.1f} s",
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# multi-rank plumbing (replicas over RB shards; no data-path collective)
# ---------------------------------------------------------------------------

def rank_seed(seed, rank):
    """Each rank detects its own seeded copy of the workload (weak scaling)."""
    return seed + 7919 * rank


def max_over_ranks(x, world, device=None):
    """Max of a per-rank scalar (device time) over all ranks."""
    if world == 1:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def job_rate(vectors_per_rank, world, total_ms, steps):
    """Whole-job vectors/s: all ranks' vectors / the slowest rank's time."""
    return world * vectors_per_rank / (total_ms / steps * 1e-3)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_gpu(args, rank, world):
    import torch

    from paper_2409_14355_b200 import _lib
    from paper_2409_14355_b200 import detect as det
    from paper_2409_14355_b200.core import constellation_for
    from paper_2409_14355_b200.workloads import CONFIGS, generate

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    cfg = CONFIGS[args.config]
    c = constellation_for(cfg.order)
    n_rb = args.n_rb or cfg.n_rb
    d = generate(cfg, seed=rank_seed(args.seed, rank), n_rb=n_rb)
    nv = float(d["nv"][0])
    h_host = torch.from_numpy(d["h"]).pin_memory()
    y_host = torch.from_numpy(d["y"]).pin_memory()
    h = h_host.to(dev)
    y = y_host.to(dev)
    nvec = y.shape[0] * y.shape[1]
    lib = _lib.load()
    # all work on one side stream (CUDA graphs cannot capture the legacy stream)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    # L2 flush buffer (> 126 MB L2)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    # device-resident step: plan + detect (stage 1 = fp32 traversal kernel, timed separately)
    plan = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
    realized = plan.n_paths
    hard = torch.empty((y.shape[0], y.shape[1], cfg.n), dtype=torch.uint8, device=dev)
    metric = torch.empty((y.shape[0], y.shape[1]), dtype=torch.float32, device=dev)
    ex = plan.expansions
    ws = torch.empty(int(lib.mpnl_workspace_bytes(nvec, cfg.n, cfg.order, ex.ctypes.data)),
                     dtype=torch.uint8, device=dev)

    def step(ev_k0=None, ev_k1=None):
        p = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
        args_ = (p.perm_dev.data_ptr(), p.r_dev.data_ptr(), p.qh_dev.data_ptr(),
                 p.tables.data_ptr(), y.data_ptr(), 0, y.shape[0], y.shape[1], cfg.m, cfg.n,
                 cfg.order, ex.ctypes.data, nv, hard.data_ptr(), metric.data_ptr(), None,
                 ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
        _lib.check(lib.mpnl_detect_hard_stage(1, *args_), "stage1")
        if ev_k0 is not None:
            ev_k0.record(stream)
        _lib.check(lib.mpnl_detect_hard_stage(2, *args_), "stage2")   # traversal kernel
        if ev_k1 is not None:
            ev_k1.record(stream)
        _lib.check(lib.mpnl_detect_hard_stage(3, *args_), "stage3")
        _lib.check(lib.mpnl_detect_hard_stage(4, *args_), "stage4")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # the step as one CUDA graph (8-10 dependent launches, no host work in the timed region)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        step()
    graph.replay()
    torch.cuda.synchronize()
    # flag statistics (outside timing)
    det_h, det_m, det_f = det.mpnl_detect_hard(plan, h, y, c, return_flags=True)
    flag_rate = float(det_f.float().mean())

    # FP32 peak probe
    probe_out = torch.empty(148 * 8 * 256, dtype=torch.float32, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lib.mpnl_ffma_probe(probe_out.data_ptr(), 148 * 8, 256, 256, stream.cuda_stream)
    e0.record(stream)
    fl = lib.mpnl_ffma_probe(probe_out.data_ptr(), 148 * 8, 256, 8192, stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    probe_tflops = fl / (e0.elapsed_time(e1) * 1e-3) / 1e12
    lib.mpnl_ffma2_probe(probe_out.data_ptr(), 148 * 8, 256, 256, stream.cuda_stream)
    e0.record(stream)
    fl2 = lib.mpnl_ffma2_probe(probe_out.data_ptr(), 148 * 8, 256, 8192, stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    probe2_tflops = fl2 / (e0.elapsed_time(e1) * 1e-3) / 1e12

    if world > 1:
        torch.distributed.barrier()
    step_ms, k_ms = [], []
    with ClockSampler(dev.index) as clk:
        for _ in range(args.steps):
            flush.zero_()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            torch.cuda.synchronize()
            ev[0].record(stream)
            graph.replay()
            ev[1].record(stream)
            torch.cuda.synchronize()
            step_ms.append(ev[0].elapsed_time(ev[1]))
        # the traversal kernel alone (eager step, events around stage 2)
        for _ in range(args.steps):
            flush.zero_()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            torch.cuda.synchronize()
            step(ev[0], ev[1])
            torch.cuda.synchronize()
            k_ms.append(ev[0].elapsed_time(ev[1]))
    tot_ms = max_over_ranks(float(np.sum(step_ms)), world, dev)
    if world > 1:
        torch.distributed.barrier()
    ms_per_step = tot_ms / args.steps
    value = job_rate(nvec, world, tot_ms, args.steps)

    # e2e through the public host-buffer API (C-ABI mpnl_detect_hard_host): pinned
    # host h, y in, pinned host labels / metrics out, copies inside the timed region
    out_h = torch.empty(hard.shape, dtype=torch.uint8).pin_memory()
    out_m = torch.empty(metric.shape, dtype=torch.float32).pin_memory()
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        det.mpnl_hard_output(h_host, y_host, nv, cfg.n_paths, c, out=(out_h, out_m))
        a1.record(stream)
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append(a0.elapsed_time(a1))
    e2e_ok = bool(torch.equal(out_h, hard.cpu()) and torch.equal(out_m, metric.cpu()))
    e2e_tot = max_over_ranks(float(np.sum(e2e_ms)), world, dev)
    e2e_val = job_rate(nvec, world, e2e_tot, args.steps)
    h2d = h_host.numel() * h_host.element_size() + y_host.numel() * y_host.element_size()
    d2h = out_h.numel() + out_m.numel() * 4

    flops_vec = realized * 4 * cfg.n * (cfg.n + 1)
    # kernels per step: plan, prep, select (per partial layer), traverse, verify, check, fp64 fix-up
    n_partial = int(sum(1 for e in ex if 1 < e < cfg.order))
    k_avg = float(np.mean(k_ms))
    achieved = flops_vec * nvec / (k_avg * 1e-3) / 1e12
    peak = max(SPEC_FP32_TFLOPS, probe_tflops, probe2_tflops)
    traffic, traffic_src = _traffic(cfg.name, n_rb, cfg.n_rb)
    line = {
        "metric": "detected MIMO vectors/sec",
        "value": round(value, 1),
        "unit": "vectors/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 (fp64 plan + fp64 fix-up of guarded vectors)",
        "data": "synthetic: seeded BASELINE-shaped channels/symbols/noise (workloads.py)",
        "config": {"workload": f"{cfg.name}: {cfg.n}x{cfg.m} {cfg.order}-QAM, P={realized}, "
                               f"{n_rb} RB x 168 RE x {len(cfg.snr_db)} SNR = {nvec} vectors/rank",
                   "n_rb": n_rb, "snr_db": list(cfg.snr_db), "l2": "flushed (256 MB write) "
                   "between timed steps", "step": "mpnl_plan_batch + mpnl_detect_hard "
                   "(replayed as one CUDA graph)",
                   "parallelism": f"replicas over RB shards x{world}"},
        "gbit_per_s": round(value * cfg.n * (cfg.order.bit_length() - 1) / 1e9, 3),
        "flag_rate": flag_rate,
        "roofline": {"bound": "fp32", "achieved": round(achieved, 3), "peak": round(peak, 2),
                     "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_source": traffic_src,
                     "algorithmic_bytes": round(cfg.bytes_per_vector() * nvec),
                     "kernel": f"traverse_kernel<{cfg.n},{int(round(c.order ** 0.5))}>",
                     "kernel_ms": round(k_avg, 4),
                     "flops_per_vector": flops_vec,
                     "peak_source": f"max(spec 148x128x2x1.965GHz = {SPEC_FP32_TFLOPS:.1f}, "
                                    f"live FFMA probe = {probe_tflops:.1f}, "
                                    f"live FFMA2 probe = {probe2_tflops:.1f})",
                     "hbm_peak_gbs": _peaks().get("hbm_gbs")},
        "e2e": {"value": round(e2e_val, 1), "unit": "vectors/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "api": "detect.mpnl_hard_output -> C-ABI "
                "mpnl_detect_hard_host (chunked, upload/compute/download overlapped)",
                "matches_device_path": e2e_ok},
        "gpu_launches": (6 + n_partial) * args.steps,
        "clocks": clk.summary(),
    }
    return line


def run_reference(args):
    """The reference algorithm on host cores (oracle port), same config/metric."""
    from oracle import mpnl_oracle as orc
    from paper_2409_14355_b200.workloads import CONFIGS, generate

    cfg = CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    base = cpu_rate(args.config, target_s=2.0, seed=args.seed)
    n_rb = int(base["n_rb"])
    d = generate(cfg, seed=args.seed, n_rb=n_rb)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        orc.detect_rb_parallel(d["h"], d["y"], d["nv"][0], cfg.n_paths, cfg.order,
                               workers=cores, rbs_per_task=1)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    vec = n_rb * cfg.vectors_per_channel
    ms = float(np.mean(times)) * 1e3
    val = vec / (ms * 1e-3)
    return {
        "impl": "reference", "metric": "detected MIMO vectors/sec", "value": round(val, 1),
        "unit": "vectors/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (same generator/seed)",
        "config": {"workload": f"{cfg.name} sample: {n_rb} RB = {vec} vectors per step",
                   "n_rb": n_rb},
        "cpu_baseline": {"value": round(val, 1), "unit": "vectors/s", "cores": cores,
                         "kind": "port", "sample": f"{n_rb} RBs ({vec} vectors) of {cfg.name} "
                         "per step; numpy restatement of the reference path, ProcessPool",
                         "cpu": _cpu_model()},
        "e2e": {"value": round(val, 1), "unit": "vectors/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--n-rb", type=int, default=0)
    ap.add_argument("--seed", type=int, default=2409)
    ap.add_argument("--impl", default="mpnl", choices=["mpnl", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "mpnl" else args.warmup

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        torch.distributed.init_process_group("nccl")
    line = run_gpu(args, rank, world)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_rate(args.config, seed=args.seed)
            line["cpu_baseline"].pop("n_rb", None)
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
