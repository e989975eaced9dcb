"""MPNL detector benchmark (driver contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5P1024]
                    [--scaling weak|strong] [--impl mpnl|reference]

A *step* = one pass of the hot path over one batch: `mpnl_plan_batch` (fp64
sorted QR of every RB channel) + `mpnl_detect_hard` (fp32 traversal kernel +
fp64 fix-up) over all the workload's received vectors, inputs resident in HBM.

Default workload = the largest single-GPU BASELINE configuration (BASELINE.json
quotes its metric on no particular config): C5, 24x24 64-QAM, 2,048 RBs x 168
REs = 344,064 vectors, at the heaviest point of its path sweep, P = 1024.  The
other sweep points (P = 16 / 64 / 256, same 2,048 RBs) are measured in the same
run and reported under "sweep"; the other configs are under `--config`.

* value  = vectors/s over all ranks.  Ranks shard RB ranges with no data-path
  collective: weak scaling (default) gives rank r the RBs [r*C, (r+1)*C) of one
  long seeded RB sequence; `--scaling strong` splits the config's C RBs;
* e2e    = the same metric through the public host-buffer API
  (`detect.mpnl_hard_output` -> C-ABI `mpnl_detect_hard_host`): H2D of H and y
  from pinned host memory, plan + detect, D2H of labels + metrics, every step;
* roofline = the traversal kernel (dominant): algorithmic path FLOPs
  P*4N(N+1) per vector / its CUDA-event duration, against the FP32 peak (max of
  a live FFMA probe and the spec 148 SM x 128 x 2 x 1.965 GHz); `step_frac` =
  the whole step against the same peak;
* cpu_baseline = the unmodified reference package (`baseline/_ref/mpnlsim`) on
  this host's cores, on a bounded sample of the same workload; its outputs are
  compared with the GPU's on the same vectors ("parity"), and the whole
  workload against the cached full reference run when present ("parity_full").
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
DEFAULT_CONFIG = "C5P1024"
SWEEPS = {"C5P1024": ["C5P16", "C5P64", "C5P256"]}
TIE_REL, METRIC_REL = 1e-5, 1e-4


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
# clocks sampler (NVML during the timed region)
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


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# multi-rank plumbing (RB-range shards; no data-path collective)
# ---------------------------------------------------------------------------

def shard(n_rb, rank, world, scaling):
    """(RBs of this rank, first RB index).  weak: every rank detects n_rb RBs,
    rank r the range [r*n_rb, (r+1)*n_rb) of one seeded RB sequence; strong: the
    n_rb RBs are split into `world` contiguous near-equal ranges."""
    if scaling == "weak":
        return n_rb, rank * n_rb
    lo = rank * n_rb // world
    hi = (rank + 1) * n_rb // world
    return hi - lo, lo


def max_over_ranks(x, world, device=None):
    """Max of a per-rank scalar (device time) over all ranks."""
    if world == 1:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def job_rate(total_vectors, total_ms, steps):
    """Whole-job vectors/s: all ranks' vectors / the slowest rank's time."""
    return total_vectors / (total_ms / steps * 1e-3)


# ---------------------------------------------------------------------------
# CPU side: the unmodified reference package on host cores
# ---------------------------------------------------------------------------

def _reference_runner():
    from oracle import reference_runner as rr
    if not rr.available():
        raise RuntimeError("reference package missing: install it into baseline/_ref "
                           "(see DESIGN.md §2)")
    return rr


def cpu_sample(cfg, d, target_s, cores, pool=None):
    """Reference hard output on a bounded sample of workload `d` (its first RBs,
    whole or cut into per-core sub-batches), sized to about `target_s` seconds
    on `cores` processes.  Returns (result dict, (hard, m1, m2), (n_rb, v))."""
    rr = _reference_runner()
    nv = float(d["nv"][0])
    v = d["y"].shape[1]
    # pilot: 16 vectors of the first RB in this process
    t0 = time.perf_counter()
    rr.detect_rb_hard((d["h"][:1], d["y"][:1, :16], nv, cfg.n_paths, cfg.order))
    per_vec = (time.perf_counter() - t0) / 16
    budget = int(target_s * cores / max(per_vec, 1e-7))
    if budget >= v:
        n_rb, nvec = min(d["h"].shape[0], max(1, budget // v)), v
    else:
        n_rb, nvec = 1, max(8, budget)
        nvec = min(nvec, v)
    per_task = max(1, -(-nvec // cores)) if n_rb == 1 else nvec
    tasks, index = rr.split_tasks(d["h"][:n_rb], d["y"][:n_rb, :nvec], nv, cfg.n_paths,
                                  cfg.order, per_task)
    own = pool is None
    pool = pool or rr.make_pool(cores)
    try:
        list(pool.map(int, [0] * cores))   # start the workers outside the timed region
        t0 = time.perf_counter()
        out = rr.run_tasks(pool, tasks, index, (n_rb, nvec, cfg.n))
        dt = time.perf_counter() - t0
    finally:
        if own:
            pool.shutdown()
    vec = n_rb * nvec
    res = {"value": vec / dt, "unit": "vectors/s", "cores": cores, "kind": "reference",
           "sample": f"{vec} vectors ({n_rb} RB x {nvec} RE) of {cfg.name} from its first RB; "
                     f"unmodified mpnlsim 0.1.0 ({rr.ref_path()}), plan per RB tiled, "
                     f"mpnl_detect_batch + hard composition, ProcessPool x{cores}, {dt:.1f} s",
           "cpu": _cpu_model()}
    return res, out, (n_rb, nvec)


def parity_block(hard, metric, ref_hard, m1, m2):
    """Compare GPU (hard, metric) with the reference (hard, m1, m2) on the same
    vectors: mismatches outside the 1e-5 tie exemption, max metric rel err."""
    hard = np.asarray(hard).reshape(ref_hard.shape)
    metric = np.asarray(metric, dtype=np.float64).reshape(m1.shape)
    exempt = (m2 - m1) <= TIE_REL * m1
    diff = np.any(hard != ref_hard, axis=-1)
    same = ~diff
    rel = np.abs(metric - m1) / np.maximum(m1, 1e-30)
    return {"vectors": int(diff.size), "label_mismatches": int(diff.sum()),
            "non_exempt_mismatches": int((diff & ~exempt).sum()),
            "tie_exempt": int(exempt.sum()),
            "max_metric_rel": float(rel[same].max()) if same.any() else None,
            "ok": bool(not (diff & ~exempt).any() and (not same.any()
                                                       or rel[same].max() <= METRIC_REL))}


def parity_full(cfg, hard, metric):
    """The whole workload against the cached full reference run
    (tools/oracle_full.py -> baseline/_ref/oracle_full/<cfg>.npz)."""
    path = ROOT / "baseline" / "_ref" / "oracle_full" / f"{cfg.name}.npz"
    if not path.exists():
        return None
    z = np.load(path)
    if z["hard"].shape != tuple(hard.shape):
        return None
    out = parity_block(hard, metric, z["hard"], z["m1"], z["m2"])
    out["source"] = f"baseline/_ref/oracle_full/{cfg.name}.npz (reference on all RBs)"
    return out


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def _launches_per_step(ex, order):
    # plan, prep, select (each partial layer the prep kernel does not fuse),
    # traverse, verify, check, fp64 fix-up
    partial = [e for e in ex if 1 < e < order]
    extra = max(0, len(partial) - 1) if partial and min(partial) in (2, 4) else len(partial)
    return 6 + extra


def measure_device(cfg, d, dev, stream, steps, warmup, lib, flush):
    """Device-resident step (plan + detect) as one CUDA graph, L2 flushed
    between timed steps; the traversal kernel timed by events around stage 2."""
    import torch

    from paper_2409_14355_b200 import _lib
    from paper_2409_14355_b200 import detect as det
    from paper_2409_14355_b200.core import constellation_for

    c = constellation_for(cfg.order)
    nv = float(d["nv"][0])
    h = torch.from_numpy(d["h"]).to(dev)
    y = torch.from_numpy(d["y"]).to(dev)
    nvec = y.shape[0] * y.shape[1]
    plan = det.mpnl_plan_batch(h, nv, cfg.n_paths, c)
    ex = plan.expansions
    hard = torch.empty((y.shape[0], y.shape[1], cfg.n), dtype=torch.uint8, device=dev)
    metric = torch.empty((y.shape[0], y.shape[1]), dtype=torch.float32, device=dev)
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

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        step()
    graph.replay()
    torch.cuda.synchronize()
    _, _, det_f = det.mpnl_detect_hard(plan, h, y, c, return_flags=True)
    flag_rate = float(det_f.float().mean())

    step_ms, k_ms = [], []
    for _ in range(steps):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        ev[0].record(stream)
        graph.replay()
        ev[1].record(stream)
        torch.cuda.synchronize()
        step_ms.append(ev[0].elapsed_time(ev[1]))
    for _ in range(steps):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        step(ev[0], ev[1])
        torch.cuda.synchronize()
        k_ms.append(ev[0].elapsed_time(ev[1]))
    del graph
    return {"step_ms": step_ms, "k_ms": k_ms, "flag_rate": flag_rate, "nvec": nvec,
            "realized": plan.n_paths, "ex": ex, "hard": hard, "metric": metric,
            "h": h, "y": y, "nv": nv, "c": c,
            "launches": _launches_per_step(ex, cfg.order)}


def fp32_peak(lib, stream, dev):
    import torch
    probe_out = torch.empty(148 * 8 * 256, dtype=torch.float32, device=dev)
    out = []
    for fn in (lib.mpnl_ffma_probe, lib.mpnl_ffma2_probe):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn(probe_out.data_ptr(), 148 * 8, 256, 256, stream.cuda_stream)
        e0.record(stream)
        fl = fn(probe_out.data_ptr(), 148 * 8, 256, 8192, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        out.append(fl / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return out


def run_gpu(args, rank, world):
    import torch

    from paper_2409_14355_b200 import _lib
    from paper_2409_14355_b200 import detect as det
    from paper_2409_14355_b200.workloads import CONFIGS, generate

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    cfg = CONFIGS[args.config]
    full_rb = args.n_rb or cfg.n_rb
    n_rb, rb0 = shard(full_rb, rank, world, args.scaling)
    d = generate(cfg, seed=args.seed, n_rb=n_rb, rb_offset=rb0)
    lib = _lib.load()
    stream = torch.cuda.Stream(dev)   # graphs cannot capture the legacy stream
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    probe, probe2 = fp32_peak(lib, stream, dev)
    peak = max(SPEC_FP32_TFLOPS, probe, probe2)

    if world > 1:
        torch.distributed.barrier()
    with ClockSampler(dev.index) as clk:
        r = measure_device(cfg, d, dev, stream, args.steps, args.warmup, lib, flush)
    nvec = r["nvec"]
    tot_ms = max_over_ranks(float(np.sum(r["step_ms"])), world, dev)
    # weak: every rank detects nvec vectors; strong: the ranks split one workload
    total_vec = nvec * world if args.scaling == "weak" else cfg.vectors_per_channel * full_rb
    if world > 1:
        torch.distributed.barrier()
    ms_per_step = tot_ms / args.steps
    value = job_rate(total_vec, tot_ms, args.steps)

    # e2e through the public host-buffer API (C-ABI mpnl_detect_hard_host): pinned
    # host h, y in, pinned host labels / metrics out, copies inside the timed region
    h_host = torch.from_numpy(d["h"]).pin_memory()
    y_host = torch.from_numpy(d["y"]).pin_memory()
    out_h = torch.empty(tuple(r["hard"].shape), dtype=torch.uint8).pin_memory()
    out_m = torch.empty(tuple(r["metric"].shape), dtype=torch.float32).pin_memory()
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        det.mpnl_hard_output(h_host, y_host, r["nv"], cfg.n_paths, r["c"], out=(out_h, out_m))
        a1.record(stream)
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append(a0.elapsed_time(a1))
    hard_cpu, metric_cpu = r["hard"].cpu(), r["metric"].cpu()
    e2e_ok = bool(torch.equal(out_h, hard_cpu) and torch.equal(out_m, metric_cpu))
    e2e_tot = max_over_ranks(float(np.sum(e2e_ms)), world, dev)
    e2e_val = job_rate(total_vec, e2e_tot, args.steps)
    h2d = h_host.numel() * h_host.element_size() + y_host.numel() * y_host.element_size()
    d2h = out_h.numel() + out_m.numel() * 4

    flops_vec = r["realized"] * 4 * cfg.n * (cfg.n + 1)
    k_avg = float(np.mean(r["k_ms"]))
    achieved = flops_vec * nvec / (k_avg * 1e-3) / 1e12
    step_tflops = flops_vec * nvec / (float(np.mean(r["step_ms"])) * 1e-3) / 1e12
    traffic, traffic_src = _traffic(cfg.name, n_rb if rb0 == 0 else -1, cfg.n_rb)
    line = {
        "metric": "detected MIMO vectors/sec",
        "value": round(value, 1),
        "unit": "vectors/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f32 (fp64 plan + fp64 fix-up of guarded vectors)",
        "data": "synthetic: seeded BASELINE-shaped channels/symbols/noise (workloads.py)",
        "config": {"workload": f"{cfg.name}: {cfg.n}x{cfg.m} {cfg.order}-QAM, P={r['realized']}, "
                               f"{n_rb} RB x 168 RE x {len(cfg.snr_db)} SNR = {nvec} vectors/rank",
                   "n_rb": n_rb, "rb_offset_rank0": rb0, "snr_db": list(cfg.snr_db),
                   "l2": "flushed (256 MB write) between timed steps",
                   "step": "mpnl_plan_batch + mpnl_detect_hard (replayed as one CUDA graph)",
                   "parallelism": f"RB-range shards x{world} ({args.scaling} scaling, no "
                                  "data-path collective)"},
        "gbit_per_s": round(value * cfg.n * (cfg.order.bit_length() - 1) / 1e9, 3),
        "flag_rate": r["flag_rate"],
        "roofline": {"bound": "fp32", "achieved": round(achieved, 3), "peak": round(peak, 2),
                     "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                     "step_frac": round(step_tflops / peak, 4),
                     "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes": round(cfg.bytes_per_vector() * nvec),
                     "kernel": f"traverse_kernel<{cfg.n},{int(round(cfg.order ** 0.5))}>",
                     "kernel_ms": round(k_avg, 4),
                     "flops_per_vector": flops_vec,
                     "peak_source": f"max(spec 148x128x2x1.965GHz = {SPEC_FP32_TFLOPS:.1f}, "
                                    f"live FFMA probe = {probe:.1f}, "
                                    f"live FFMA2 probe = {probe2:.1f})",
                     "hbm_peak_gbs": _peaks().get("hbm_gbs")},
        "e2e": {"value": round(e2e_val, 1), "unit": "vectors/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "copy_gbs": round((h2d + d2h) / (float(np.mean(e2e_ms)) * 1e-3) / 1e9, 2),
                # the chunked pipeline overlaps the copies with the kernels: when the
                # e2e step is close to the device step the copies are hidden
                "bound": ("compute (copies overlapped)"
                          if float(np.mean(e2e_ms)) < 1.25 * ms_per_step else "pcie copies"),
                "api": "detect.mpnl_hard_output -> C-ABI mpnl_detect_hard_host (chunked, "
                       "upload/compute/download overlapped on 3 streams)",
                "matches_device_path": e2e_ok},
        "gpu_launches": r["launches"] * args.steps,
        "clocks": clk.summary(),
    }
    # the rest of the path-count sweep on the same RBs (same timing rules)
    if world == 1 and not args.no_sweep:
        sweep = {}
        for name in SWEEPS.get(cfg.name, []):
            sc = CONFIGS[name]
            sd = generate(sc, seed=args.seed, n_rb=n_rb, rb_offset=rb0)
            with ClockSampler(dev.index) as sclk:
                s = measure_device(sc, sd, dev, stream, args.steps, args.warmup, lib, flush)
            fv = s["realized"] * 4 * sc.n * (sc.n + 1)
            sms, kms = float(np.mean(s["step_ms"])), float(np.mean(s["k_ms"]))
            sweep[name] = {"P": s["realized"], "vectors/s": round(s["nvec"] / (sms * 1e-3), 1),
                           "ms_per_step": round(sms, 4), "kernel_ms": round(kms, 4),
                           "frac": round(fv * s["nvec"] / (kms * 1e-3) / 1e12 / peak, 4),
                           "step_frac": round(fv * s["nvec"] / (sms * 1e-3) / 1e12 / peak, 4),
                           "flag_rate": s["flag_rate"], "sm_mhz": sclk.summary()["sm_mhz"]}
            pf = parity_full(sc, s["hard"].cpu().numpy(), s["metric"].cpu().numpy())
            if pf is not None:
                sweep[name]["parity_full"] = {k: pf[k] for k in ("vectors",
                                                                 "non_exempt_mismatches", "ok")}
            del s
        if sweep:
            line["sweep"] = sweep
    if rank == 0 and rb0 == 0:
        pf = parity_full(cfg, hard_cpu.numpy(), metric_cpu.numpy())
        if pf is not None:
            line["parity_full"] = pf
    return line, (d, hard_cpu.numpy(), metric_cpu.numpy())


# ---------------------------------------------------------------------------
# reference arm: the unmodified reference package on host cores
# ---------------------------------------------------------------------------

def run_reference(args):
    """`bench.py --impl reference`: the reference's own CPU implementation
    (mpnlsim from baseline/_ref, unmodified) on the same config/metric, each
    step a bounded sample of the workload on all host cores."""
    from paper_2409_14355_b200.workloads import CONFIGS, generate

    rr = _reference_runner()
    cfg = CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    d = generate(cfg, seed=args.seed, n_rb=min(cfg.n_rb, 64))
    pool = rr.make_pool(cores)
    try:
        res, _, (n_rb, nvec) = cpu_sample(cfg, d, args.ref_step_s, cores, pool)
        nv = float(d["nv"][0])
        per_task = nvec if n_rb > 1 else max(1, -(-nvec // cores))
        tasks, index = rr.split_tasks(d["h"][:n_rb], d["y"][:n_rb, :nvec], nv, cfg.n_paths,
                                      cfg.order, per_task)
        times = []
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            rr.run_tasks(pool, tasks, index, (n_rb, nvec, cfg.n))
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
    finally:
        pool.shutdown()
    vec = n_rb * nvec
    ms = float(np.mean(times)) * 1e3
    val = vec / (ms * 1e-3)
    return {
        "impl": "reference", "metric": "detected MIMO vectors/sec", "value": round(val, 1),
        "unit": "vectors/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (same generator/seed)",
        "config": {"workload": f"{cfg.name} sample: {vec} vectors ({n_rb} RB x {nvec} RE) "
                               "per step", "n_rb": n_rb},
        "cpu_baseline": {"value": round(val, 1), "unit": "vectors/s", "cores": cores,
                         "kind": "reference",
                         "sample": f"{vec} vectors of {cfg.name} per step; unmodified mpnlsim "
                                   f"0.1.0 ({rr.ref_path()}), plan per RB tiled, "
                                   "mpnl_detect_batch + hard composition, ProcessPool",
                         "cpu": _cpu_model()},
        "e2e": {"value": round(val, 1), "unit": "vectors/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def _spawn(args_list, n):
    """`--gpus N` without a launcher: re-run under torch.distributed.run."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *args_list]
    return subprocess.call(cmd)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--n-rb", type=int, default=0)
    ap.add_argument("--seed", type=int, default=2409)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--impl", default="mpnl", choices=["mpnl", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--cpu-s", type=float, default=15.0, help="cpu_baseline sample seconds")
    ap.add_argument("--ref-step-s", type=float, default=3.0, help="reference arm s/step")
    args = ap.parse_args(argv)
    if args.impl == "mpnl":
        args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_spawn(argv, args.gpus))
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
    line, (d, hard, metric) = run_gpu(args, rank, world)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            from paper_2409_14355_b200.workloads import CONFIGS
            cfg = CONFIGS[args.config]
            cores = len(os.sched_getaffinity(0))
            res, (rh, m1, m2), (n_rb, nvec) = cpu_sample(cfg, d, args.cpu_s, cores)
            line["cpu_baseline"] = res
            par = parity_block(hard[:n_rb, :nvec], metric[:n_rb, :nvec], rh, m1, m2)
            par["source"] = "cpu_baseline sample (same vectors, reference run live)"
            line["parity"] = par
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
