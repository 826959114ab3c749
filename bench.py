#!/usr/bin/env python3
"""bench.py -- the fused AR + residual-add + RMSNorm hot path on B200.

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1 workload: BASELINE.json configs[2] at TP=1 -- the Qwen2.5-72B / Llama
layer-boundary shape 8192 tokens x 8192 hidden bf16 (configs[1], TP=8 on
8xB200, does not fit one GPU).  At TP=1 the fused op degenerates to kernel K2
(fused residual-add + RMSNorm, HBM-bound).  A "step" is one fused op over one
[T,H] batch.  `value` = device time per op (CUDA events on the launching
stream, max over ranks), microseconds, lower is better.

N>1 (torchrun, one process per GPU): TP=N fused AllReduce + residual + RMSNorm
(kernel K1) over the multi-process communicator, strong scaling (same T).

--impl reference: the reference's own CPU implementation of the path
(oracle/_ref = proj/src/numerics.cpp + collectives.cpp compiled unmodified)
on the host cores, same config/metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused AR+RMSNorm µs & NVLink GB/s, 1024–8192 tok × 8192 hid, TP=1/2/4/8"
UNIT = "us"
T_DEFAULT = 8192
H_DEFAULT = 8192
EPS = 1e-5


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int = 0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        cmd = ["nvidia-smi", f"--id={self.index}", "--query-gpu=" + ",".join(self.FIELDS),
               "--format=csv,noheader,nounits", "-lms", "100"]
        try:
            p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        try:
            while not self._stop.is_set():
                line = p.stdout.readline()
                if not line:
                    break
                parts = [x.strip() for x in line.split(",")]
                if len(parts) == len(self.FIELDS):
                    self.samples.append(parts)
        finally:
            p.terminate()
            try:
                p.wait(timeout=2)
            except Exception:
                p.kill()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        time.sleep(0.2)
        self._stop.set()
        self._t.join(timeout=3)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower().startswith("active")})
        loaded = [x for x in sm if x > 0.5 * (max(mx) if mx else 0)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_reference_times(T, H, steps, threads):
    """The reference rmsnorm_residual (oracle/_ref) timed on the host cores."""
    import oracle  # cpu_baseline leg only
    ref = oracle.RefLib()
    return [ref.time_rmsnorm(T, H, threads, 1) for _ in range(steps)]


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    T, H = args.tokens, args.hidden
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_times(T, H, 1, threads)
    t0 = time.perf_counter()
    ms = cpu_reference_times(T, H, args.steps, threads)
    wall = time.perf_counter() - t0
    us = 1e3 * sum(ms) / len(ms)
    line = {
        "impl": "reference", "metric": METRIC, "value": us, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": us / 1e3, "higher_is_better": False,
        "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic U(-1,1) inputs, unit weight",
        "config": {"workload": f"reference rmsnorm_residual (TP=1 degenerate fused op), {T} tok x {H} hid",
                   "tokens": T, "hidden": H, "tp": 1},
        "cpu_baseline": {"value": us, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"full workload per step ({T}x{H} fp32), token rows chunked over {threads} "
                                   f"threads each calling weavesim::rmsnorm_residual; wall {wall:.1f}s"},
        "e2e": {"value": us, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def k2_single_gpu(args):
    import torch
    import paper_2505_11329_b200 as tw

    T, H = args.tokens, args.hidden
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream()
    g = torch.Generator(device=dev).manual_seed(0)
    x = (torch.rand(T, H, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    r = (torch.rand(T, H, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    w = torch.rand(H, device=dev, generator=g) + 0.5
    out = torch.empty_like(x)
    rout = torch.empty_like(x)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # 256 MiB > 126 MB L2

    def step():
        tw.rmsnorm_residual(x, r, w, EPS, residual_out=rout, out=out, stream=stream)

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # L2 flush, outside the event pair
            starts[i].record(stream)
            step()
            ends[i].record(stream)
    torch.cuda.synchronize()
    times_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    return times_ms, (x, r, w, out, rout)


def k2_sweep(tokens_list, H, reps=20):
    """Per-T K2 latency (same method) for the TP=1 column of the report."""
    import torch
    import paper_2505_11329_b200 as tw
    dev = torch.device("cuda:0")
    res = {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for T in tokens_list:
        x = torch.randn(T, H, device=dev, dtype=torch.bfloat16)
        r = torch.randn(T, H, device=dev, dtype=torch.bfloat16)
        w = torch.ones(H, device=dev)
        out, rout = torch.empty_like(x), torch.empty_like(x)
        for _ in range(3):
            tw.rmsnorm_residual(x, r, w, EPS, residual_out=rout, out=out)
        ts = []
        for i in range(reps):
            flush.fill_(i & 0xFF)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            tw.rmsnorm_residual(x, r, w, EPS, residual_out=rout, out=out)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        us = 1e3 * statistics.median(ts)
        nbytes = 4 * T * H * 2 + 4 * H
        res[str(T)] = {"us": round(us, 2), "hbm_gbs": round(nbytes / us / 1e3, 1)}
    return res


def unfused_baseline(T, H, reps=20):
    """Unfused TP=1 baseline on the same box: torch add + torch rms_norm
    (two kernels, the 'AR+RMSNorm' row's RMSNorm half without the AR)."""
    import torch
    dev = torch.device("cuda:0")
    x = torch.randn(T, H, device=dev, dtype=torch.bfloat16)
    r = torch.randn(T, H, device=dev, dtype=torch.bfloat16)
    w = torch.ones(H, device=dev, dtype=torch.bfloat16)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        y = torch.nn.functional.rms_norm(x + r, (H,), w, EPS)
    ts = []
    for i in range(reps):
        flush.fill_(i & 0xFF)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        rr = x + r
        y = torch.nn.functional.rms_norm(rr, (H,), w, EPS)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return round(1e3 * statistics.median(ts), 2)


def k2_e2e(args, bufs):
    """Same op through the public C-ABI with HOST buffers: pinned H2D of input
    and residual, the kernel, D2H of output and residual_out, per step."""
    import torch
    import paper_2505_11329_b200 as tw
    T, H = args.tokens, args.hidden
    x, r, w, out, rout = bufs
    hx = torch.empty(T, H, dtype=torch.bfloat16, pin_memory=True)
    hr = torch.empty(T, H, dtype=torch.bfloat16, pin_memory=True)
    ho = torch.empty(T, H, dtype=torch.bfloat16, pin_memory=True)
    hro = torch.empty(T, H, dtype=torch.bfloat16, pin_memory=True)
    hx.copy_(x)
    hr.copy_(r)
    stream = torch.cuda.Stream()
    steps = max(3, min(args.steps, 20))

    def step():
        x.copy_(hx, non_blocking=True)
        r.copy_(hr, non_blocking=True)
        tw.rmsnorm_residual(x, r, w, EPS, residual_out=rout, out=out, stream=stream)
        ho.copy_(out, non_blocking=True)
        hro.copy_(rout, non_blocking=True)

    with torch.cuda.stream(stream):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        s.record(stream)
        for _ in range(steps):
            step()
        e.record(stream)
    torch.cuda.synchronize()
    us = 1e3 * s.elapsed_time(e) / steps
    nb = T * H * 2
    return {"value": round(us, 2), "unit": UNIT, "h2d_bytes_per_step": 2 * nb, "d2h_bytes_per_step": 2 * nb,
            "steps": steps, "path": "tw_rmsnorm_residual via ctypes C-ABI, pinned host buffers"}


def load_profile_traffic(name):
    p = os.path.join(ROOT, "profiles", name)
    try:
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def run_ours_single(args):
    import torch
    T, H = args.tokens, args.hidden
    peak, peak_kind = measured_peaks()
    with ClockSampler(0) as clk:
        t0 = time.perf_counter()
        times_ms, bufs = k2_single_gpu(args)
        e2e = k2_e2e(args, bufs)
        wall = time.perf_counter() - t0
    avg_us = 1e3 * sum(times_ms) / len(times_ms)
    alg_bytes = 4 * T * H * 2 + 4 * H  # read in+res, write res_out+out (bf16), read fp32 weight
    achieved = alg_bytes / (avg_us * 1e-6) / 1e9
    line = {
        "metric": METRIC, "value": round(avg_us, 3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(avg_us / 1e3, 6), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic U(-1,1) bf16 activations, U(0.5,1.5) fp32 weight",
        "config": {"workload": f"TP=1 fused residual-add+RMSNorm (K2), {T} tok x {H} hid bf16 "
                               "(Qwen2.5-72B/Llama-3.3-70B layer-boundary shape)",
                   "tokens": T, "hidden": H, "tp": 1, "l2": "flushed between steps (256 MiB write)",
                   "sm_budget": "whole GPU"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                     "alg_bytes_per_launch": alg_bytes,
                     "traffic": load_profile_traffic("k2_ncu_r01.json")},
        "e2e": e2e,
        "gpu_launches": args.steps,
        "kernel_us": {"median": round(1e3 * statistics.median(times_ms), 3), "min": round(1e3 * min(times_ms), 3),
                      "max": round(1e3 * max(times_ms), 3)},
    }
    clocks = clk.summary()
    line["clocks"] = clocks
    if not args.quick:
        line["tp1_sweep"] = k2_sweep([1024, 2048, 4096, 8192], H)
        line["unfused_torch_add_rmsnorm_us"] = unfused_baseline(T, H)
        threads = os.cpu_count() or 1
        sample_T = 2048
        ms = cpu_reference_times(sample_T, H, 3, threads)
        cpu_us = 1e3 * statistics.median(ms) * (T / sample_T)
        line["cpu_baseline"] = {"value": round(cpu_us, 1), "unit": UNIT, "cores": threads, "kind": "reference",
                                "sample": f"weavesim::rmsnorm_residual (oracle/_ref) on {sample_T}x{H} fp32, "
                                          f"median of 3, scaled x{T // sample_T} to {T} tokens"}
    line["wall_s"] = round(wall, 2)
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--tokens", type=int, default=T_DEFAULT)
    ap.add_argument("--hidden", type=int, default=H_DEFAULT)
    ap.add_argument("--quick", action="store_true", help="skip sweeps/baselines (profiling runs)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from tools.bench_tp import run_tp  # multi-process TP=N path
        return run_tp(args)
    return run_ours_single(args)


if __name__ == "__main__":
    sys.exit(main())
