#!/usr/bin/env python3
"""bench.py -- the fused AR + residual-add + RMSNorm hot path on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1 workload: BASELINE.json configs[2] at TP=1 -- the Qwen2.5-72B /
Llama-3.3-70B layer-boundary shape, 8192 tokens x 8192 hidden, bf16
(configs[1] is TP=8 on 8xB200 and does not fit one GPU).  At TP=1 the fused
op degenerates to kernel K2 (fused residual-add + RMSNorm, HBM-bound).  A
"step" is one fused op over one [T,H] batch; `value` = device time per op
(CUDA events on the launching stream, max over ranks), microseconds, lower is
better.  `e2e` is the same op through the C-ABI with pinned HOST buffers
(H2D of input+residual and D2H of output+residual inside the timed region).

N>1 (torchrun, one process per GPU): TP=N fused AllReduce + residual + RMSNorm
(kernel K1) over the multi-process NVLS communicator at an 8-SM budget
(tools/bench_tp.py; NVLS or fail -- no silent PEER fallback).  Without
torchrun, `--gpus N` re-launches itself under torch.distributed.run.

--impl reference: the reference's own CPU implementation of the path
(oracle/_ref = proj/src/numerics.cpp / collectives.cpp compiled unmodified) on
the host cores, same config / metric / unit: rmsnorm_residual at N=1,
fused_allreduce_rmsnorm(parallel=true) with N ranks at N>1, full workload.
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
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
# NOTE: the product package is imported only inside our arm (main(), after the
# --impl dispatch), so the reference arm's process maps oracle/_ref alone.

METRIC = "fused AR+RMSNorm µs & NVLink GB/s, 1024–8192 tok × 8192 hid, TP=1/2/4/8"
UNIT = "us"
EPS = 1e-5
FLUSH_NOTE = ("L2 flushed between steps outside the event pair: 256 MiB buffer written then read back "
              "(> 126 MB L2; leaves clean lines, none of the op's inputs); working set 512 MiB > L2")


def measured_hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured copy bandwidth (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class L2Flush:
    def __init__(self, device):
        import torch
        self.buf = torch.empty(256 << 20, dtype=torch.uint8, device=device)
        self.sink = torch.empty(1, dtype=torch.float32, device=device)

    def __call__(self, i: int):
        self.buf.fill_(i & 0x7F)
        self.sink.copy_(self.buf.view(-1).view(__import__("torch").float32).sum().reshape(1))


def smi_id(local_index: int) -> str:
    """nvidia-smi's id for CUDA device `local_index`: its UUID (CUDA_VISIBLE_DEVICES
    may renumber devices, nvidia-smi does not), else the index."""
    try:
        import torch
        u = str(torch.cuda.get_device_properties(local_index).uuid)
        return u if u.startswith("GPU-") else f"GPU-{u}"
    except Exception:
        return str(local_index)


class ClockSampler:
    """nvidia-smi SM clocks + throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int = 0):
        self.index = smi_id(index)
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
        num = lambda s: s.replace(".", "", 1).isdigit()  # noqa: E731
        sm = [float(s[0]) for s in self.samples if num(s[0])]
        mx = [float(s[1]) for s in self.samples if num(s[1])]
        reasons = sorted({self.NAMES[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        top = max(mx) if mx else 0.0
        loaded = [x for x in sm if x > 0.5 * top] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": top or None,
                "reasons": reasons, "samples": len(self.samples)}


def bind_to_gpu_numa(index: int) -> dict:
    """Pin this process to the host cores NVML reports as local to GPU
    `index` (its PCIe root's NUMA node), so pinned staging buffers allocated
    afterwards are first-touched on that node: host<->device copies then do
    not cross the socket interconnect.  Returns what was done (for the line)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        ncpu = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1 and w * 64 + b < ncpu}
        try:
            node = pynvml.nvmlDeviceGetNumaNodeId(h)
        except Exception:  # noqa: BLE001
            node = None
        pynvml.nvmlShutdown()
        if cpus and len(cpus) < ncpu:
            os.sched_setaffinity(0, cpus)
        return {"gpu_numa_node": node, "cpus_bound": len(cpus) if cpus and len(cpus) < ncpu else "all",
                "host_cpus": ncpu}
    except Exception as exc:  # noqa: BLE001 -- informational
        return {"error": str(exc)[:120]}


# ---- reference CPU arm ----------------------------------------------------------------

def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_rmsnorm_each_ms(T, H, threads, iters):
    """weavesim::rmsnorm_residual (oracle/_ref, the reference sources compiled
    unmodified), token rows chunked over `threads` host threads; every
    iteration's ms on one set of inputs (generated once, outside the clock)."""
    import oracle  # cpu_baseline / --impl reference legs only
    return oracle.RefLib().time_rmsnorm(T, H, threads, iters, each=True)


def oracle_fused_ms(world, T, H, iters=3):
    """The reference's fused_allreduce_rmsnorm(parallel=true), median ms (cpu_baseline leg only)."""
    import oracle  # cpu_baseline / --impl reference legs only
    return oracle.RefLib().time_fused(world, T, H, True, iters)


def _reference_line(args, world, us, ms, sample, cores, workload):
    return {
        "impl": "reference", "metric": METRIC, "value": round(us, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(us / 1e3, 3), "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic U(-1,1) fp32 inputs, unit weight (mt19937_64, the reference tests' draws)",
        "config": {"workload": workload, "tokens": args.tokens, "hidden": args.hidden, "tp": world},
        "cpu_baseline": {"value": round(us, 1), "unit": UNIT, "cores": cores, "kind": "reference",
                         "cpu": cpu_model(), "host_threads_available": os.cpu_count(), "sample": sample},
        "e2e": {"value": round(us, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_ms": [round(x, 2) for x in ms],
        "gpu_launches": 0,
    }


def run_reference_arm(args):
    """The reference's own CPU code (oracle/_ref), full workload every step:
    N = 1 -> weavesim::rmsnorm_residual over all host threads (token chunks);
    N > 1 -> weavesim::fused_allreduce_rmsnorm with N ranks, parallel=true
    (proj/src/collectives.cpp:157-182: one std::thread per rank, validation
    included).  Under torchrun only rank 0 runs."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    world = max(args.gpus, int(os.environ.get("WORLD_SIZE", "1")))
    T, H = args.tokens, args.hidden
    t0 = time.perf_counter()
    if world > 1:
        import oracle  # --impl reference leg only
        ms = oracle.RefLib().time_fused(world, T, H, True, args.warmup + args.steps, each=True)[args.warmup:]
        cores = world
        sample = (f"full workload every step ({world} ranks x {T}x{H} fp32 partials + residual shards), "
                  f"weavesim::fused_allreduce_rmsnorm(parallel=true): one std::thread per rank")
        workload = (f"TP={world} fused AllReduce+residual+RMSNorm, {T} tok x {H} hid "
                    f"(reference CPU path, {world} in-process ranks)")
    else:
        cores = os.cpu_count() or 1
        ms = reference_rmsnorm_each_ms(T, H, cores, args.warmup + args.steps)[args.warmup:]
        sample = (f"full workload every step ({T}x{H} fp32): token rows chunked over {cores} threads, "
                  f"each calling weavesim::rmsnorm_residual")
        workload = f"TP=1 fused residual-add+RMSNorm, {T} tok x {H} hid (reference CPU path)"
    wall = time.perf_counter() - t0
    us = 1e3 * sum(ms) / len(ms)
    line = _reference_line(args, world, us, ms, sample + f"; wall {wall:.1f}s incl. input generation", cores,
                           workload)
    print(json.dumps(line), flush=True)
    return 0


# ---- our arm, N = 1 -------------------------------------------------------------------

def k2_timed(T, H, steps, warmup, flush, seed=0):
    """Per-step CUDA-event times (ms) of K2 on a dedicated stream."""
    import torch
    import paper_2505_11329_b200 as tw
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(seed)
    x = (torch.rand(T, H, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    r = (torch.rand(T, H, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    w = torch.rand(H, device=dev, generator=g) + 0.5
    out, rout = torch.empty_like(x), torch.empty_like(x)
    stream = torch.cuda.Stream()
    # warm-up = the timed loop's exact sequence (flush, then the op), so the
    # first timed step does not pay the flush path's first-use costs (it ran
    # ~140 us instead of ~85 when the warm-up skipped the flush)
    with torch.cuda.stream(stream):
        for i in range(max(warmup, 3)):
            flush(i)
            tw.rmsnorm_residual(x, r, w, EPS, residual_out=rout, out=out, stream=stream)
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    with torch.cuda.stream(stream):
        for i in range(steps):
            flush(i)
            starts[i].record(stream)
            tw.rmsnorm_residual(x, r, w, EPS, residual_out=rout, out=out, stream=stream)
            ends[i].record(stream)
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in zip(starts, ends)], (x, r, w, out, rout)


def k2_e2e(T, H, bufs, steps, dtype=None):
    """The same op through the public C-ABI with HOST buffers:
    tw_rmsnorm_residual_host pipelines H2D | K2 | D2H in chunks.  Every step
    moves the whole input+residual host->device and output+residual_out
    device->host; the clock covers all of it (CUDA events on the caller's
    stream, which the C-ABI joins back before returning).  dtype=torch.float32:
    the reference's dtype (fp32 host matrices, fp32 K2)."""
    import torch
    import paper_2505_11329_b200 as tw
    x, r, w, _, _ = bufs
    dt = dtype or torch.bfloat16
    hx = x.to(dt).cpu().pin_memory()
    hr = r.to(dt).cpu().pin_memory()
    hw = w.cpu()
    ho = torch.empty(T, H, dtype=dt).pin_memory()
    hro = torch.empty(T, H, dtype=dt).pin_memory()
    stream = torch.cuda.Stream()
    for _ in range(2):
        tw.rmsnorm_residual_host(hx, hr, hw, EPS, residual_out=hro, out=ho, stream=stream)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(stream)
    for i in range(steps):
        tw.rmsnorm_residual_host(hx, hr, hw, EPS, residual_out=hro, out=ho, stream=stream)
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    per = sorted(1e3 * ev[i].elapsed_time(ev[i + 1]) for i in range(steps))
    nb = T * H * hx.element_size()
    # the host results of the last step, checked (outside the clock)
    if dt == torch.bfloat16:  # vs the device K2 (itself checked by k2_parity): r' bitwise, out at the bf16 bar
        _, _, _, out, rout = bufs
        d = (ho.cuda().float() - out.float()).abs()
        worst = float((d - (2e-2 * out.float().abs() + 2e-2)).max())
        res_ok = bool(torch.equal(hro.cuda(), rout))
        parity = {"residual_bitwise_vs_device_k2": res_ok, "output_max_abs_diff_vs_device_k2": float(d.max()),
                  "ok": res_ok and worst <= 0.0}
        del d
    else:  # fp32: r' = x + r exactly, out vs a float64 restatement (the tests' 1e-5 bar)
        xs, rs = hx.to("cuda", torch.float64), hr.to("cuda", torch.float64)
        r64 = xs + rs
        want = r64 * torch.rsqrt(r64.pow(2).mean(dim=1, keepdim=True) + EPS) * w.to(torch.float64)
        err = float((ho.to("cuda", torch.float64) - want).abs().max())
        parity = {"residual_bitwise": bool(torch.equal(hro.cuda(), (hx.cuda() + hr.cuda()))),
                  "max_abs_err_output_vs_f64": err, "ok": err <= 1e-5}
        del xs, rs, r64, want
    # median step: one slow step (host memory contention on a shared box)
    # moved a 20-step mean by 60 % once; mean / min / max are reported beside it
    return {"value": round(per[len(per) // 2], 2), "unit": UNIT, "h2d_bytes_per_step": 2 * nb + 4 * H,
            "d2h_bytes_per_step": 2 * nb, "steps": steps, "stat": "median of per-step CUDA-event times",
            "mean": round(sum(per) / len(per), 2), "min": round(per[0], 2), "max": round(per[-1], 2),
            "path": "tw_rmsnorm_residual_host (C-ABI via ctypes): pinned host input/residual -> chunked "
                    "H2D | K2 | D2H pipeline over 3 streams -> pinned host output/residual_out",
            "parity": parity}


def k2_parity(bufs):
    """The timed K2's results on the line's own inputs against a torch fp32
    restatement of rmsnorm_residual (proj/src/numerics.cpp:30-64) at the
    tests' bf16 bar: r' = RNE(x + r) bit for bit; out within 2e-2*|want| + 2e-2
    (K2 normalises the bf16-rounded r', as does the restatement)."""
    import torch
    x, r, w, out, rout = bufs
    worst, max_abs, res_ok = -1.0, 0.0, True
    for a in range(0, x.shape[0], 1024):  # row blocks: bounded fp32 temporaries
        rb = (x[a:a + 1024].float() + r[a:a + 1024].float()).to(torch.bfloat16)
        res_ok &= bool(torch.equal(rout[a:a + 1024], rb))
        rf = rb.float()
        want = rf * torch.rsqrt(rf.pow(2).mean(dim=1, keepdim=True) + EPS) * w
        d = (out[a:a + 1024].float() - want).abs()
        worst = max(worst, float((d - (2e-2 * want.abs() + 2e-2)).max()))
        max_abs = max(max_abs, float(d.max()))
    return {"residual_bitwise": res_ok, "max_abs_err_output": round(max_abs, 5), "ok": res_ok and worst <= 0.0,
            "bar": "r' = RNE(x + r) bitwise; |out - want| <= 2e-2*|want| + 2e-2",
            "checker": "torch fp32 restatement on the device (not timed)"}


def unfused_torch(T, H, flush, reps=20):
    """Unfused TP=1 baseline on the same box: torch add + torch rms_norm."""
    import torch
    x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
    r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
    w = torch.ones(H, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        torch.nn.functional.rms_norm(x + r, (H,), w, EPS)
    ts = []
    for i in range(reps):
        flush(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.nn.functional.rms_norm(x + r, (H,), w, EPS)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return round(1e3 * statistics.median(ts), 2)


def k1_colocated(T, H, world, budget, flush, reps=10):
    """K1 with `world` simulated ranks on this GPU (PEER transport): a
    correctness-scale check of the fused path at full size.  HBM-bound here,
    NOT an NVLink number."""
    import torch
    import paper_2505_11329_b200 as tw
    comm = tw.Communicator(world, [0] * world, T * H * 2, tw.TW_TRANSPORT_PEER)
    for q in range(world):
        comm.buffer(q, tw.TW_BUF_INPUT, (T, H), torch.bfloat16).normal_()
    ranges = tw.token_shard_map(T, world)
    shards = [torch.randn(e - b, H, device="cuda", dtype=torch.bfloat16) for b, e in ranges]
    w = [torch.ones(H, device="cuda")] * world
    for _ in range(3):
        comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=budget)
    ts = []
    for i in range(reps):
        flush(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=budget)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    comm.check()
    comm.close()
    return round(1e3 * statistics.median(ts), 1)


def k2_after_dirty_l2(bufs, steps):
    """K2 after a 256 MiB WRITE (no read-back): the L2 is left full of dirty
    lines, as a producer GEMM's output leaves it at a real layer boundary, and
    their write-back lands inside the op's event pair.  Mean of `steps`."""
    import torch
    import paper_2505_11329_b200 as tw
    x, r, w, out, rout = bufs
    dirty = torch.empty(256 << 20, dtype=torch.uint8, device=x.device)
    stream = torch.cuda.Stream()
    evs = []
    with torch.cuda.stream(stream):
        for i in range(steps + 3):
            dirty.fill_(i & 0x7F)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            tw.rmsnorm_residual(x, r, w, EPS, residual_out=rout, out=out, stream=stream)
            e.record(stream)
            evs.append((s, e))
    torch.cuda.synchronize()
    ts = [1e3 * s.elapsed_time(e) for s, e in evs[3:]]
    return sum(ts) / len(ts)


def k2_back_to_back(bufs, steps, stream_reps=1):
    """Steady-state K2: `steps` launches back to back (no flush between them),
    one event pair around the batch, so each launch also pays the previous
    one's dirty-line write-back -- reported beside the flushed per-step mean."""
    import torch
    import paper_2505_11329_b200 as tw
    x, r, w, out, rout = bufs
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for _ in range(3):
            tw.rmsnorm_residual(x, r, w, EPS, residual_out=rout, out=out, stream=stream)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(steps):
        tw.rmsnorm_residual(x, r, w, EPS, residual_out=rout, out=out, stream=stream)
    e.record(stream)
    torch.cuda.synchronize()
    return 1e3 * s.elapsed_time(e) / steps


def dropin_f32_e2e(T, H, steps):
    """The reference's own C++ API and dtype through the drop-in:
    weavesim::rmsnorm_residual(TokenMatrix fp32, ...) from
    build/bench/dropin_bench (tools/dropin_bench.cpp, linked against
    libweavesim_b200.so) -- host fp32 matrices in and out, the reference's
    validation order, H2D | K2 | D2H inside; wall clock per call."""
    exe = os.path.join(ROOT, "build", "bench", "dropin_bench")
    if not os.path.exists(exe):
        return {"error": f"{exe} not built (make benchtools)"}
    try:
        p = subprocess.run([exe, "rmsnorm", str(T), str(H), "2", str(steps)], capture_output=True, text=True,
                           timeout=600)
        d = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    except Exception as exc:  # noqa: BLE001 -- reported, not fatal
        return {"error": str(exc)[:200]}
    return {"value": round(1e3 * d["median_ms"], 1), "unit": UNIT, "dtype": "f32",
            "h2d_bytes_per_step": d["h2d_bytes"], "d2h_bytes_per_step": d["d2h_bytes"], "steps": steps,
            "stat": "median wall time per call", "mean": round(1e3 * d["mean_ms"], 1),
            "min": round(1e3 * d["min_ms"], 1), "max": round(1e3 * d["max_ms"], 1),
            "path": "weavesim::rmsnorm_residual (reference C++ API, proj/include/weavesim/numerics.hpp:42-43) "
                    "linked against libweavesim_b200.so: fp32 TokenMatrix in/out, same config and dtype as "
                    "--impl reference"}


def dropin_fused_f32(world, T, H, steps):
    """The reference's TP operator through the drop-in: weavesim::
    fused_allreduce_rmsnorm(RankGroup&, NormParams, ShardMap, parallel=true)
    with `world` fp32 ranks (tools/dropin_bench.cpp fused), the ranks
    co-located on this one GPU (K1 over PEER) -- host matrices in and out."""
    exe = os.path.join(ROOT, "build", "bench", "dropin_bench")
    if not os.path.exists(exe):
        return {"error": f"{exe} not built (make benchtools)"}
    try:
        p = subprocess.run([exe, "fused", str(world), str(T), str(H), "2", str(steps)], capture_output=True,
                           text=True, timeout=600)
        d = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    except Exception as exc:  # noqa: BLE001 -- reported, not fatal
        return {"error": str(exc)[:200]}
    return {"value": round(1e3 * d["median_ms"], 1), "unit": UNIT, "dtype": "f32", "world": world, "T": T, "H": H,
            "steps": steps, "stat": "median wall time per call", "min": round(1e3 * d["min_ms"], 1),
            "max": round(1e3 * d["max_ms"], 1)}


def k2_traffic():
    """DRAM bytes per K2 launch from the newest committed ncu --set full capture."""
    for name in ("k2_ncu_r02.json", "k2_ncu_r01.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                return json.load(f).get("dram_bytes_per_launch"), name
        except Exception:
            continue
    return None, None


def run_ours_single(args):
    import torch
    T, H = args.tokens, args.hidden
    torch.cuda.set_device(0)
    flush = L2Flush("cuda:0")
    peak, peak_kind = measured_hbm_peak()
    all_cpus = os.sched_getaffinity(0)
    numa = bind_to_gpu_numa(0)
    with ClockSampler(0) as clk:
        t0 = time.perf_counter()
        times_ms, bufs = k2_timed(T, H, args.steps, args.warmup, flush)
        e2e = k2_e2e(T, H, bufs, max(3, min(args.steps, 20)))
        wall = time.perf_counter() - t0
    e2e_f32 = None if args.quick else dropin_f32_e2e(T, H, max(3, min(args.steps, 10)))  # same host binding
    e2e_cabi_f32 = None if args.quick else k2_e2e(T, H, bufs, max(3, min(args.steps, 10)), torch.float32)
    os.sched_setaffinity(0, all_cpus)  # the CPU baseline below uses every host core
    avg_us = 1e3 * sum(times_ms) / len(times_ms)
    alg_bytes = 4 * T * H * 2 + 4 * H  # read input+residual, write residual_out+output (bf16) + fp32 weight
    achieved = alg_bytes / (avg_us * 1e-6) / 1e9
    traffic, traffic_src = k2_traffic()
    line = {
        "metric": METRIC, "value": round(avg_us, 3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(avg_us / 1e3, 6), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: U(-1,1) bf16 input/residual, U(0.5,1.5) fp32 weight",
        "config": {"workload": f"TP=1 fused residual-add+RMSNorm (kernel K2), {T} tok x {H} hid bf16 "
                               "(Qwen2.5-72B / Llama-3.3-70B layer-boundary shape, BASELINE configs[2] at TP=1)",
                   "tokens": T, "hidden": H, "tp": 1, "sm_budget": "whole GPU (148 SMs)", "l2": FLUSH_NOTE},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                     "alg_bytes_per_launch": alg_bytes, "traffic": traffic, "traffic_source": traffic_src},
        "e2e": dict(e2e, host_binding=numa),
        "gpu_launches": args.steps,
        "kernel_us": {"mean": round(avg_us, 3), "median": round(1e3 * statistics.median(times_ms), 3),
                      "min": round(1e3 * min(times_ms), 3), "max": round(1e3 * max(times_ms), 3),
                      "back_to_back_no_flush": round(k2_back_to_back(bufs, args.steps), 3),
                      "after_dirty_l2": round(k2_after_dirty_l2(bufs, args.steps), 3),
                      "after_dirty_l2_note": "each step after a 256 MiB write (L2 full of a producer's dirty "
                                             "lines, their write-back inside the event pair); the value above "
                                             "uses the write+read flush (clean L2)"},
        "clocks": clk.summary(),
        "parity": k2_parity(bufs),
    }
    if not args.quick:
        line["e2e_dropin_f32"] = dict(e2e_f32, host_binding=numa)
        # the TP path through the reference's own API: N fp32 ranks co-located on this GPU
        line["dropin_fused_allreduce_rmsnorm_f32"] = {
            f"tp{n}": dropin_fused_f32(n, 1024, H, max(3, min(args.steps, 5))) for n in (2, 8)}
        line["dropin_fused_note"] = ("weavesim::fused_allreduce_rmsnorm(parallel=true) through libweavesim_b200.so, "
                                     "1024 tok x H fp32, N ranks co-located on this one GPU (K1 over PEER, not "
                                     "NVLink); the reference's own CPU path at the same N is cpu_baseline."
                                     "fused_allreduce_rmsnorm_us")
        # the reference's dtype through the C-ABI over pinned buffers (no TokenMatrix vectors)
        line["e2e_f32"] = dict(e2e_cabi_f32, dtype="f32", host_binding=numa,
                               path="tw_rmsnorm_residual_host (C-ABI via ctypes), TW_F32: pinned fp32 host "
                                    "input/residual -> chunked H2D | K2 (fp32) | D2H -> pinned fp32 output/residual_out; "
                                    "same dtype and config as --impl reference")
        sweep = {}
        for t in (256, 1024, 2048, 4096, 8192, 16384):
            ts, _ = k2_timed(t, H, 20, 3, flush, seed=1)
            us = 1e3 * statistics.median(ts)
            sweep[str(t)] = {"us": round(us, 2), "hbm_gbs": round((4 * t * H * 2) / us / 1e3, 1),
                             "frac": round((4 * t * H * 2) / us / 1e3 / peak, 3)}
        line["tp1_sweep"] = sweep
        line["unfused_torch_add_rmsnorm_us"] = unfused_torch(T, H, flush)
        # simulated ranks share this GPU: the whole GPU split between them (the
        # library clamps the budget to what its engine can co-schedule)
        line["k1_colocated_peer_us"] = {f"tp{n}": k1_colocated(T, H, n, 296 // n, flush) for n in (2, 4, 8)}
        line["k1_colocated_note"] = ("N simulated ranks on this one GPU (PEER): HBM-bound data-movement stand-in, "
                                     "not an NVLink number")
        # the weave: one Llama-3.3-70B layer at TP = 8 per-GPU
        # GEMM shapes, T = 8192, boundary op K2 (the one-GPU stand-in for K1)
        try:
            from paper_2505_11329_b200 import weave
            r = weave.LayerRunner("llama-70b", tp=8, max_tokens=T)
            a, _, _, _ = weave.make_split_plan(T, threshold=r.threshold)
            line["weave_llama70b_tp8_shapes_us"] = {
                "T": T, "prefix": a, "unfused": round(r.run(T, "unfused", layers=6), 1),
                "fuseonly": round(r.run(T, "fuseonly", layers=6), 1),
                "tokenweave_by_boundary_sms": {str(b): round(r.run(T, "tokenweave", prefix=a, boundary_sms=b,
                                                                   layers=6), 1) for b in (16, 32, 64)},
                "nocomm": round(r.run(T, "nocomm", layers=6), 1),
                "cublas_version": r.cublas_version,
                "note": "per-layer device time, eager launches, every boundary budget reported (none selected); "
                        "GEMMs are cuBLAS load (not product); boundary op = K2 on one GPU"}
            r.close()
        except Exception as exc:  # libtw_weave / cuBLAS unavailable: report, do not fail the bench
            line["weave_llama70b_tp8_shapes_us"] = {"error": str(exc)[:200]}
        threads = os.cpu_count() or 1
        cpu_ms = reference_rmsnorm_each_ms(T, H, threads, 4)[1:]
        # the reference's API as one caller uses it: ONE rmsnorm_residual call on one thread
        one_ms = reference_rmsnorm_each_ms(T, H, 1, 2)[1:]
        line["cpu_baseline"] = {
            "value": round(1e3 * statistics.median(cpu_ms), 1), "unit": UNIT, "cores": threads, "kind": "reference",
            "cpu": cpu_model(),
            "sample": f"full workload: weavesim::rmsnorm_residual (oracle/_ref, reference sources compiled "
                      f"unmodified) on {T}x{H} fp32, token rows chunked over {threads} threads (as "
                      f"--impl reference), median of 3 after one warm-up; ms {[round(x, 1) for x in cpu_ms]}",
            "single_call_1thread_us": round(1e3 * one_ms[0], 1),
            "fused_allreduce_rmsnorm_us": {  # the reference's TP operator, parallel=true (one thread per rank)
                f"tp{n}": round(1e3 * oracle_fused_ms(n, 1024, H), 1) for n in (2, 8)},
            "single_call_note": "one weavesim::rmsnorm_residual call on the whole matrix (the API is single-threaded; "
                                "the drop-in's e2e_dropin_f32 is the same single call)"}
    line["wall_s"] = round(wall, 2)
    print(json.dumps(line), flush=True)
    return 0


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` without torchrun: spawn the N ranks ourselves
    (same command line under torch.distributed.run, 127.0.0.1 rendezvous)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=8192)
    ap.add_argument("--sm-budget", type=int, default=8, help="K1 CTAs (= SMs) per rank (N>1)")
    ap.add_argument("--gather-residual", action="store_true", help="K1 G=2 (N>1)")
    ap.add_argument("--transport", choices=["nvls", "peer", "auto"], default="auto",
                    help="N>1 on distinct GPUs: auto (default: NVLS, or PEER over NVLink with the line labelled "
                         "and a stderr warning when the multicast object cannot be built), nvls (fail if "
                         "unavailable) or peer")
    ap.add_argument("--quick", action="store_true", help="skip sweeps/baselines (profiling runs)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    # our arm: the package loads the CUDA toolkit's cuBLAS before torch
    # (paper_2505_11329_b200/_lib.py), so it is imported before anything else
    import paper_2505_11329_b200  # noqa: F401
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        from tools.bench_tp import run_tp
        return run_tp(args)
    if args.gpus > 1:
        return relaunch_under_torchrun(args)
    return run_ours_single(args)


if __name__ == "__main__":
    sys.exit(main())
