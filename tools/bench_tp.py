"""TP = N leg of bench.py: one process per GPU (torchrun), kernel K1 (fused
AllReduce + residual-add + RMSNorm) over the multi-process communicator
(tw_comm_create_mp), strong scaling at the same T.

Transport.  Ranks on distinct GPUs run the NVLS kernel (multimem ld_reduce /
st over an NVSwitch multicast object).  If the multicast object cannot be
built (no NVSwitch multicast in the box or container), the default `auto`
falls back collectively to K1's PEER engine over NVLink P2P -- still a
multi-GPU NVLink measurement of the fused kernel, but not the NVLS one -- and
says so: a warning on stderr, `config.transport` = "peer", a top-level
`nvls_unavailable` key and PEER's algorithmic bytes in the roofline.
`--transport nvls` fails instead.  Ranks sharing one GPU (the
two-process test topology of a one-GPU box) cannot bind a multicast object;
they run PEER and the line says "colocated": such numbers are plumbing checks,
not NVLink measurements.

Parity.  Before timing, one K1 launch on the line's own inputs is checked
against a torch fp32 restatement on every rank (`parity` in the line).

Timing.  Each step: L2 flush on the rank's stream (a 256 MiB write + read,
outside the events), a device-side cross-rank sync (a one-element NCCL
all_reduce on the same stream, so every rank's K1 starts within the
collective's exit skew rather than a host barrier's), then CUDA events around
the op on the launching stream.  `value` = max over ranks of the mean
per-step time.  SM budget defaults to 8 CTAs (one per SM) per rank.

The host-side pieces (rendezvous id, max-over-ranks, algorithmic bytes) are
exercised on CPU by tests/test_mp_cpu.py with the gloo backend."""
from __future__ import annotations

import ctypes
import json
import os
import re
import statistics
import subprocess
import sys
import time
import uuid

EPS = 1e-5
METRIC = "fused AR+RMSNorm µs & NVLink GB/s, 1024–8192 tok × 8192 hid, TP=1/2/4/8"
NVLINK_PEAK_GBS = 900.0  # per direction per GPU (NVLink 5, 18 links); SURVEY.md §8d


def rendezvous_id(dist) -> str:
    """A job-unique id chosen by rank 0 and broadcast to every rank."""
    obj = [f"{os.environ.get('MASTER_PORT', '0')}-{uuid.uuid4().hex[:12]}" if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(value: float, dist, device=None) -> float:
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def algorithmic_nvlink_bytes(T: int, H: int, world: int, gather_residual: bool, elem: int = 2) -> float:
    """Per GPU per direction, NVLS: B = S*(G + 1/N), S = T*H*elem.
    Ingress: S/N reduced rows returned by ld_reduce + G*S multicast stores from
    every rank; egress: S read by the switch for the reductions + G*S/N."""
    S = T * H * elem
    G = 2 if gather_residual else 1
    return S * (G + 1.0 / world)


def algorithmic_peer_bytes(T: int, H: int, world: int, gather_residual: bool, elem: int = 2) -> float:
    """Per GPU per direction, PEER (P2P loads/stores over NVLink): B = S*(1+G)*(N-1)/N.
    Ingress: this rank's shard of every peer's partial, (N-1)*S/N; egress:
    G*(N-1)*S/N of normed output (and r') stored into every peer."""
    S = T * H * elem
    G = 2 if gather_residual else 1
    return S * (1 + G) * (world - 1) / world


def alg_bytes(transport: str, T: int, H: int, world: int, gather_residual: bool) -> float:
    if transport == "nvls":
        return algorithmic_nvlink_bytes(T, H, world, gather_residual)
    return algorithmic_peer_bytes(T, H, world, gather_residual)


def nvlink_counters(device_index: int):
    """(tx_bytes, rx_bytes) summed over the GPU's NVLink links from the
    driver's data counters (`nvidia-smi nvlink -gt d`), or None."""
    try:
        from bench import smi_id
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", smi_id(device_index)], capture_output=True,
                             text=True, timeout=30).stdout
    except (OSError, subprocess.SubprocessError):
        return None
    return parse_nvlink_counters(out)


def parse_nvlink_counters(out: str):
    """Sum the per-link "Data Tx/Rx: N KiB" lines of `nvidia-smi nvlink -gt d`."""
    tx = rx = 0
    seen = False
    for m in re.finditer(r"Link \d+: Data (Tx|Rx): (\d+) KiB", out):
        seen = True
        if m.group(1) == "Tx":
            tx += int(m.group(2)) * 1024
        else:
            rx += int(m.group(2)) * 1024
    return (tx, rx) if seen else None


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class _Rank:
    """This process's rank of the TP communicator plus its buffers and streams."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        import paper_2505_11329_b200 as tw
        from paper_2505_11329_b200 import _lib
        self.tw, self._lib, self.torch, self.dist = tw, _lib, torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", args.gpus))
        self.rank = int(os.environ.get("RANK", "0"))
        ndev = torch.cuda.device_count()
        self.colocated = ndev < self.world
        self.local = int(os.environ.get("LOCAL_RANK", self.rank)) % max(ndev, 1)
        torch.cuda.set_device(self.local)
        if not self.colocated:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{self.local}"))
            self.red_device = "cuda"
        else:  # ranks share GPUs (test topology): NCCL refuses duplicate devices
            dist.init_process_group("gloo")
            self.red_device = None
        self.T, self.H = args.tokens, args.hidden
        want = {"nvls": _lib.TW_TRANSPORT_NVLS, "peer": _lib.TW_TRANSPORT_PEER, "auto": _lib.TW_TRANSPORT_AUTO}
        tname = args.transport if not self.colocated else "peer"
        rid = rendezvous_id(dist)
        h = ctypes.c_void_p()
        st = _lib.lib.tw_comm_create_mp(self.world, self.rank, self.local, self.T * self.H * 2, rid.encode(),
                                        want[tname], ctypes.byref(h))
        if st != 0:
            raise RuntimeError(f"rank {self.rank}: tw_comm_create_mp({tname}) failed: "
                               f"{_lib.lib.tw_last_error().decode()} -- no fallback: a TP line must be an "
                               f"{tname.upper()} measurement (use --transport auto to allow PEER)")
        self.h = h
        wsz, tr, nb = ctypes.c_int(), ctypes.c_int(), ctypes.c_size_t()
        _lib.check(_lib.lib.tw_comm_info(h, ctypes.byref(wsz), ctypes.byref(tr), ctypes.byref(nb)))
        self.transport = _lib.TRANSPORT_NAMES[tr.value]
        self.nvls_unavailable = None
        if not self.colocated and self.transport != "nvls":
            self.nvls_unavailable = (f"transport {tname}: the NVLS multicast object was not available on this box; "
                                     f"K1 ran its PEER engine over NVLink P2P")
            if self.rank == 0:
                print(f"WARNING: {self.nvls_unavailable} -- the TP line is a PEER number, not NVLS",
                      file=sys.stderr, flush=True)
        self.stream = torch.cuda.Stream()
        self.tiny = torch.zeros(1, device="cuda")

    def buffer(self, which, T):
        tw, _lib, torch = self.tw, self._lib, self.torch
        p = ctypes.c_void_p()
        _lib.check(_lib.lib.tw_comm_buffer(self.h, self.rank, which, ctypes.byref(p)))
        raw = torch.as_tensor(tw._DevBuf(p.value, (T * self.H,), "<i2"), device="cuda")
        return raw.view(torch.bfloat16).view(T, self.H)

    def sync(self):
        """Device-side rendezvous of every rank's stream (NCCL), or a host
        barrier for co-located (gloo) ranks."""
        if self.red_device == "cuda":
            with self.torch.cuda.stream(self.stream):
                self.dist.all_reduce(self.tiny)
        else:
            self.torch.cuda.synchronize()
            self.dist.barrier()

    def fused(self, T, residual, weight, budget, gather=False):
        _lib = self._lib
        ranges = self.tw.token_shard_map(T, self.world)
        flat = (ctypes.c_int64 * (2 * self.world))(*[v for rg in ranges for v in rg])
        flags = _lib.TW_GATHER_RESIDUAL if gather else 0
        _lib.check(_lib.lib.tw_fused_allreduce_rmsnorm(self.h, T, self.H, 0, flat, residual.data_ptr(),
                                                       weight.data_ptr(), EPS, _lib.TW_BF16, budget, flags,
                                                       self.stream.cuda_stream))

    def timed(self, fn, steps, flush, warmup=3):
        """Per-step CUDA-event times (ms) of fn() on this rank's stream, each
        step after an L2 flush and a cross-rank sync (outside the events)."""
        torch = self.torch
        for i in range(warmup):
            with torch.cuda.stream(self.stream):
                flush(i)
            self.sync()
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for i in range(steps):
            with torch.cuda.stream(self.stream):
                flush(i)
            self.sync()
            ev[i][0].record(self.stream)
            fn()
            ev[i][1].record(self.stream)
        torch.cuda.synchronize()
        self._lib.check(self._lib.lib.tw_comm_check(self.h))
        return [a.elapsed_time(b) for a, b in ev]

    def max_mean_us(self, times_ms):
        return max_over_ranks(1e3 * sum(times_ms) / len(times_ms), self.dist, self.red_device)

    def close(self):
        self._lib.lib.tw_comm_destroy(self.h)
        self.dist.barrier()
        self.dist.destroy_process_group()


def run_tp(args):
    import torch

    from bench import ClockSampler, L2Flush
    R = _Rank(args)
    tw, _lib = R.tw, R._lib
    world, rank, T, H = R.world, R.rank, R.T, R.H
    gather = bool(args.gather_residual)
    budget = int(args.sm_budget)
    flush = L2Flush("cuda")
    b, e = tw.token_shard_map(T, world)[rank]
    g = torch.Generator(device="cuda").manual_seed(rank)
    inp = R.buffer(_lib.TW_BUF_INPUT, T)
    inp.copy_((torch.rand(T, H, device="cuda", generator=g) - 0.5).to(torch.bfloat16))
    residual = (torch.rand(max(e - b, 1), H, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    # the RMSNorm weight is replicated (as a TP model's is): the same draw on every rank
    weight = torch.rand(H, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1 << 20)) + 0.5

    # ---- parity first: one K1 call against a torch fp32 restatement ----
    parity = check_parity(R, inp, residual, weight, T, budget, gather)

    # ---- the headline: K1 at T, `budget` SMs, per-step events ----
    clk = ClockSampler(R.local) if rank == 0 else None
    if clk:
        clk.__enter__()
    nvl0 = nvlink_counters(R.local) if rank == 0 and not R.colocated else None
    t0 = time.perf_counter()
    times = R.timed(lambda: R.fused(T, residual, weight, budget, gather), args.steps, flush,
                    warmup=max(args.warmup, 3))
    wall = time.perf_counter() - t0
    nvl1 = nvlink_counters(R.local) if rank == 0 and not R.colocated else None
    if clk:
        clk.__exit__(None, None, None)
    us = R.max_mean_us(times)
    us_med = max_over_ranks(1e3 * statistics.median(times), R.dist, R.red_device)
    n_launch = args.steps + max(args.warmup, 3)  # the counters span the warm-up steps too

    # ---- e2e: pinned host buffers through the same C-ABI call ----
    h_in = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
    h_in.copy_(inp.cpu())
    h_res = residual.cpu().pin_memory()
    h_out = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
    h_res_out = torch.empty_like(h_res).pin_memory()
    out_buf = R.buffer(_lib.TW_BUF_OUTPUT, T)
    dev_res = residual.clone()

    def e2e_step():
        with torch.cuda.stream(R.stream):
            inp.copy_(h_in, non_blocking=True)
            dev_res.copy_(h_res, non_blocking=True)
        R.fused(T, dev_res, weight, budget, gather)
        with torch.cuda.stream(R.stream):
            h_out.copy_(out_buf, non_blocking=True)
            h_res_out.copy_(dev_res, non_blocking=True)

    e2e_steps = max(3, min(args.steps, 20))
    e2e_times = R.timed(e2e_step, e2e_steps, lambda i: None, warmup=2)
    e2e_us = max_over_ranks(1e3 * statistics.median(e2e_times), R.dist, R.red_device)
    shard_bytes = (e - b) * H * 2

    extra = {}
    if not args.quick:
        # SM-budget sweep at T (configs[4]) and token sweep at the budget (configs[1]/[2])
        sweep_b = {}
        for bud in (2, 4, 8, 16):
            ts = R.timed(lambda: R.fused(T, residual, weight, bud, gather), 10, flush)
            u = R.max_mean_us(ts)
            sweep_b[str(bud)] = {"us": round(u, 2),
                                 "nvlink_gbs": round(alg_bytes(R.transport, T, H, world, gather) / u / 1e3, 1)}
        extra["sm_budget_sweep"] = sweep_b
        sweep_t = {}
        for t in (256, 1024, 2048, 4096, 8192):
            if t > T:
                continue
            ts = R.timed(lambda: R.fused(t, residual, weight, budget, gather), 10, flush)
            u = R.max_mean_us(ts)
            sweep_t[str(t)] = {"us": round(u, 2),
                               "nvlink_gbs": round(alg_bytes(R.transport, t, H, world, gather) / u / 1e3, 1)}
        extra["token_sweep"] = sweep_t
        ts = R.timed(lambda: R.fused(T, residual, weight, budget, True), 10, flush)
        extra["gather_residual_G2_us"] = round(R.max_mean_us(ts), 2)
        # unfused baselines on the same box: AllReduce
        # over the full T, then K2 over the full T on every rank
        summed = R.buffer(_lib.TW_BUF_OUTPUT, T)
        full_res = torch.zeros(T, H, device="cuda", dtype=torch.bfloat16)
        normed = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
        base = {}
        for kb in (16, 32):
            def k3_k2(kb=kb):
                _lib.check(_lib.lib.tw_allreduce(R.h, T, H, 0, _lib.TW_BF16, kb, R.stream.cuda_stream))
                tw.rmsnorm_residual(summed, full_res, weight, residual_out=full_res, out=normed, stream=R.stream)
            base[f"k3_allreduce_{kb}sm_plus_k2_us"] = round(R.max_mean_us(R.timed(k3_k2, 10, flush)), 2)
        if R.red_device == "cuda":
            nccl_buf = torch.zeros(T, H, device="cuda", dtype=torch.bfloat16)

            def nccl_k2():
                with torch.cuda.stream(R.stream):
                    R.dist.all_reduce(nccl_buf)
                tw.rmsnorm_residual(nccl_buf, full_res, weight, residual_out=full_res, out=normed, stream=R.stream)
            base["nccl_allreduce_plus_k2_us"] = round(R.max_mean_us(R.timed(nccl_k2, 10, flush)), 2)
        extra["unfused_baselines"] = base
        # the weave at TP = N: one Llama-3.3-70B layer at this
        # TP's per-GPU GEMM shapes with K1 as the boundary op (tw_weave_create_tp)
        try:
            from paper_2505_11329_b200 import weave
            r = weave.LayerRunner("llama-70b", tp=world, max_tokens=T, comm=R.h)
            a, _, _, mode = weave.make_split_plan(T, threshold=r.threshold)
            lay = {"T": T, "prefix": a if mode == 2 else None, "boundary_sms": budget}
            for name, kw in (("unfused", {}), ("fuseonly", {}), ("nocomm", {}),
                             ("tokenweave", {"prefix": a, "boundary_sms": budget})):
                if name == "tokenweave" and mode != 2:
                    continue
                us_l = r.run(T, name, layers=4, **kw)
                lay[name] = round(max_over_ranks(us_l, R.dist, R.red_device), 1)
            lay["cublas_version"] = r.cublas_version
            lay["note"] = ("per-layer device time, max over ranks, eager; GEMMs are cuBLAS load (not product); "
                           "unfused = K3 AllReduce + add + RMSNorm on every rank")
            r.close()
            extra["weave_llama70b_layer_us"] = lay
        except Exception as exc:  # noqa: BLE001 -- reported, never fatal
            extra["weave_llama70b_layer_us"] = {"error": str(exc)[:200]}

    # ---- the reference CPU path at the same N (rank 0; others wait) ----
    cpu = None
    if rank == 0:
        cpu = cpu_baseline_fused(world, T, H)
    R.dist.barrier()

    alg = alg_bytes(R.transport, T, H, world, gather)
    alg_formula = "S*(G+1/N), S = T*H*2 (NVLS)" if R.transport == "nvls" else "S*(1+G)*(N-1)/N, S = T*H*2 (PEER)"
    achieved = alg / (us * 1e-6) / 1e9
    traffic = None
    if nvl0 and nvl1:
        tx, rx = (nvl1[0] - nvl0[0]) / n_launch, (nvl1[1] - nvl0[1]) / n_launch
        traffic = {"tx_bytes_per_launch": round(tx), "rx_bytes_per_launch": round(rx),
                   "max_dir_bytes_per_launch": round(max(tx, rx)),
                   "source": "nvidia-smi nvlink -gt d (driver link data counters, rank 0's GPU, "
                             f"{n_launch} launches incl. warm-up)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(us, 3), "unit": "us", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(us / 1e3, 6), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic U(-0.5,0.5) bf16 partial sums and residual, U(0.5,1.5) fp32 weight",
            "config": {"workload": f"TP={world} fused AllReduce+residual+RMSNorm (K1 over {R.transport.upper()}), "
                                   f"{T} tok x {H} hid bf16 (Llama-3.3-70B / Qwen2.5-72B layer boundary)",
                       "tokens": T, "hidden": H, "tp": world, "sm_budget": budget, "gather_residual": gather,
                       "transport": R.transport, "colocated": R.colocated,
                       "l2": "flushed before every step (256 MiB write + read, outside the events); "
                             "ranks synced on the device (NCCL) before each step"},
            "roofline": {"bound": "nvlink" if not R.colocated else "hbm",
                         "achieved": round(achieved, 1), "peak": NVLINK_PEAK_GBS, "unit": "GB/s",
                         "frac": round(achieved / NVLINK_PEAK_GBS, 4),
                         "peak_kind": "nominal NVLink 5 per direction per GPU",
                         "alg_bytes_per_launch": alg, "alg_bytes_formula": alg_formula,
                         "traffic": traffic},
            "kernel_us": {"mean": round(us, 3), "median": round(us_med, 3)},
            "sms_consumed": budget,
            "e2e": {"value": round(e2e_us, 2), "unit": "us",
                    "h2d_bytes_per_step": T * H * 2 + shard_bytes, "d2h_bytes_per_step": T * H * 2 + shard_bytes,
                    "per": "rank (every rank moves its own partial in and the replicated output out)",
                    "path": "pinned host partial + residual shard -> H2D -> tw_fused_allreduce_rmsnorm (C-ABI) -> "
                            "D2H output + residual shard; max over ranks of the median step"},
            "gpu_launches": args.steps, "wall_s": round(wall, 3),
            "clocks": clk.summary() if clk else None,
            "cpu_baseline": cpu,
        }
        line["parity"] = parity
        if R.nvls_unavailable:
            line["nvls_unavailable"] = R.nvls_unavailable
        if R.colocated:
            line["note"] = ("ranks share one GPU: PEER transport, time-sliced -- a plumbing check, "
                            "not an NVLink measurement")
        line.update(extra)
        print(json.dumps(line), flush=True)
    R.close()
    return 0


def check_parity(R, inp, residual, weight, T, budget, gather):
    """One K1 launch on the line's own inputs against a torch fp32
    restatement of fused_allreduce_rmsnorm (proj/src/collectives.cpp:134-153):
    v = sum over ranks of the bf16 partials (a torch.distributed all_reduce
    in fp32: the checker, not the measured path), r' = v + residual,
    out = r' * rsqrt(mean(r'^2) + eps) * w.  bf16 bar as the tests': |err| <=
    2e-2 * |want| + 2e-2 (the hardware reduction order is not fixed and v is
    rounded to bf16 before the add).  Checks the replicated output on every
    rank and the rank's own r' rows; restores the residual afterwards."""
    torch = R.torch
    b, e = R.tw.token_shard_map(T, R.world)[R.rank]
    res0 = residual.clone()
    R.sync()
    R.fused(T, residual, weight, budget, gather)
    torch.cuda.synchronize()
    R._lib.check(R._lib.lib.tw_comm_check(R.h))
    out = R.buffer(R._lib.TW_BUF_OUTPUT, T).float()
    dev = "cuda" if R.red_device == "cuda" else "cpu"
    v = inp.float().to(dev)
    R.dist.all_reduce(v)
    full_res = torch.zeros(T, R.H, dtype=torch.float32, device=dev)
    if e > b:
        full_res[b:e] = res0[: e - b].float().to(dev)
    R.dist.all_reduce(full_res)
    r = (v + full_res).to(out.device)
    want = r * torch.rsqrt(r.pow(2).mean(dim=1, keepdim=True) + EPS) * weight.float()

    def excess(got, ref):  # > 0 where the bf16 bar is broken
        return float(((got - ref).abs() - (2e-2 * ref.abs() + 2e-2)).max()) if got.numel() else -1.0

    worst_out = excess(out, want)
    worst_res = excess(residual[: e - b].float(), r[b:e]) if e > b else -1.0
    max_abs = float((out - want).abs().max())
    residual.copy_(res0)
    torch.cuda.synchronize()
    worst = max_over_ranks(max(worst_out, worst_res), R.dist, R.red_device)
    max_abs = max_over_ranks(max_abs, R.dist, R.red_device)
    return {"ok": worst <= 0.0, "max_abs_err_output": round(max_abs, 5),
            "bar": "|err| <= 2e-2*|want| + 2e-2 (bf16), output on every rank and each rank's r' rows",
            "checker": "torch fp32 restatement; partials summed by a torch.distributed all_reduce (not timed)",
            "T": T, "gather_residual": gather}


def cpu_baseline_fused(world, T, H, iters=3):
    """The reference's weavesim::fused_allreduce_rmsnorm (oracle/_ref: the
    reference sources compiled unmodified) with parallel=true -- one
    std::thread per rank, its fastest mode -- on the full T x H fp32 workload,
    validation included, median of `iters`."""
    try:
        import oracle  # cpu_baseline leg only
        ref = oracle.RefLib()
        ms = ref.time_fused(world, T, H, True, iters, each=True)
        return {"value": round(1e3 * statistics.median(ms), 1), "unit": "us", "cores": world, "kind": "reference",
                "cpu": cpu_model(), "host_threads_available": os.cpu_count(),
                "sample": f"full workload ({world} ranks x {T}x{H} fp32), parallel=true (one std::thread per "
                          f"rank), median of {iters}; per-iteration ms {[round(x, 1) for x in ms]}"}
    except Exception as exc:  # noqa: BLE001 -- reported, never fatal
        return {"value": None, "unit": "us", "cores": 0, "kind": "reference", "sample": f"unavailable: {exc}"[:200]}
