"""TP=N leg of bench.py: one process per GPU (torchrun), kernel K1 over the
multi-process NVLS communicator (tw_comm_create_mp), strong scaling at the
same T.  Timing: per-step CUDA events on the launching stream, barrier +
synchronize around the timed loop, the MAX over ranks reported by rank 0.

The host-side pieces (rendezvous id, max-over-ranks) are exercised on CPU by
tests/test_mp_cpu.py with the gloo backend."""
from __future__ import annotations

import ctypes
import json
import os
import statistics
import time
import uuid


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
    """Per GPU per direction, NVLS: B = S*(G + 1/N)."""
    S = T * H * elem
    G = 2 if gather_residual else 1
    return S * (G + 1.0 / world)


def run_tp(args):
    import torch
    import torch.distributed as dist

    import paper_2505_11329_b200 as tw
    from paper_2505_11329_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    ndev = torch.cuda.device_count()
    local = int(os.environ.get("LOCAL_RANK", rank)) % max(ndev, 1)
    torch.cuda.set_device(local)
    if ndev >= world:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        red_device = "cuda"
    else:  # ranks share GPUs (test topologies): NCCL refuses duplicate devices
        dist.init_process_group("gloo")
        red_device = None
    T, H = args.tokens, args.hidden
    gather = bool(getattr(args, "gather_residual", False))
    rid = rendezvous_id(dist)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib.tw_comm_create_mp(world, rank, local, T * H * 2, rid.encode(), _lib.TW_TRANSPORT_AUTO,
                                          ctypes.byref(h)))
    wsz, tr, nb = ctypes.c_int(), ctypes.c_int(), ctypes.c_size_t()
    _lib.check(_lib.lib.tw_comm_info(h, ctypes.byref(wsz), ctypes.byref(tr), ctypes.byref(nb)))
    transport = _lib.TRANSPORT_NAMES[tr.value]
    ranges = tw.token_shard_map(T, world)
    b, e = ranges[rank]
    flat = (ctypes.c_int64 * (2 * world))(*[v for rg in ranges for v in rg])
    g = torch.Generator(device="cuda").manual_seed(rank)
    p_in = ctypes.c_void_p()
    _lib.check(_lib.lib.tw_comm_buffer(h, rank, _lib.TW_BUF_INPUT, ctypes.byref(p_in)))
    inp = torch.as_tensor(tw._DevBuf(p_in.value, (T * H,), "<i2"), device="cuda").view(torch.bfloat16).view(T, H)
    inp.copy_((torch.rand(T, H, device="cuda", generator=g) - 0.5).to(torch.bfloat16))
    residual = (torch.rand(max(e - b, 1), H, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    weight = torch.rand(H, device="cuda", generator=g) + 0.5
    stream = torch.cuda.Stream()
    budget = int(getattr(args, "sm_budget", 16))
    if transport == "peer":
        # the P2P fallback hides NVLink load latency with more CTAs in flight
        # (no in-switch reduction: every rank's vector crosses the link)
        budget = max(budget, 48)
    flags = _lib.TW_GATHER_RESIDUAL if gather else 0

    def step():
        _lib.check(_lib.lib.tw_fused_allreduce_rmsnorm(h, T, H, 0, flat, residual.data_ptr(), weight.data_ptr(), EPS,
                                                       _lib.TW_BF16, budget, flags, stream.cuda_stream))

    EPS = 1e-5
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    wall = time.perf_counter() - t0
    _lib.check(_lib.lib.tw_comm_check(h))
    times = [s.elapsed_time(x) for s, x in zip(starts, ends)]
    us_local = 1e3 * sum(times) / len(times)
    us = max_over_ranks(us_local, dist, device=red_device)
    # Unfused baselines on the same box (not timed in `value`): our one-shot
    # AllReduce (K3) + K2 over the full T, and NCCL all_reduce + K2.
    out_p = ctypes.c_void_p()
    _lib.check(_lib.lib.tw_comm_buffer(h, rank, _lib.TW_BUF_OUTPUT, ctypes.byref(out_p)))
    summed = torch.as_tensor(tw._DevBuf(out_p.value, (T * H,), "<i2"), device="cuda").view(torch.bfloat16).view(T, H)
    full_res = torch.zeros(T, H, device="cuda", dtype=torch.bfloat16)
    normed = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)

    def timed_baseline(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(reps):
            fn()
        e.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(1e3 * s.elapsed_time(e) / reps, dist, red_device)

    def k3_k2():
        _lib.check(_lib.lib.tw_allreduce(h, T, H, 0, _lib.TW_BF16, budget, stream.cuda_stream))
        tw.rmsnorm_residual(summed, full_res, weight, residual_out=full_res, out=normed, stream=stream)

    baselines = {"k3_allreduce_plus_k2_us": round(timed_baseline(k3_k2), 2)}
    if red_device == "cuda":
        nccl_buf = torch.zeros(T, H, device="cuda", dtype=torch.bfloat16)

        def nccl_k2():
            with torch.cuda.stream(stream):
                dist.all_reduce(nccl_buf)
            tw.rmsnorm_residual(nccl_buf, full_res, weight, residual_out=full_res, out=normed, stream=stream)

        baselines["nccl_allreduce_plus_k2_us"] = round(timed_baseline(nccl_k2), 2)
    _lib.check(_lib.lib.tw_comm_check(h))
    nvl = algorithmic_nvlink_bytes(T, H, world, gather)
    achieved = nvl / (us * 1e-6) / 1e9
    if rank == 0:
        line = {
            "metric": "fused AR+RMSNorm µs & NVLink GB/s, 1024–8192 tok × 8192 hid, TP=1/2/4/8",
            "value": round(us, 3), "unit": "us", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(us / 1e3, 6), "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic U(-0.5,0.5) bf16 partial sums",
            "config": {"workload": f"TP={world} fused AllReduce+residual+RMSNorm (K1, {transport.upper()}), "
                                   f"{T} tok x {H} hid bf16",
                       "tokens": T, "hidden": H, "tp": world, "sm_budget": budget, "gather_residual": gather,
                       "transport": transport,
                       "l2": "inputs in HBM; NVLink-bound"},
            "roofline": {"bound": "nvlink", "achieved": round(achieved, 1), "peak": 900.0, "unit": "GB/s",
                         "frac": round(achieved / 900.0, 4), "peak_kind": "nominal per direction",
                         "alg_bytes_per_launch": nvl, "traffic": None},
            "gpu_launches": args.steps, "wall_s": round(wall, 3), "unfused_baselines": baselines,
        }
        print(json.dumps(line), flush=True)
    _lib.lib.tw_comm_destroy(h)
    dist.barrier()
    dist.destroy_process_group()
    return 0
