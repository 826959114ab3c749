"""BASELINE configs[2]/[4] at TP = N (torchrun, one process per GPU):
token sweep x SM-budget sweep of the fused op (K1, G = 1 and G = 2) next to
the unfused baselines on the same box -- our one-shot AllReduce (K3) + K2, and
NCCL all_reduce + K2 (when ranks are on distinct GPUs).  Every number is the
median of per-launch CUDA-event times, max over ranks.  Writes JSON and the
reference's microbench CSV layout (proj/README.md:60-62).

  python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
      tools/sweep_tp.py --out profiles/sweep_tp8.json
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--hidden", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2505_11329_b200 as tw
    from paper_2505_11329_b200 import _lib
    from tools.bench_tp import algorithmic_nvlink_bytes, max_over_ranks, rendezvous_id

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    ndev = torch.cuda.device_count()
    local = int(os.environ.get("LOCAL_RANK", rank)) % max(ndev, 1)
    torch.cuda.set_device(local)
    distinct = ndev >= world
    dist.init_process_group("nccl" if distinct else "gloo")
    red_dev = "cuda" if distinct else None
    H = args.hidden
    tokens = [4, 16, 64, 256, 512, 1024, 2048, 4096, 8192, 16384]
    budgets = [2, 4, 8, 16]
    if args.quick:
        tokens, budgets = [64, 1024], [8]
    Tmax = max(tokens)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib.tw_comm_create_mp(world, rank, local, Tmax * H * 2, rendezvous_id(dist).encode(),
                                          _lib.TW_TRANSPORT_AUTO, ctypes.byref(h)))
    tr = ctypes.c_int()
    _lib.check(_lib.lib.tw_comm_info(h, None, ctypes.byref(tr), None))
    p = ctypes.c_void_p()
    _lib.check(_lib.lib.tw_comm_buffer(h, rank, _lib.TW_BUF_INPUT, ctypes.byref(p)))
    inp = torch.as_tensor(tw._DevBuf(p.value, (Tmax * H,), "<i2"), device="cuda").view(torch.bfloat16)
    inp.copy_(torch.randn(Tmax * H, device="cuda").to(torch.bfloat16) * 0.1)
    _lib.check(_lib.lib.tw_comm_buffer(h, rank, _lib.TW_BUF_OUTPUT, ctypes.byref(p)))
    outbuf = torch.as_tensor(tw._DevBuf(p.value, (Tmax * H,), "<i2"), device="cuda").view(torch.bfloat16)
    residual = torch.randn(Tmax, H, device="cuda", dtype=torch.bfloat16)
    full_res = torch.randn(Tmax, H, device="cuda", dtype=torch.bfloat16)
    normed = torch.empty(Tmax, H, device="cuda", dtype=torch.bfloat16)
    weight = torch.ones(H, device="cuda")
    nccl_buf = torch.randn(Tmax, H, device="cuda", dtype=torch.bfloat16) if distinct else None
    stream = torch.cuda.current_stream().cuda_stream

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        ts = []
        for _ in range(args.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        return max_over_ranks(1e3 * statistics.median(ts), dist, red_dev)

    rows = []
    for T in tokens:
        ranges = tw.token_shard_map(T, world)
        flat = (ctypes.c_int64 * (2 * world))(*[v for rg in ranges for v in rg])
        row = {"T": T, "message_bytes": T * H * 2}
        for b in budgets:
            for g, flag in ((1, 0), (2, _lib.TW_GATHER_RESIDUAL)):
                us = timed(lambda: _lib.check(_lib.lib.tw_fused_allreduce_rmsnorm(
                    h, T, H, 0, flat, residual.data_ptr(), weight.data_ptr(), 1e-5, _lib.TW_BF16, b, flag, stream)))
                row[f"fused_G{g}_sms{b}_us"] = round(us, 2)
                row[f"fused_G{g}_sms{b}_nvlink_gbs"] = round(algorithmic_nvlink_bytes(T, H, world, g == 2) / us / 1e3,
                                                             1)
        ar = timed(lambda: _lib.check(_lib.lib.tw_allreduce(h, T, H, 0, _lib.TW_BF16, 16, stream)))
        norm = timed(lambda: tw.rmsnorm_residual(outbuf[:T * H].view(T, H), full_res[:T], weight,
                                                 residual_out=full_res[:T], out=normed[:T]))
        row["allreduce_k3_us"] = round(ar, 2)
        row["rmsnorm_us"] = round(norm, 2)
        if distinct:
            row["allreduce_nccl_us"] = round(timed(lambda: dist.all_reduce(nccl_buf[:T])), 2)
        rows.append(row)
        if rank == 0:
            print(json.dumps(row), flush=True)
    _lib.check(_lib.lib.tw_comm_check(h))
    if rank == 0:
        res = {"world": world, "hidden": H, "transport": _lib.TRANSPORT_NAMES[tr.value], "rows": rows}
        if args.out:
            with open(args.out, "w") as f:
                json.dump(res, f, indent=1)
            b = 16 if 16 in budgets else budgets[-1]
            csv = [["series", "unit"] + [str(r["T"]) for r in rows],
                   ["allreduce", "us"] + [f"{r['allreduce_k3_us']:.2f}" for r in rows],
                   ["rmsnorm", "us"] + [f"{r['rmsnorm_us']:.2f}" for r in rows],
                   ["ar_plus_rmsnorm", "us"] + [f"{r['allreduce_k3_us'] + r['rmsnorm_us']:.2f}" for r in rows],
                   ["fused", "us"] + [f"{r[f'fused_G1_sms{b}_us']:.2f}" for r in rows],
                   ["speedup", "x"] + [f"{(r['allreduce_k3_us'] + r['rmsnorm_us']) / r[f'fused_G1_sms{b}_us']:.3f}"
                                       for r in rows]]
            with open(os.path.splitext(args.out)[0] + "_microbench.csv", "w") as f:
                f.write("\n".join(",".join(c) for c in csv) + "\n")
    _lib.lib.tw_comm_destroy(h)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
