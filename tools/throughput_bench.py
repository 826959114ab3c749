"""Measured serving throughput: chunked-prefill batches
(form_batches, proj/src/workloads.cpp:68-109) run layer by layer through the
two-stream runner (tw_weave_throughput), per mode -- the reference's
simulate_throughput (:111-141) with every iteration MEASURED instead of priced.

Workloads (tests/golden/make_golden.py throughput_cases): the reference CLI's
own `throughput` defaults -- fixed-2048x128 (64 requests) and chatlike (96
lognormal requests, seed 42) at chunk 2048 (proj/src/commands.cpp:432-446) --
plus chunk-8192 variants for Llama and Mixtral.  Per workload: tokens/s of the
unfused sequential layer, fuse-only, TokenWeave (decode-only and
below-threshold batches run fuse-only, scheduler.cpp:333-341) and the no-comm
bound, each iteration = measured per-layer time x num_layers (80 for
Llama-3.3-70B, 56 for Mixtral-8x22B).  The reference simulator's predicted
tokens/s for the same trace (b200 profile) is printed beside it, read from the
golden fixtures (no oracle import here).

One GPU: GEMM shapes are one GPU's share at --tp, the boundary op is K2.
Under torchrun (WORLD_SIZE > 1) the boundary op is K1 over a multi-process
communicator and every number is the max over ranks.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# before torch: the layer runner binds the CUDA toolkit's cuBLAS (see _lib.py)
import paper_2505_11329_b200  # noqa: E402,F401

NUM_LAYERS = {"llama-70b": 80, "qwen-72b": 80, "mixtral-8x22b": 56}  # proj/src/presets.cpp:72-97
MODES = ("unfused", "fuseonly", "tokenweave", "nocomm")
# measured mode -> the reference BaselineMode it is compared with (Multimem =
# the unfused sequential layer with the best AllReduce, scheduler.cpp:153-164)
PRED_MODE = {"unfused": "multimem", "fuseonly": "fuseonly", "tokenweave": "tokenweave", "nocomm": "nocomm"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, default=8, help="GEMM shapes = one GPU's share at this TP (1 GPU)")
    ap.add_argument("--layers-measured", type=int, default=2)
    ap.add_argument("--boundary-sms", type=int, default=-1,
                    help="fused-op SM budget of weaved batches; -1 = measured per batch size over 16/32/64")
    ap.add_argument("--graph", action="store_true", help="time each batch's layers as one CUDA-graph replay")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--emulate-comm", action="store_true",
                    help="what-if: boundary op = emulation holding --boundary-sms SMs for the paper's 8xB200 "
                         "fused / AllReduce latency (tw_weave_emulate_comm), one GPU only")
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    from paper_2505_11329_b200 import weave
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        cases = json.load(f)["throughput_pred"]
    if args.quick:
        cases = cases[:1]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    dist = dev = comm = None
    rank = 0
    tp = args.tp
    if world > 1:
        import ctypes

        import torch
        import torch.distributed as dist

        from paper_2505_11329_b200 import _lib
        from tools.bench_tp import rendezvous_id
        rank = int(os.environ["RANK"])
        ndev = torch.cuda.device_count()
        local = int(os.environ.get("LOCAL_RANK", rank)) % max(ndev, 1)
        torch.cuda.set_device(local)
        dist.init_process_group("nccl" if ndev >= world else "gloo")
        dev = "cuda" if ndev >= world else None
        tp = world

    res = {"device": f"{world}x B200" if world > 1 else "1x B200", "tp_shapes": tp,
           "boundary_op": "K1 (fused AR+residual+RMSNorm)" if world > 1 else "K2 (fused residual+RMSNorm)",
           "iteration": "measured per-layer device time (CUDA events, warm-up layer excluded) x num_layers",
           "layers_measured": args.layers_measured, "boundary_sms": args.boundary_sms, "cuda_graph": args.graph,
           "emulated_comm": "paper's 8xB200 fused/AllReduce latencies, SMs held (what-if)" if args.emulate_comm
           else None,
           "rows": []}
    for case in cases:
        model = case["model"]
        reqs = [(p, o, 0.0) for p, o in case["requests"]]
        batches = weave.form_batches(reqs, case["chunk_size"])
        max_t = max(b[0] for b in batches)
        kw = {}
        if world > 1:
            H = weave.PRESETS[model]["hidden"]
            h = ctypes.c_void_p()
            _lib.check(_lib.lib.tw_comm_create_mp(world, rank, local, max_t * H * 2, rendezvous_id(dist).encode(),
                                                  _lib.TW_TRANSPORT_AUTO, ctypes.byref(h)))
            comm = h
            kw["comm"] = h
        r = weave.LayerRunner(model, tp=tp, max_tokens=max_t, **kw)
        res["cublas_version"] = r.cublas_version
        if args.emulate_comm:
            with open(os.path.join(ROOT, "profiles", "microbench_b200_measured.json")) as f:
                ser = json.load(f)["series"]
            ar = {p["tokens"]: p["microseconds"] for p in ser["allreduce"]}
            r.emulate_comm([p["tokens"] for p in ser["fused"]], [p["microseconds"] for p in ser["fused"]],
                           [ar[p["tokens"]] for p in ser["fused"]], args.boundary_sms if args.boundary_sms > 0 else 16)
        row = {"name": case["name"], "model": model, "requests": len(reqs),
               "prompt_tokens": sum(p for p, _, _ in reqs), "output_tokens": sum(o for _, o, _ in reqs),
               "chunk_size": case["chunk_size"], "iterations": len(batches),
               "num_layers": NUM_LAYERS[model],
               "overlap_batches": sum(1 for b in batches if b[3] and weave.make_split_plan(
                   b[0], threshold=r.threshold)[3] == 2)}
        for mode in MODES:
            t = r.throughput(reqs, case["chunk_size"], mode, num_layers=NUM_LAYERS[model],
                             layers_measured=args.layers_measured, boundary_sms=args.boundary_sms, graph=args.graph)
            secs = t["total_seconds"]
            if dist is not None:
                from tools.bench_tp import max_over_ranks
                secs = max_over_ranks(secs, dist, dev)
            row[mode] = {"tokens_per_sec": t["total_tokens"] / secs, "total_seconds": secs,
                         "mean_iteration_ms": 1e3 * secs / t["iterations"],
                         "prefill_iteration_ms": [round(1e3 * x, 3) for x, b in zip(t["iteration_latencies"], batches)
                                                  if b[3]][:8]}
            row[mode]["reference_model_tokens_per_sec"] = case[PRED_MODE[mode]]["tokens_per_sec"]
        row["tokenweave_vs_fuseonly"] = row["tokenweave"]["tokens_per_sec"] / row["fuseonly"]["tokens_per_sec"]
        row["tokenweave_vs_unfused"] = row["tokenweave"]["tokens_per_sec"] / row["unfused"]["tokens_per_sec"]
        row["fuseonly_vs_unfused"] = row["fuseonly"]["tokens_per_sec"] / row["unfused"]["tokens_per_sec"]
        r.close()
        if comm is not None:
            _lib.lib.tw_comm_destroy(comm)
            comm = None
        if rank == 0:
            res["rows"].append(row)
            print(json.dumps(row), flush=True)
    if rank == 0 and args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
