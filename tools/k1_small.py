"""K1 at decode sizes (W simulated ranks, PEER, H = 8192 bf16): the fixed
cost of the fused op -- entry/exit rank barriers, ring fill, one launch --
per T.  Median of CUDA-event times over back-to-back launches (no flush: the
working set is L2-resident at these sizes), eager and replayed from a CUDA
graph.  An HBM/L2-bound stand-in for the NVLink case, not an NVLink number.

    python tools/k1_small.py [--transport peer|nvls_sim] [--out FILE]
    TW_FORCE_SYS_SCOPE=1 python tools/k1_small.py ...   # system-scope barriers
                                                         # (what ranks on different GPUs pay)
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_11329_b200 as tw  # noqa: E402  (toolkit cuBLAS/cudart before torch)
import torch  # noqa: E402


def median_us(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return round(statistics.median(ts), 2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--transport", choices=["peer", "nvls_sim"], default="peer")
    args = ap.parse_args()
    H = 8192
    rows = []
    for W in (2, 4, 8):
        Tmax = 256
        tr = tw.TW_TRANSPORT_PEER if args.transport == "peer" else tw.TW_TRANSPORT_NVLS_SIM
        comm = tw.Communicator(W, [0] * W, Tmax * H * 2, tr)
        for q in range(W):
            comm.buffer(q, tw.TW_BUF_INPUT, (Tmax, H), torch.bfloat16).normal_()
        w = [torch.ones(H, device="cuda")] * W
        for T in (W, 16, 64, 256):
            ranges = tw.token_shard_map(T, W)
            shards = [torch.randn(max(e - b, 1), H, device="cuda", dtype=torch.bfloat16) for b, e in ranges]
            budget = max(1, min(148 // W, 16))
            eager = median_us(lambda: comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=budget))
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=budget)
                with torch.cuda.graph(g, stream=s):
                    for _ in range(10):
                        comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=budget)
            torch.cuda.current_stream().wait_stream(s)
            graph10 = median_us(g.replay, reps=50)
            # the same graph of K2 launches over the op's T rows with as many
            # CTAs (W x budget) and no rank barriers: launch + row work, so
            # graph_us_per_op - this = what the cross-rank barriers cost
            x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
            r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
            o, ro = torch.empty_like(x), torch.empty_like(x)
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                tw.rmsnorm_residual(x, r, w[0], residual_out=ro, out=o, sm_budget=W * budget, stream=s)
                with torch.cuda.graph(g2, stream=s):
                    for _ in range(10):
                        tw.rmsnorm_residual(x, r, w[0], residual_out=ro, out=o, sm_budget=W * budget, stream=s)
            torch.cuda.current_stream().wait_stream(s)
            floor10 = median_us(g2.replay, reps=50)
            row = {"tp": W, "T": T, "transport": args.transport,
                   "barrier_scope": "system" if os.environ.get("TW_FORCE_SYS_SCOPE") == "1" else "device",
                   "sm_budget_per_rank": budget, "eager_us": eager,
                   "graph_us_per_op": round(graph10 / 10, 2),
                   "k2_same_rows_graph_us_per_op": round(floor10 / 10, 2),
                   "barrier_overhead_us": round((graph10 - floor10) / 10, 2)}
            print(json.dumps(row), flush=True)
            rows.append(row)
        torch.cuda.synchronize()
        comm.check()
        comm.close()
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"what": __doc__.split("\n\n")[0], "hidden": H, "dtype": "bf16", "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
