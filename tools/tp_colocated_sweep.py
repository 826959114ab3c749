"""TP = 2/4/8 on ONE GPU: N simulated ranks (PEER transport, one grid) -- the
fused op K1 next to the unfused baseline of the same ranks (K3 one-shot
AllReduce, then K2 over the full T on every rank, SURVEY §8d baseline (ii)),
H = 8192 bf16, T = 1024..8192 (BASELINE configs[1]/[2] shapes).  Everything
is HBM-bound here (all ranks share one GPU's HBM): a correctness-scale,
same-box comparison of the fused and unfused DATA MOVEMENT, NOT an NVLink
measurement.  Per point: median of CUDA-event times with an L2 flush between
launches, and the algorithmic HBM bytes of each variant.

    python tools/tp_colocated_sweep.py --out profiles/tp_colocated_r01.json
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, flush, reps):
    import torch
    for _ in range(3):
        fn()
    ts = []
    for i in range(reps):
        flush(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return 1e3 * statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch
    import paper_2505_11329_b200 as tw
    from bench import L2Flush
    flush = L2Flush("cuda:0")
    H = 8192
    res = {"what": "N simulated ranks on one B200 (PEER transport): fused K1 vs unfused K3 + K2, HBM-bound stand-in",
           "hidden": H, "dtype": "bf16", "rows": []}
    for N in (2, 4, 8):
        for T in (1024, 2048, 4096, 8192):
            S = T * H * 2
            comm = tw.Communicator(N, [0] * N, S, tw.TW_TRANSPORT_PEER)
            for q in range(N):
                comm.buffer(q, tw.TW_BUF_INPUT, (T, H), torch.bfloat16).normal_()
            ranges = tw.token_shard_map(T, N)
            shards = [torch.randn(e - b, H, device="cuda", dtype=torch.bfloat16) for b, e in ranges]
            w = [torch.ones(H, device="cuda")] * N
            budget = 296 // N  # every rank's CTAs co-resident (the grid holds all ranks)
            k1 = timed(lambda: comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=budget), flush, args.reps)
            # unfused: K3 AllReduce into every rank's OUTPUT, then K2 over all T rows on every rank
            res_full = [torch.randn(T, H, device="cuda", dtype=torch.bfloat16) for _ in range(N)]
            outs = [comm.buffer(q, tw.TW_BUF_OUTPUT, (T, H), torch.bfloat16) for q in range(N)]
            normed = [torch.empty(T, H, device="cuda", dtype=torch.bfloat16) for _ in range(N)]

            def unfused():
                comm.allreduce(T, H, torch.bfloat16, sm_budget=budget)
                for q in range(N):
                    tw.rmsnorm_residual(outs[q], res_full[q], w[q], residual_out=res_full[q], out=normed[q])

            un = timed(unfused, flush, args.reps)
            comm.check()
            comm.close()
            # algorithmic HBM bytes on the shared GPU: K1 reads N partial rows per
            # owned row (N*S over all ranks), reads+writes the residual shards
            # (2*S), writes the output to every rank (N*S); K3 reads N*S and
            # writes N*S, then K2 on every rank moves 4*S.
            b_k1 = (2 * N + 2) * S
            b_un = 2 * N * S + 4 * N * S
            row = {"tp": N, "T": T, "k1_us": round(k1, 1), "unfused_k3_k2_us": round(un, 1),
                   "fused_speedup": round(un / k1, 3), "k1_hbm_gbs": round(b_k1 / k1 / 1e3, 1),
                   "unfused_hbm_gbs": round(b_un / un / 1e3, 1), "k1_alg_bytes": b_k1, "unfused_alg_bytes": b_un,
                   "ctas_per_rank": budget}
            res["rows"].append(row)
            print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
