"""Measured weave vs sequential layer latency on one B200 (tw_weave.h runner).

For each model/T: fuse-only (sequential), no-comm (lower bound), and the
weave with (a) the analytic split of make_split_plan, (b) the equal split,
(c) the measured Alg-1 sweep (smart_offset_sweep driven by real layer
times).  GEMM shapes are one GPU's share at TP=8; the boundary op is K2.
Prints one JSON object; --out writes it too.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=6)
    ap.add_argument("--out", default="")
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    from paper_2505_11329_b200 import weave
    import oracle
    ref = None
    try:
        ref = oracle.RefLib()
    except Exception:
        pass
    cases = [("llama-70b", [1024, 2048, 4096, 8192]), ("mixtral-8x22b", [4096, 8192])]
    if args.quick:
        cases = [("llama-70b", [2048, 8192])]
    res = {"gemm_shapes": "per GPU at TP=8", "boundary_op": "K2 (tw_rmsnorm_residual) on the split rows",
           "layers_timed": args.layers, "rows": []}
    for model, tokens in cases:
        r = weave.LayerRunner(model, tp=8, max_tokens=max(tokens))
        for T in tokens:
            row = {"model": model, "T": T}
            row["fuseonly_us"] = r.run(T, "fuseonly", layers=args.layers)
            row["nocomm_us"] = r.run(T, "nocomm", layers=args.layers)
            a, b, off, mode = weave.make_split_plan(T, threshold=r.threshold)
            row["plan"] = {"prefix": a, "suffix": b, "offset": off, "mode": weave.SPLIT_MODES[mode]}
            best = None
            for sms in (8, 16, 32):
                if mode == 2:
                    us = r.run(T, "tokenweave", prefix=a, boundary_sms=sms, layers=args.layers)
                    row[f"weave_analytic_sms{sms}_us"] = us
                    best = us if best is None else min(best, us)
                eq = r.run(T, "tokenweave", prefix=T // 2, boundary_sms=sms, layers=args.layers)
                row[f"weave_equal_sms{sms}_us"] = eq
                best = eq if best is None else min(best, eq)
            # Alg. 1: measured sweep over the offset grid (boundary 16 SMs)
            times = {}

            def fwd(pa, pb):
                times[pa] = r.run(T, "tokenweave", prefix=pa, boundary_sms=16, layers=args.layers)
                return times[pa]

            off_sweep = weave.smart_offset_sweep(T, fwd)
            row["alg1_offset"] = off_sweep
            row["alg1_us"] = times[T // 2 + off_sweep]
            row["weave_best_us"] = min(best, row["alg1_us"])
            row["speedup_vs_fuseonly"] = row["fuseonly_us"] / row["weave_best_us"]
            r.run(T, "tokenweave", prefix=T // 2 + off_sweep, boundary_sms=16, layers=args.layers)
            row["timeline"] = r.trace()
            if ref is not None:
                row["reference_model_us"] = {m: 1e6 * ref.layer_latency("b200", model, T, m)
                                             for m in ("fuseonly", "tokenweave", "nocomm", "multimem")}
            res["rows"].append(row)
            print(json.dumps({k: v for k, v in row.items() if k != "timeline"}), flush=True)
        r.close()
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
