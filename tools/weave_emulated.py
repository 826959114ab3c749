"""What-if (NOT the product, NOT a multi-GPU measurement): the weave against
real B200 cuBLAS GEMMs with the TP = 8 boundary op EMULATED -- an op that holds
16 SMs for the latency the paper measured on 8x B200 for the fused AR+RMSNorm
kernel or the multimem AllReduce at that
token count.  One GPU cannot run the NVLink-bound op itself; this asks whether
the two-stream schedule hides an op of that duration and SM footprint behind
real GEMMs, next to the reference simulator's prediction for the same layer.

Modes: unfused = emulated AllReduce + the real residual add and RMSNorm
kernels; fuse-only = emulated fused op; TokenWeave = emulated fused op on each
split (analytic, equal and measured Alg-1 splits); no-comm = GEMMs only.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# before torch: the layer runner binds the CUDA toolkit's cuBLAS (see _lib.py)
import paper_2505_11329_b200  # noqa: E402,F401


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=6)
    ap.add_argument("--sms", type=int, default=16, help="SMs the emulated op holds (paper: ~8-16 on B200)")
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    from paper_2505_11329_b200 import weave
    with open(os.path.join(ROOT, "profiles", "microbench_b200_measured.json")) as f:
        series = json.load(f)["series"]
    toks = [p["tokens"] for p in series["fused"]]
    fused = [p["microseconds"] for p in series["fused"]]
    ar = {p["tokens"]: p["microseconds"] for p in series["allreduce"]}
    ar = [ar[t] for t in toks]
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        pred = {(r["model"], r["T"]): r for r in json.load(f)["layer_latency_s"]}
    res = {"what": "weave with an EMULATED TP=8 boundary op (published 8xB200 latencies, "
                   f"{args.sms} SMs held) against real cuBLAS GEMMs at TP=8 per-GPU shapes, 1x B200",
           "sms_held": args.sms, "layers_timed": args.layers, "cuda_graph": args.graph, "rows": []}
    # Llama / Mixtral layer shapes, and the Qwen2.5-72B token sweep of BASELINE configs[2]
    for model, tokens in (("llama-70b", [1024, 2048, 4096, 8192]), ("mixtral-8x22b", [4096, 8192]),
                          ("qwen-72b", [256, 512, 1024, 2048, 4096, 8192, 16384])):
        r = weave.LayerRunner(model, tp=8, max_tokens=max(tokens))
        res["cublas_version"] = r.cublas_version
        r.emulate_comm(toks, fused, ar, args.sms)
        for T in tokens:
            a, b, off, mode = weave.make_split_plan(T, threshold=r.threshold)
            run = lambda m, **kw: r.run(T, m, layers=args.layers, graph=args.graph, **kw)  # noqa: E731
            row = {"model": model, "T": T, "unfused_us": run("unfused"), "fuseonly_us": run("fuseonly"),
                   "nocomm_us": run("nocomm"), "plan": {"prefix": a, "suffix": b, "mode": weave.SPLIT_MODES[mode]}}
            cands = {"equal": T // 2}
            if mode == 2 and a != T // 2:
                cands["analytic"] = a
            for name, pa in cands.items():
                row[f"weave_{name}_us"] = run("tokenweave", prefix=pa, boundary_sms=args.sms)
            times = {}

            def fwd(pa, pb):
                times[pa] = run("tokenweave", prefix=pa, boundary_sms=args.sms)
                return times[pa]

            o = weave.smart_offset_sweep(T, fwd)
            row["weave_alg1_us"] = times[T // 2 + o]
            row["alg1_offset"] = o
            best = min(v for k, v in row.items() if k.startswith("weave_") and k.endswith("_us"))
            row["weave_best_us"] = best
            row["weave_vs_unfused"] = row["unfused_us"] / best
            row["weave_vs_fuseonly"] = row["fuseonly_us"] / best
            row["fuseonly_vs_unfused"] = row["unfused_us"] / row["fuseonly_us"]
            if (model, T) in pred:
                p = pred[(model, T)]
                row["reference_model_us"] = {m: round(1e6 * p[m], 1) for m in ("multimem", "fuseonly", "tokenweave",
                                                                                 "nocomm")}
            res["rows"].append(row)
            print(json.dumps(row), flush=True)
        r.close()
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
