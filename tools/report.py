"""Measured results in the reference's CSV layouts (proj/README.md:60-66):

  microbench : series,unit,<token counts...> rows allreduce, rmsnorm,
               ar_plus_rmsnorm, fused (us) and speedup (x)
  latency    : tokens,default_ms,multimem_ms,nocomm_ms,fuseonly_ms,
               tokenweave_ms,tokenweave_speedup_x,fuseonly_speedup_x

from profiles/sweep_rNN.json (TP=1 op sweep) and profiles/weave_rNN.json
(`python tools/report.py r02`)
(measured layers).  At TP=1 there is no AllReduce (0 us); `rmsnorm` is the
unfused baseline on the same box (torch add + rms_norm) and `fused` is K2 on
the whole GPU.  In `latency`, `multimem` is our unfused sequential layer
(the reference's Multimem chain) and `default` is not measured (nan).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def microbench(sweep):
    toks = [r["T"] for r in sweep["k2"]]
    fused = [r["sms148"]["us"] for r in sweep["k2"]]
    unf = {u["T"]: u["us"] for u in sweep["unfused_torch"]}
    rms = [unf[t] for t in toks]
    rows = [["series", "unit"] + [str(t) for t in toks],
            ["allreduce", "us"] + ["0"] * len(toks),
            ["rmsnorm", "us"] + [f"{v:.2f}" for v in rms],
            ["ar_plus_rmsnorm", "us"] + [f"{v:.2f}" for v in rms],
            ["fused", "us"] + [f"{v:.2f}" for v in fused],
            ["speedup", "x"] + [f"{a / b:.3f}" for a, b in zip(rms, fused)]]
    return "\n".join(",".join(r) for r in rows) + "\n"


def latency(weave, model, tp):
    out = ["tokens,default_ms,multimem_ms,nocomm_ms,fuseonly_ms,tokenweave_ms,tokenweave_speedup_x,fuseonly_speedup_x"]
    for r in weave["rows"]:
        if r["model"] != model or r["tp_shapes"] != tp:
            continue
        mm, fo, tw = r["unfused_us"], r["fuseonly_us"], r["weave_best_us"]
        out.append(f"{r['T']},nan,{mm / 1e3:.4f},{r['nocomm_us'] / 1e3:.4f},{fo / 1e3:.4f},{tw / 1e3:.4f},"
                   f"{mm / tw:.3f},{mm / fo:.3f}")
    return "\n".join(out) + "\n"


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"  # which round's sweep_/weave_ JSONs to render
    prof = os.path.join(ROOT, "profiles")
    sweep = json.load(open(os.path.join(prof, f"sweep_{rnd}.json")))
    weave = json.load(open(os.path.join(prof, f"weave_{rnd}.json")))
    with open(os.path.join(prof, f"microbench_tp1_{rnd}.csv"), "w") as f:
        f.write(microbench(sweep))
    for model, tp in (("llama-70b", 8), ("llama-70b", 1), ("mixtral-8x22b", 8)):
        with open(os.path.join(prof, f"latency_{model}_tp{tp}shapes_{rnd}.csv"), "w") as f:
            f.write(latency(weave, model, tp))
    print(open(os.path.join(prof, f"microbench_tp1_{rnd}.csv")).read())
    return 0


if __name__ == "__main__":
    sys.exit(main())
