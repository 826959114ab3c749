"""BASELINE configs[4] on one B200: SM-budget sweep (2..148) x message-size
sweep (S = T*H*2 from 64 KB to 256 MB at H = 8192) for the fused op at TP=1
(K2), next to the unfused baseline on the same box (torch add + rms_norm).
Also the TP=1 token sweep 256..16384 of configs[2].  L2 flushed (write +
read-back of 256 MiB) between timed launches; median of `reps` CUDA-event
timings.  Writes JSON (--out)."""
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
    ap.add_argument("--reps", type=int, default=15)
    args = ap.parse_args()
    import torch
    import paper_2505_11329_b200 as tw
    from bench import L2Flush
    flush = L2Flush("cuda:0")
    H = 8192
    res = {"hidden": H, "dtype": "bf16", "method": "median CUDA-event time, L2 write+read flush", "k2": [],
           "unfused_torch": []}
    tokens = [4, 16, 64, 256, 512, 1024, 2048, 4096, 8192, 16384]
    budgets = [2, 4, 8, 16, 32, 64, 148]
    for T in tokens:
        x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        w = torch.ones(H, device="cuda")
        wb = torch.ones(H, device="cuda", dtype=torch.bfloat16)
        o, ro = torch.empty_like(x), torch.empty_like(x)
        nbytes = 4 * T * H * 2
        row = {"T": T, "message_bytes": T * H * 2}
        for b in budgets:
            us = timed(lambda: tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o, sm_budget=b), flush, args.reps)
            row[f"sms{b}"] = {"us": round(us, 2), "hbm_gbs": round(nbytes / us / 1e3, 1)}
        res["k2"].append(row)
        us = timed(lambda: torch.nn.functional.rms_norm(x + r, (H,), wb, 1e-5), flush, args.reps)
        res["unfused_torch"].append({"T": T, "us": round(us, 2)})
        print(json.dumps(row), "unfused", round(us, 2), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
