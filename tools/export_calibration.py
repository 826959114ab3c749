"""Measured microbenchmarks in the reference's CalibrationTable JSON schema
(proj/data/microbench_b200.json; parsed by CalibrationTable::from_json_file,
proj/src/calibration.cpp:15-38), so the reference's own calibrate /
microbench / latency commands can run on B200-measured numbers.

Series written (hidden 8192, bf16, the paper's token list 32..65536):
  rmsnorm          MEASURED: K2 over the full T on one B200 (the paper's
                   "RMSNorm" row is likewise unsharded over T on one GPU,
                   PAPER.md:610-611), write+read L2 flush, median of 20.
  rmsnorm_unfused  MEASURED: torch add + rms_norm on the same box (context).
  allreduce, fused PUBLISHED: a one-GPU box cannot
                   measure NVLink collectives; copied so calibrate() has the
                   series it requires.  The "provenance" key says which is which
                   (ignored by the reference parser).

  python tools/export_calibration.py --out profiles/microbench_b200_measured.json
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TOKENS = [32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536]
PAPER_AR = [26.08, 28.80, 32.29, 35.20, 45.55, 60.26, 95.86, 166.61, 305.78, 578.48, 1131.55, 2240.93]
PAPER_FUSED = [30.46, 32.45, 34.14, 39.18, 49.31, 63.62, 100.48, 170.14, 307.71, 581.55, 1130.69, 2236.02]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "microbench_b200_measured.json"))
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    import paper_2505_11329_b200 as tw
    from bench import L2Flush
    flush = L2Flush("cuda:0")
    H = 8192
    k2, unf = [], []
    for T in TOKENS:
        x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        w = torch.ones(H, device="cuda")
        wb = torch.ones(H, device="cuda", dtype=torch.bfloat16)
        o, ro = torch.empty_like(x), torch.empty_like(x)
        for name, fn, sink in (("k2", lambda: tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o), k2),
                               ("unf", lambda: torch.nn.functional.rms_norm(x + r, (H,), wb, 1e-5), unf)):
            for _ in range(3):
                fn()
            ts = []
            for i in range(args.reps):
                flush(i)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                fn()
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e))
            sink.append(round(1e3 * statistics.median(ts), 2))
        del x, r, o, ro
        print(T, k2[-1], unf[-1], flush=True)

    def series(vals):
        return [{"tokens": t, "microseconds": v} for t, v in zip(TOKENS, vals)]

    table = {
        "hidden": H, "bytes_per_element": 2,
        "provenance": {"rmsnorm": "measured: K2 fused residual+RMSNorm, 1x B200, bench methodology",
                       "rmsnorm_unfused": "measured: torch add + rms_norm, same box",
                       "allreduce": "published, PAPER.md:606-607 (not measurable on a 1-GPU box)",
                       "fused": "published, PAPER.md:622-623 (not measurable on a 1-GPU box)"},
        "series": {"allreduce": series(PAPER_AR), "rmsnorm": series(k2), "rmsnorm_unfused": series(unf),
                   "fused": series(PAPER_FUSED)},
    }
    with open(args.out, "w") as f:
        json.dump(table, f, indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
