"""Decode-size K2 (T = 1..1024, H = 8192 bf16) per engine (TW_K2_ENGINE):
timed inside a CUDA graph of 50 back-to-back launches (no host launch cost,
inputs L2-resident: the decode regime) and cold (L2 flushed, one launch per
CUDA-event pair, launch cost included)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(tag):
    import torch
    import paper_2505_11329_b200 as tw
    H = 8192
    w = torch.ones(H, device="cuda")
    from bench import L2Flush
    from tools.sweep import timed
    flush = L2Flush("cuda:0")
    out = {"engine": tag, "graph_hot_us": {}, "cold_us": {}}
    for T in (1, 8, 32, 64, 128, 256, 512, 1024):
        x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        o, ro = torch.empty_like(x), torch.empty_like(x)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(50):
                tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) * 1e3 / 50)
        out["graph_hot_us"][T] = round(best, 2)
        out["cold_us"][T] = round(timed(lambda: tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o), flush, 20), 2)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        child(sys.argv[1])
    else:
        for eng, g in (("default", None), ("tma", "1"), ("tma", "2"), ("rows", None), ("flat", None)):
            env = dict(os.environ)
            if eng != "default":
                env["TW_K2_ENGINE"] = eng
            if g:
                env["TW_K2_GROUPS"] = g
            subprocess.run([sys.executable, __file__, f"{eng}-g{g or 'auto'}"], env=env, check=True)
