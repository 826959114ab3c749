"""Per-SM efficiency of the K2 engines under a small SM budget (the weave's
boundary-op regime): T=8192, H=8192 bf16, budgets 8..148."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child():
    import torch
    import paper_2505_11329_b200 as tw
    from bench import L2Flush
    from tools.sweep import timed
    flush = L2Flush("cuda:0")
    T, H = 8192, 8192
    x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
    r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
    w = torch.ones(H, device="cuda")
    o, ro = torch.empty_like(x), torch.empty_like(x)
    out = {}
    for b in (8, 16, 32, 64, 148):
        us = timed(lambda: tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o, sm_budget=b), flush, 10)
        out[b] = (round(us, 1), round(4 * T * H * 2 / us / 1e3 / b, 1))
    print(os.environ.get("TW_K2_ENGINE"), "budget -> (us, GB/s per SM)", out, flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        child()
    else:
        for eng in ("tma", "bulk", "rows", "flat"):
            subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, TW_K2_ENGINE=eng), check=True)
