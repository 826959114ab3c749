"""TMA/bulk K2 engines with 1 vs 2 CTAs per SM (TW_K2_CTAS_PER_SM)."""
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
    H = int(sys.argv[2])
    res = {}
    for T in (1024, 2048, 4096, 8192):
        x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        w = torch.ones(H, device="cuda")
        o, ro = torch.empty_like(x), torch.empty_like(x)
        res[T] = round(timed(lambda: tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o), flush, 20), 2)
    budgets = {}
    T = 8192
    x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
    r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
    w = torch.ones(H, device="cuda")
    o, ro = torch.empty_like(x), torch.empty_like(x)
    for b in (16, 64):
        budgets[b] = round(timed(lambda: tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o, sm_budget=b), flush, 5), 1)
    print(os.environ.get("TW_K2_ENGINE"), "cps", os.environ.get("TW_K2_CTAS_PER_SM"), "H", H, res, "budget8192", budgets,
          flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
    else:
        for H in ("8192", "6144"):
            for eng in ("tma", "bulk"):
                for cps in ("1", "2"):
                    env = dict(os.environ, TW_K2_ENGINE=eng, TW_K2_CTAS_PER_SM=cps)
                    subprocess.run([sys.executable, __file__, "child", H], env=env, check=True)
