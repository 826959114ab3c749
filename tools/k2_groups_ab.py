"""K2 TMA engine: one vs two consumer row groups per CTA (TW_K2_GROUPS), under
an SM budget (the weave's boundary-op regime; one CTA per SM) and over the
whole GPU (vs two CTAs per SM).  T x H bf16, write+read L2 flush, median."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(tag):
    import torch
    import paper_2505_11329_b200 as tw
    from bench import L2Flush
    from tools.sweep import timed
    flush = L2Flush("cuda:0")
    out = {"config": tag}
    for H in (8192, 6144):
        w = torch.ones(H, device="cuda")
        T = 8192
        x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        o, ro = torch.empty_like(x), torch.empty_like(x)
        bud = {}
        for b in (8, 16, 32, 64, 148):
            us = timed(lambda: tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o, sm_budget=b), flush, 10)
            bud[b] = (round(us, 1), round(4 * T * H * 2 / us / 1e3 / b, 1))
        out[f"H{H}_budget_us_gbs_per_sm"] = bud
        full = {}
        for T2 in (1024, 2048, 4096, 8192, 16384):
            x2 = torch.randn(T2, H, device="cuda", dtype=torch.bfloat16)
            r2 = torch.randn(T2, H, device="cuda", dtype=torch.bfloat16)
            o2, ro2 = torch.empty_like(x2), torch.empty_like(x2)
            full[T2] = round(timed(lambda: tw.rmsnorm_residual(x2, r2, w, residual_out=ro2, out=o2), flush, 20), 2)
        out[f"H{H}_full_gpu_us"] = full
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--groups":  # TMA engine, 1 / 2 row groups
        for g in ("1", "2"):
            env = dict(os.environ, TW_K2_ENGINE="tma", TW_K2_CTAS_PER_SM="1", TW_K2_GROUPS=g)
            subprocess.run([sys.executable, __file__, f"tma-cps1-g{g}"], env=env, check=True)
    elif len(sys.argv) > 1:
        child(sys.argv[1])
    else:
        for eng, cps, g in (("tma", "1", "1"), ("tma", "2", "1"), ("tma", "1", "2"), ("bulk", "1", "1"),
                            ("flat", "1", "1"), ("rows", "1", "1")):
            env = dict(os.environ, TW_K2_ENGINE=eng, TW_K2_CTAS_PER_SM=cps, TW_K2_GROUPS=g)
            subprocess.run([sys.executable, __file__, f"{eng}-cps{cps}-g{g}"], env=env, check=True)
