"""The default K2 engine choice (no env overrides) over T x H, bf16, write+read
L2 flush, median of 20 -- the numbers DESIGN.md quotes for the shipped policy,
plus per-SM rates under an SM budget."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2505_11329_b200 as tw  # noqa: E402
from bench import L2Flush  # noqa: E402
from tools.sweep import timed  # noqa: E402

flush = L2Flush("cuda:0")
out = {}
for H in (4096, 6144, 8192):
    w = torch.ones(H, device="cuda")
    row = {}
    for T in (256, 1024, 2048, 4096, 8192, 16384):
        x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        o, ro = torch.empty_like(x), torch.empty_like(x)
        us = timed(lambda: tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o), flush, 20)
        row[T] = (round(us, 2), round(4 * T * H * 2 / us / 1e3, 1))
    out[f"H{H}_us_gbs"] = row
    T = 8192
    x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
    r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
    o, ro = torch.empty_like(x), torch.empty_like(x)
    bud = {}
    for b in (8, 16, 32, 64):
        us = timed(lambda: tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o, sm_budget=b), flush, 10)
        bud[b] = (round(us, 1), round(4 * T * H * 2 / us / 1e3 / b, 1))
    out[f"H{H}_T8192_budget_us_gbs_per_sm"] = bud
print(json.dumps(out))
