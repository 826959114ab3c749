"""K2 on fp32 activations (the drop-in's TokenMatrix dtype), default policy,
T x H = {1024..8192} x 8192, L2 flushed; us and GB/s of algorithmic bytes."""
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
for H in (4096, 8192):
    w = torch.ones(H, device="cuda")
    row = {}
    for T in (1024, 2048, 4096, 8192):
        x = torch.randn(T, H, device="cuda")
        r = torch.randn(T, H, device="cuda")
        o, ro = torch.empty_like(x), torch.empty_like(x)
        us = timed(lambda: tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o), flush, 15)
        row[T] = (round(us, 2), round(4 * T * H * 4 / us / 1e3, 1))
    out[f"fp32_H{H}"] = row
print(json.dumps(out))
