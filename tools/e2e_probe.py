"""e2e host-buffer pipeline: chunk size sweep (T=8192, H=8192 bf16, pinned)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_11329_b200 as tw  # noqa: E402

T, H = 8192, 8192
hx = torch.randn(T, H, dtype=torch.bfloat16).pin_memory()
hr = torch.randn(T, H, dtype=torch.bfloat16).pin_memory()
ho = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
hro = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
hw = torch.ones(H)
s = torch.cuda.Stream()
# raw copy-engine rates for reference
d = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(hx, non_blocking=True)), ("d2h", lambda: ho.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(name, "GB/s", round(5 * T * H * 2 / (a.elapsed_time(b) * 1e-3) / 1e9, 1))
for chunk in (128, 256, 512, 1024, 2048, 4096):
    tw.rmsnorm_residual_host(hx, hr, hw, residual_out=hro, out=ho, chunk_rows=chunk, stream=s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(10):
        tw.rmsnorm_residual_host(hx, hr, hw, residual_out=hro, out=ho, chunk_rows=chunk, stream=s)
    b.record(s)
    torch.cuda.synchronize()
    print("chunk_rows", chunk, "us", round(1e3 * a.elapsed_time(b) / 10, 1))
