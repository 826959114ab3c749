"""One K2 launch under an SM budget (the weave's boundary-op regime), for ncu:
`ncu --set full -k regex:k2_tma -s 2 -c 1 python tools/k2_budget_profile.py [budget]`."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_11329_b200 as tw  # noqa: E402

budget = int(sys.argv[1]) if len(sys.argv) > 1 else 16
T, H = 8192, 8192
x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
w = torch.ones(H, device="cuda")
o, ro = torch.empty_like(x), torch.empty_like(x)
for _ in range(3):
    tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o, sm_budget=budget)
torch.cuda.synchronize()
print("ok")
