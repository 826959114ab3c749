"""Host-side cost of one C-ABI call (ctypes included): wall time per call of
the fused ops at decode sizes over 2000 back-to-back calls, the GPU kept
ahead (launches are asynchronous; the queue never fills at these sizes)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_11329_b200 as tw  # noqa: E402
import torch  # noqa: E402


def per_call_us(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return round((t1 - t0) / n * 1e6, 2)


H = 8192
out = {}
x = torch.randn(8, H, device="cuda", dtype=torch.bfloat16)
r = torch.randn(8, H, device="cuda", dtype=torch.bfloat16)
w = torch.ones(H, device="cuda")
o, ro = torch.empty_like(x), torch.empty_like(x)
out["k2_T8"] = per_call_us(lambda: tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o))
# the bare C-ABI call through ctypes (arguments prepared once)
from paper_2505_11329_b200 import _lib  # noqa: E402
args = (x.data_ptr(), r.data_ptr(), ro.data_ptr(), o.data_ptr(), w.data_ptr(), 8, H, 1e-5, tw.TW_BF16, 0,
        torch.cuda.current_stream().cuda_stream)
fn = _lib.lib.tw_rmsnorm_residual
out["k2_T8_bare_ctypes"] = per_call_us(lambda: fn(*args))
out["torch_current_stream"] = per_call_us(lambda: torch.cuda.current_stream().cuda_stream)
for W in (2, 8):
    comm = tw.Communicator(W, [0] * W, 64 * H * 2, tw.TW_TRANSPORT_PEER)
    ranges = tw.token_shard_map(W, W)
    shards = [torch.randn(1, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    ws = [w] * W
    out[f"k1_tp{W}_T{W}"] = per_call_us(lambda: comm.fused_allreduce_rmsnorm(W, H, shards, ws, sm_budget=16), 500)
    torch.cuda.synchronize()
    comm.close()
print(json.dumps(out))
if len(sys.argv) > 2 and sys.argv[1] == "--out":
    with open(sys.argv[2], "w") as f:
        json.dump({"what": "host wall time per call, us (tools/host_overhead.py)", **out}, f, indent=1)
