"""Weave timing stability check, optionally after other work in the same
process (argv[1]: 'k1' = co-located K1 first, 'k2' = big K2 first)."""
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_2505_11329_b200 as tw  # noqa: E402
from paper_2505_11329_b200 import weave  # noqa: E402

T = 8192
pre = sys.argv[1] if len(sys.argv) > 1 else ""
if pre == "k1":
    H = 8192
    comm = tw.Communicator(8, [0] * 8, T * H * 2, tw.TW_TRANSPORT_PEER)
    ranges = tw.token_shard_map(T, 8)
    shards = [torch.randn(e - b, H, device="cuda", dtype=torch.bfloat16) for b, e in ranges]
    for _ in range(5):
        comm.fused_allreduce_rmsnorm(T, H, shards, [torch.ones(H, device="cuda")] * 8, sm_budget=37)
    torch.cuda.synchronize()
    comm.close()
if pre == "k2":
    x = torch.randn(T, 8192, device="cuda", dtype=torch.bfloat16)
    for _ in range(5):
        tw.rmsnorm_residual(x, x.clone(), torch.ones(8192, device="cuda"))
    torch.cuda.synchronize()
r = weave.LayerRunner("llama-70b", tp=8, max_tokens=T)
for rep in range(2):
    print(pre, rep, {m: round(r.run(T, m, layers=6), 1) for m in ("unfused", "fuseonly", "nocomm")},
          {b: round(r.run(T, "tokenweave", prefix=4096, boundary_sms=b, layers=6), 1) for b in (16, 32, 64)},
          flush=True)
