"""Weave timing stability check (imports torch FIRST, so the runner binds
torch's bundled cuBLAS 12.8 unless the package was loaded earlier -- compare
tools/weave_repeat_notorch.py, which binds the toolkit's 12.9), optionally after other work in the same
process (argv[1]: 'k1' = co-located K1 first, 'k2' = big K2 first, 'tp1' = a
TP=1-shape runner created, run and freed first, 'allocN' = N GB allocated and
freed first)."""
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
if pre == "tp1":  # weave_bench's order: a TP=1-shape runner first, then freed
    r1 = weave.LayerRunner("llama-70b", tp=1, max_tokens=T)
    r1.run(T, "fuseonly", layers=2)
    r1.close()
if pre.startswith("alloc"):  # only allocate and free device memory first (GB in the suffix)
    blob = torch.empty(int(pre[5:]) << 30, dtype=torch.uint8, device="cuda")
    del blob
    torch.cuda.empty_cache()
r = weave.LayerRunner("llama-70b", tp=8, max_tokens=T)
if pre == "part":  # one weaved run with a cuBLAS SM-count target first
    r.run(T, "tokenweave", prefix=4096, boundary_sms=64, gemm_sms=84, layers=2)
if pre == "small":  # weave_bench's order: smaller batches on the same runner first
    for t in (1024, 2048, 4096):
        for m in ("unfused", "fuseonly", "nocomm"):
            r.run(t, m, layers=2)
        r.run(t, "tokenweave", prefix=t // 2, boundary_sms=64, layers=2)
for rep in range(2):
    print(pre, rep, {m: round(r.run(T, m, layers=6), 1) for m in ("unfused", "fuseonly", "nocomm")},
          {b: round(r.run(T, "tokenweave", prefix=4096, boundary_sms=b, layers=6), 1) for b in (16, 32, 64)},
          flush=True)
