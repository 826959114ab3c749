"""Small K1/K2/K3 launches for compute-sanitizer (memcheck / racecheck /
synccheck): every engine, both dtypes, colocated ranks (W 2/4/8), gather residual."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_11329_b200 as tw  # noqa: E402

for H in (8192, 6144, 4096, 33):
    for dt in (torch.bfloat16, torch.float32):
        x = torch.randn(37, H, device="cuda", dtype=dt)
        r = torch.randn(37, H, device="cuda", dtype=dt)
        w = torch.rand(H, device="cuda") + 0.5
        tw.rmsnorm_residual(x, r, w)
        tw.rmsnorm_residual(x, r, w, residual_out=r)
        # two CTAs: each walks ~18 rows, wrapping the smem ring (both row groups)
        tw.rmsnorm_residual(x, r, w, sm_budget=2)
# K1 PEER bulk-copy engine: one stage per row (W 2/4), two stages per row with
# a lazily released (H 1024) and an immediately released (H 8192) ring
for W, H in ((2, 1024), (4, 1024), (8, 1024), (8, 8192), (2, 8192)):
    T = 29
    comm = tw.Communicator(W, [0] * W, T * H * 4, tw.TW_TRANSPORT_PEER)
    for dt in (torch.bfloat16, torch.float32):
        for q in range(W):
            comm.buffer(q, 0, (T, H), dt).normal_()
        ranges = tw.token_shard_map(T, W)
        shards = [torch.randn(e - b, H, device="cuda", dtype=dt) for b, e in ranges]
        comm.fused_allreduce_rmsnorm(T, H, shards, [torch.ones(H, device="cuda")] * W, sm_budget=2,
                                     gather_residual=True, dtype=dt)
        comm.allreduce(T, H, dt, sm_budget=2)
    torch.cuda.synchronize()
    comm.check()
    comm.close()
# K1 over NVLS (the north_star kernel) on simulated ranks: every pipeline
# depth, G = 1/2, both dtypes, an uneven shard map
for W, H, T in ((2, 8192, 29), (4, 1024, 13), (8, 8192, 21)):
    comm = tw.Communicator(W, [0] * W, T * H * 4, tw.TW_TRANSPORT_NVLS_SIM)
    for dt in (torch.bfloat16, torch.float32):
        for q in range(W):
            comm.buffer(q, 0, (T, H), dt).normal_()
        ranges = tw.token_shard_map(T, W)
        shards = [torch.randn(max(e - b, 1), H, device="cuda", dtype=dt) for b, e in ranges]
        for depth in (1, 2, 3):
            comm.fused_allreduce_rmsnorm(T, H, shards, [torch.ones(H, device="cuda")] * W, sm_budget=3,
                                         gather_residual=depth == 2, dtype=dt, nvls_depth=depth)
        comm.allreduce(T, H, dt, sm_budget=2)
    torch.cuda.synchronize()
    comm.check()
    comm.close()
print("sanitize workload done")
