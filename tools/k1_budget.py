"""K1 co-located (PEER) timing vs per-rank CTA budget: T=8192, H=8192 bf16."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_11329_b200 as tw  # noqa: E402
from bench import L2Flush  # noqa: E402
from tools.sweep import timed  # noqa: E402

flush = L2Flush("cuda:0")
T, H = 8192, 8192
for W in (2, 8):
    comm = tw.Communicator(W, [0] * W, T * H * 2, tw.TW_TRANSPORT_PEER)
    for q in range(W):
        comm.buffer(q, tw.TW_BUF_INPUT, (T, H), torch.bfloat16).normal_()
    ranges = tw.token_shard_map(T, W)
    shards = [torch.randn(e - b, H, device="cuda", dtype=torch.bfloat16) for b, e in ranges]
    w = [torch.ones(H, device="cuda")] * W
    res = {}
    for b in (8, 16, 148 // W, 296 // W):
        us = timed(lambda: comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=b), flush, 10)
        nbytes = W * (T * H * 2) * 2 + 2 * T * H * 2  # all ranks: read N*S/N each of N inputs, write N copies, residual
        res[b] = (round(us, 1), round(nbytes / us / 1e3, 1))
    comm.check()
    comm.close()
    print(f"W={W} budget -> (us, GB/s)", res, flush=True)
