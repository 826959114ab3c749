"""K1 launches (W simulated ranks, PEER, T x H=8192 bf16, whole GPU) for ncu:
`ncu --set full -k regex:rownorm_kernel -c 1 python tools/k1_profile.py [W] [T]`
(W <= 4 runs the bulk-copy engine: `-k regex:k1_peer_tma`)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_11329_b200 as tw  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8   # W <= 4: the PEER bulk-copy engine
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
H = 8192
comm = tw.Communicator(W, [0] * W, T * H * 2, tw.TW_TRANSPORT_PEER)
for q in range(W):
    comm.buffer(q, tw.TW_BUF_INPUT, (T, H), torch.bfloat16).normal_()
ranges = tw.token_shard_map(T, W)
shards = [torch.randn(e - b, H, device="cuda", dtype=torch.bfloat16) for b, e in ranges]
w = [torch.ones(H, device="cuda")] * W
for _ in range(int(os.environ.get("REPS", "3"))):
    comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=296 // W)
torch.cuda.synchronize()
comm.check()
print("k1 profile workload done")
