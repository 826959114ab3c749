"""K1 launches (W simulated ranks on one GPU, T x H=8192 bf16) for ncu:

    ncu --set full -k regex:k1_ -s 2 -c 1 python tools/k1_profile.py [W] [T] [peer|nvls_sim]

peer: the PEER bulk-copy engine (k1_peer_tma_kernel), the whole GPU split
between the ranks.  nvls_sim: the NVLS kernel (k1_nvls_kernel<..., MmSim>)
at the north_star budget (SM_BUDGET, default 8 CTAs per rank)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_11329_b200 as tw  # noqa: E402  (loads before torch)
import torch  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
mode = sys.argv[3] if len(sys.argv) > 3 else "peer"
H = 8192
tr = tw.TW_TRANSPORT_PEER if mode == "peer" else tw.TW_TRANSPORT_NVLS_SIM
budget = int(os.environ.get("SM_BUDGET", 296 // W if mode == "peer" else 8))
comm = tw.Communicator(W, [0] * W, T * H * 2, tr)
for q in range(W):
    comm.buffer(q, tw.TW_BUF_INPUT, (T, H), torch.bfloat16).normal_()
ranges = tw.token_shard_map(T, W)
shards = [torch.randn(e - b, H, device="cuda", dtype=torch.bfloat16) for b, e in ranges]
w = [torch.ones(H, device="cuda")] * W
for _ in range(int(os.environ.get("REPS", "3"))):
    comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=budget)
torch.cuda.synchronize()
comm.check()
print("k1 profile workload done")
