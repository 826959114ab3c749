"""K1 over PEER with W co-located ranks at T x 8192 bf16: median µs with an L2
flush between launches (any W, unlike tp_colocated_sweep.py's 2/4/8).

    python tools/k1_w_time.py W [T ...]
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_11329_b200 as tw  # noqa: E402
import torch  # noqa: E402

W = int(sys.argv[1])
Ts = [int(t) for t in sys.argv[2:]] or [1024, 8192]
H = 8192
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
comm = tw.Communicator(W, [0] * W, max(Ts) * H * 2, tw.TW_TRANSPORT_PEER)
for q in range(W):
    comm.buffer(q, tw.TW_BUF_INPUT, (max(Ts), H), torch.bfloat16).normal_()
w = [torch.ones(H, device="cuda")] * W
for T in Ts:
    ranges = tw.token_shard_map(T, W)
    shards = [torch.randn(e - b, H, device="cuda", dtype=torch.bfloat16) for b, e in ranges]
    ts = []
    for i in range(23):
        flush.fill_(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=296 // W)
        e.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(s.elapsed_time(e) * 1e3)
    print(f"W={W} T={T} k1_us={statistics.median(ts):.1f}", flush=True)
comm.check()
