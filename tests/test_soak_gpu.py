"""Soak: many back-to-back K1 / K3 launches on one communicator with random
shapes, SM budgets, token offsets, G and dtypes (the barrier generations,
per-CTA counters and row windows must stay consistent across thousands of
launches), checked against a torch fp32 restatement on every launch."""
import random

import pytest

pytestmark = pytest.mark.gpu


def test_k1_k3_soak_random_launches(cuda):
    import torch
    import paper_2505_11329_b200 as tw
    rng = random.Random(1234)
    W, Tmax, Hmax = 4, 96, 2048
    comm = tw.Communicator(W, [0] * W, Tmax * Hmax * 4, tw.TW_TRANSPORT_PEER)
    checked = 0
    for it in range(600):
        dt = rng.choice([torch.bfloat16, torch.float32])
        H = rng.choice([8, 24, 64, 1000, 1024, 2048])
        T = rng.randint(1, Tmax // 2)
        off = rng.randint(0, Tmax - T)
        budget = rng.choice([1, 2, 3, 8, 17, 37])
        op = rng.random()
        parts = [torch.randn(off + T, H, device="cuda").to(dt) for _ in range(W)]
        for q in range(W):
            comm.buffer(q, 0, (off + T, H), dt).copy_(parts[q])
        want_sum = sum(p[off:].float() for p in parts)
        if op < 0.2:  # K3 AllReduce baseline on the row window
            comm.allreduce(T, H, dt, sm_budget=budget, token_offset=off)
            torch.cuda.synchronize()
            got = comm.buffer(rng.randrange(W), 1, (off + T, H), dt)[off:].float()
            tol = 0 if dt == torch.float32 else 2e-2
            assert torch.allclose(got, want_sum, rtol=tol, atol=tol * want_sum.abs().max().item() + 1e-6)
        else:
            gather = rng.random() < 0.3
            ranges = tw.token_shard_map(T, W)
            res_full = torch.randn(T, H, device="cuda").to(dt)
            shards = [res_full[b:e].clone() for b, e in ranges]
            w = torch.rand(H, device="cuda") + 0.5
            comm.fused_allreduce_rmsnorm(T, H, shards, [w] * W, sm_budget=budget, gather_residual=gather,
                                         token_offset=off, dtype=dt)
            torch.cuda.synchronize()
            rp = (want_sum + res_full.float()).to(dt).float()
            assert torch.equal(torch.cat(shards).float(), rp) or dt == torch.bfloat16 and torch.allclose(
                torch.cat(shards).float(), rp, rtol=1e-2, atol=1e-2)
            want = rp * torch.rsqrt((rp * rp).mean(1, keepdim=True) + 1e-5) * w
            got = comm.buffer(rng.randrange(W), 1, (off + T, H), dt)[off:].float()
            rel = ((got - want).abs() / torch.maximum(want.abs(), want.pow(2).mean(1, keepdim=True).sqrt())).max()
            assert rel.item() <= (1e-5 if dt == torch.float32 else 2e-2), (it, T, H, off, budget, dt)
            if gather:
                g = comm.buffer(rng.randrange(W), 2, (off + T, H), dt)[off:].float()
                assert torch.allclose(g, torch.cat(shards).float())
        checked += 1
    comm.check()
    comm.close()
    assert checked == 600


def test_k2_soak_random_launches(cuda):
    """K2 under the shipped engine policy: 400 random (T, H, dtype, SM budget,
    in-place) launches -- engine, row-group count and ring wrap change from
    launch to launch -- each against a torch fp32 restatement (residual
    bitwise to RNE, output to the north_star tolerance)."""
    import torch
    import paper_2505_11329_b200 as tw
    rng = random.Random(4321)
    for it in range(400):
        dt = rng.choice([torch.bfloat16, torch.float32])
        H = rng.choice([8, 33, 1024, 4096, 6144, 8192])
        T = rng.choice([1, 2, 7, 64, 300, 1024, 2500])
        budget = rng.choice([0, 0, 1, 2, 8, 33, 148])
        inplace = rng.random() < 0.3
        x = torch.randn(T, H, device="cuda").to(dt)
        r = torch.randn(T, H, device="cuda").to(dt)
        w = torch.rand(H, device="cuda") + 0.5
        rp = (x.float() + r.float()).to(dt).float()
        want = rp * torch.rsqrt((rp * rp).mean(1, keepdim=True) + 1e-5) * w
        out, rout = tw.rmsnorm_residual(x, r, w, residual_out=r if inplace else None, sm_budget=budget)
        torch.cuda.synchronize()
        assert torch.equal(rout.float(), rp), (it, T, H, dt, budget)
        rel = ((out.float() - want).abs() / torch.maximum(want.abs(), want.pow(2).mean(1, keepdim=True).sqrt())).max()
        assert rel.item() <= (1e-5 if dt == torch.float32 else 2e-2), (it, T, H, dt, budget, rel.item())
