"""K1 -- fused AllReduce + residual-add + RMSNorm on the GPU vs the oracle
(weavesim::fused_allreduce_rmsnorm, proj/src/collectives.cpp:157-182).

Ranks are simulated on one device (PEER transport over one communicator, the
reference's in-process RankGroup, proj/include/weavesim/collectives.hpp:34-46);
the NVLS transport needs >= 2 NVSwitch-attached GPUs and is exercised by the
multi-GPU tests at the bottom when they are visible.

Tolerances: fp32 -- residual shards bitwise (rank-ascending fp32 sum, same as
proj/src/collectives.cpp:140-144), output <= 1e-5; bf16 -- residual shards
bitwise equal to RNE(oracle r'), output 2e-2 relative (row-rms guarded)."""
import numpy as np
import pytest

from tests.helpers import assert_abs_close, assert_bf16_close, bf16_round, group_inputs

pytestmark = pytest.mark.gpu


def setup_group(comm, inputs, residual, weight, ranges, dtype):
    import torch
    W, T, H = inputs.shape
    for r in range(W):
        comm.buffer(r, 0, (T, H), dtype).copy_(torch.from_numpy(inputs[r]).to(dtype))
        comm.buffer(r, 1, (T, H), dtype).fill_(float("nan"))
    shards = [torch.from_numpy(np.ascontiguousarray(residual[b:e])).to("cuda", dtype) for b, e in ranges]
    weights = [torch.from_numpy(weight).cuda() for _ in range(W)]
    return shards, weights


def run_k1(inputs, residual, weight, dtype, ranges=None, gather=False, sm_budget=4, comm=None):
    import torch
    import paper_2505_11329_b200 as tw
    W, T, H = inputs.shape
    if ranges is None:
        ranges = tw.token_shard_map(T, W)
    own = comm is None
    if own:
        comm = tw.Communicator(W, [0] * W, max(T * H * 4, 1), tw.TW_TRANSPORT_PEER)
    shards, weights = setup_group(comm, inputs, residual, weight, ranges, dtype)
    comm.fused_allreduce_rmsnorm(T, H, shards, weights, shard_ranges=ranges, sm_budget=sm_budget,
                                 gather_residual=gather, dtype=dtype)
    torch.cuda.synchronize()
    comm.check()
    outs = [comm.buffer(r, 1, (T, H), dtype).float().cpu().numpy() for r in range(W)]
    res = [s.float().cpu().numpy() for s in shards]
    gathered = [comm.buffer(r, 2, (T, H), dtype).float().cpu().numpy() for r in range(W)] if gather else None
    if own:
        comm.close()
    return outs, res, gathered


def oracle_case(orc, inputs, residual, weight, ranges, bf16):
    if bf16:
        inputs, residual = bf16_round(inputs), bf16_round(residual)
    shards = [residual[b:e] for b, e in ranges]
    out, new = orc.fused_allreduce_rmsnorm(list(inputs), shards, weight, ranges)
    return inputs, residual, out, new


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("T", [1, 3, 17, 40, 256])
@pytest.mark.parametrize("H", [16, 24, 33, 64, 1024])
def test_k1_fp32_matches_oracle(cuda, orc, world, T, H):
    import torch
    import paper_2505_11329_b200 as tw
    inputs, residual, weight = group_inputs(77 * world + T + H, world, T, H)
    ranges = tw.token_shard_map(T, world)
    _, _, want_out, want_res = oracle_case(orc, inputs, residual, weight, ranges, False)
    outs, res, _ = run_k1(inputs, residual, weight, torch.float32)
    for r in range(world):
        assert_abs_close(outs[r], want_out, 1e-5, f"rank {r} output")
        assert np.array_equal(res[r], want_res[r]), f"rank {r} residual shard must be bitwise"
        assert np.array_equal(outs[r], outs[0]), "replicated output must be identical on every rank"


@pytest.mark.parametrize("world", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("T,H", [(1, 16), (17, 64), (40, 33), (256, 1024), (128, 8192), (64, 6144)])
def test_k1_bf16_matches_oracle(cuda, orc, world, T, H):
    import torch
    import paper_2505_11329_b200 as tw
    inputs, residual, weight = group_inputs(5 * world + T * 3 + H, world, T, H)
    ranges = tw.token_shard_map(T, world)
    inputs, residual, want_out, want_res = oracle_case(orc, inputs, residual, weight, ranges, True)
    outs, res, _ = run_k1(inputs, residual, weight, torch.bfloat16)
    for r in range(world):
        assert_bf16_close(outs[r], want_out, what=f"rank {r} output")
        assert np.array_equal(res[r], bf16_round(want_res[r])), f"rank {r} residual shard"


def test_k1_matches_golden_fixtures(cuda, golden):
    """The reference's own outputs (tests/golden, from oracle/_ref)."""
    import torch
    meta, arrays = golden
    for case in meta["fused"]:
        inputs, residual, weight = group_inputs(case["seed"], case["world"], case["T"], case["H"])
        ranges = [tuple(r) for r in case["ranges"]]
        outs, res, _ = run_k1(inputs, residual, weight, torch.float32, ranges=ranges)
        assert_abs_close(outs[0], arrays[f"fused_{case['id']}_out"], 1e-5)
        assert np.array_equal(np.concatenate(res), arrays[f"fused_{case['id']}_res"])


@pytest.mark.parametrize("W,H", [(4, 256), (8, 1024), (8, 8192)])
@pytest.mark.parametrize("dtype_name", ["float32", "bfloat16"])
def test_k1_gather_residual(cuda, orc, dtype_name, W, H):
    """G=2 (north_star): r' is all-gathered to every rank's RESIDUAL buffer
    (W = 8: the bulk-copy engine's two-stage rows, lazily and immediately
    released rings)."""
    import torch
    import paper_2505_11329_b200 as tw
    dtype = getattr(torch, dtype_name)
    T = 37
    inputs, residual, weight = group_inputs(9, W, T, H)
    ranges = tw.token_shard_map(T, W)
    inputs, residual, want_out, want_res = oracle_case(orc, inputs, residual, weight, ranges,
                                                       dtype == torch.bfloat16)
    outs, res, gathered = run_k1(inputs, residual, weight, dtype, gather=True)
    full = np.concatenate(want_res)
    if dtype == torch.bfloat16:
        full = bf16_round(full)
    for r in range(W):
        assert np.array_equal(gathered[r], full)


@pytest.mark.parametrize("transport", ["peer", "nvls_sim"])
def test_k1_colocated_per_rank_streams_are_joined(cuda, orc, transport):
    """Co-located ranks launch as one grid on streams[0]; every other rank's
    stream is joined before the launch and released after it: rank r's input
    produced late on its own stream (behind a sleep kernel) is still what K1
    reads, and work queued on stream r after the call sees K1's output."""
    import torch
    import paper_2505_11329_b200 as tw
    W, T, H = 4, 64, 1024
    tr = tw.TW_TRANSPORT_PEER if transport == "peer" else tw.TW_TRANSPORT_NVLS_SIM
    comm = tw.Communicator(W, [0] * W, T * H * 4, tr)
    inputs, residual, weight = group_inputs(4242, W, T, H)
    ranges = tw.token_shard_map(T, W)
    inputs, residual, want_out, want_res = oracle_case(orc, inputs, residual, weight, ranges, True)
    streams = [torch.cuda.Stream() for _ in range(W)]
    shards = [torch.from_numpy(np.ascontiguousarray(residual[b:e])).cuda().bfloat16() for b, e in ranges]
    wts = [torch.from_numpy(weight).cuda() for _ in range(W)]
    host = [torch.from_numpy(inputs[r]).bfloat16().pin_memory() for r in range(W)]
    for r in range(W):
        comm.buffer(r, 0, (T, H), torch.bfloat16).fill_(float("nan"))
    torch.cuda.synchronize()
    for r in range(W):
        with torch.cuda.stream(streams[r]):
            torch.cuda._sleep(2_000_000)  # ~1 ms: the input lands well after the launch is enqueued
            comm.buffer(r, 0, (T, H), torch.bfloat16).copy_(host[r], non_blocking=True)
    comm.fused_allreduce_rmsnorm(T, H, shards, wts, shard_ranges=ranges, sm_budget=4, streams=streams)
    copies = []
    for r in range(W):
        with torch.cuda.stream(streams[r]):
            copies.append(comm.buffer(r, 1, (T, H), torch.bfloat16).float().clone())
    torch.cuda.synchronize()
    comm.check()
    for r in range(W):
        assert_bf16_close(copies[r].cpu().numpy(), want_out, what=f"rank {r} output read on its stream")
        got = shards[r].float().cpu().numpy()
        if transport == "peer":
            assert np.array_equal(got, bf16_round(want_res[r])), f"rank {r} residual"
        else:  # NVLS rounds the reduced sum once more (tests/test_nvls_gpu.py)
            assert_bf16_close(got, want_res[r], what=f"rank {r} residual")
    comm.close()


def test_k1_uneven_and_empty_shards(cuda, orc):
    """Custom shard maps, including empty ranges (T < N)."""
    import torch
    for W, T, ranges in [(8, 3, None), (4, 10, [(0, 7), (7, 7), (7, 9), (9, 10)]),
                         (2, 9, [(0, 0), (0, 9)])]:
        inputs, residual, weight = group_inputs(T + W, W, T, 64)
        if ranges is None:
            ranges = orc.token_shard_map(T, W)
        _, _, want_out, want_res = oracle_case(orc, inputs, residual, weight, ranges, False)
        outs, res, _ = run_k1(inputs, residual, weight, torch.float32, ranges=ranges)
        for r in range(W):
            assert_abs_close(outs[r], want_out, 1e-5)
            assert np.array_equal(res[r].reshape(-1), want_res[r].reshape(-1))


def test_k1_contract_and_shape_errors(cuda):
    import torch
    import paper_2505_11329_b200 as tw
    W, T, H = 4, 8, 64
    comm = tw.Communicator(W, [0] * W, T * H * 4, tw.TW_TRANSPORT_PEER)
    shards = [torch.zeros(2, H, device="cuda") for _ in range(W)]
    weights = [torch.ones(H, device="cuda") for _ in range(W)]
    bad = [(0, 2), (1, 4), (4, 6), (6, 8)]  # overlap: proj/tests/test_collectives.cpp:154-156
    with pytest.raises(tw.ContractError):
        comm.fused_allreduce_rmsnorm(T, H, shards, weights, shard_ranges=bad)
    with pytest.raises(tw.ContractError):
        comm.fused_allreduce_rmsnorm(T, H, shards, weights, shard_ranges=[(0, 2), (2, 4), (4, 6), (6, 9)])
    with pytest.raises(tw.DimensionError):  # exceeds the symmetric buffers
        comm.fused_allreduce_rmsnorm(T * 2, H, shards, weights)
    with pytest.raises(tw.NumericError):
        comm.fused_allreduce_rmsnorm(T, H, shards, weights, eps=-1.0)
    with pytest.raises(tw.ConfigError):
        tw.Communicator(1, [0], 1024, tw.TW_TRANSPORT_PEER).fused_allreduce_rmsnorm(T, H, shards[:1], weights[:1])
    comm.close()


def test_k1_repeated_launches_and_budgets(cuda, orc):
    """Signal-pad epochs stay consistent across many launches with varying
    SM budgets and shapes on one communicator (no reset, no timeout)."""
    import torch
    import paper_2505_11329_b200 as tw
    W, H = 8, 512
    comm = tw.Communicator(W, [0] * W, 300 * H * 4, tw.TW_TRANSPORT_PEER)
    for it, (T, budget) in enumerate([(1, 1), (256, 2), (17, 4), (300, 8), (64, 16), (5, 3), (200, 12)] * 3):
        inputs, residual, weight = group_inputs(it, W, T, H)
        ranges = tw.token_shard_map(T, W)
        inputs, residual, want_out, want_res = oracle_case(orc, inputs, residual, weight, ranges, True)
        outs, res, _ = run_k1(inputs, residual, weight, torch.bfloat16, sm_budget=budget, comm=comm)
        assert_bf16_close(outs[W - 1], want_out)
    comm.check()
    comm.close()


@pytest.mark.parametrize("dtype_name", ["float32", "bfloat16"])
@pytest.mark.parametrize("H", [1024, 4096, 8192])
def test_k1_world2_row_groups_across_budgets(cuda, orc, dtype_name, H):
    """World 2 runs the PEER engine with two consumer row groups
    (tw_launch.cu peer_tma_groups): parity at budgets from one CTA (every
    row of a rank in one CTA, odd and even counts) to the full grid, one
    communicator across launches."""
    import torch
    import paper_2505_11329_b200 as tw
    W = 2
    dtype = getattr(torch, dtype_name)
    bf16 = dtype == torch.bfloat16
    comm = tw.Communicator(W, [0] * W, 301 * H * 4, tw.TW_TRANSPORT_PEER)
    for it, (T, budget) in enumerate([(301, 1), (300, 2), (77, 8), (64, 74), (150, 75), (301, 148), (5, 16)]):
        inputs, residual, weight = group_inputs(31 * it + H, W, T, H)
        ranges = tw.token_shard_map(T, W)
        inputs, residual, want_out, want_res = oracle_case(orc, inputs, residual, weight, ranges, bf16)
        outs, res, gathered = run_k1(inputs, residual, weight, dtype, gather=True, sm_budget=budget, comm=comm)
        full_res = np.concatenate([bf16_round(x) if bf16 else x for x in want_res])
        for r in range(W):
            if bf16:
                assert_bf16_close(outs[r], want_out, what=f"budget {budget} rank {r} output")
                assert np.array_equal(res[r], bf16_round(want_res[r])), f"budget {budget} rank {r} residual"
            else:
                assert_abs_close(outs[r], want_out, 1e-5, f"budget {budget} rank {r} output")
                assert np.array_equal(res[r], want_res[r]), f"budget {budget} rank {r} residual"
            assert np.array_equal(gathered[r], full_res), f"budget {budget} rank {r} gathered residual"
    comm.check()
    comm.close()


_FORCED_GROUPS = r"""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2505_11329_b200 as tw
from tests.helpers import group_inputs, bf16_round
from tests.test_k1_gpu import run_k1, oracle_case
import oracle
orc = oracle.Oracle()
for W, H, T, budget in [(2, 8192, 97, 4), (2, 1024, 200, 148), (3, 8192, 97, 4), (3, 2048, 64, 3), (3, 512, 33, 98)]:
    inputs, residual, weight = group_inputs(W * 7 + H + T, W, T, H)
    ranges = tw.token_shard_map(T, W)
    inputs, residual, want_out, want_res = oracle_case(orc, inputs, residual, weight, ranges, False)
    outs, res, _ = run_k1(inputs, residual, weight, torch.float32, sm_budget=budget)
    for r in range(W):
        assert np.abs(outs[r] - want_out).max() <= 1e-5, (W, H, T, r)
        assert np.array_equal(res[r], want_res[r]), (W, H, T, r)
print("ok")
"""


@pytest.mark.parametrize("groups", ["1", "2"])
def test_k1_peer_forced_row_groups(cuda, groups):
    """TW_K1_PEER_GROUPS forces one or two row groups for worlds 2 and 3 (the
    env is read once per process, so each setting runs in its own)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TW_K1_PEER_GROUPS=groups)
    out = subprocess.run([sys.executable, "-c", _FORCED_GROUPS], cwd=root, env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stdout + out.stderr


@pytest.mark.parametrize("dtype_name", ["float32", "bfloat16"])
def test_k1_baseline_config0(cuda, orc, dtype_name):
    """BASELINE.json configs[0]: 2 ranks, 1024 tokens x 4096 hidden, vs the
    oracle on the same inputs (the reference's CPU-runnable case)."""
    import torch
    dtype = getattr(torch, dtype_name)
    W, T, H = 2, 1024, 4096
    inputs, residual, weight = group_inputs(2505, W, T, H)
    import paper_2505_11329_b200 as tw
    ranges = tw.token_shard_map(T, W)
    inputs, residual, want_out, want_res = oracle_case(orc, inputs, residual, weight, ranges,
                                                       dtype == torch.bfloat16)
    outs, res, _ = run_k1(inputs, residual, weight, dtype, sm_budget=16)
    for r in range(W):
        if dtype == torch.float32:
            assert_abs_close(outs[r], want_out, 1e-5)
            assert np.array_equal(res[r], want_res[r])
        else:
            assert_bf16_close(outs[r], want_out)
            assert np.array_equal(res[r], bf16_round(want_res[r]))


def test_k1_known_answers(cuda):
    """N=2, T=2, H=2, inputs all ones, residual 0, w 1, eps 0 ->
    out 1.0, residual 2.0; SPEC.md:104-105 -- AllReduce of N=4 ones -> 4 and of
    rank-constant r -> 6 (K3)."""
    import torch
    import paper_2505_11329_b200 as tw
    for dt in (torch.float32, torch.bfloat16):
        comm = tw.Communicator(2, [0, 0], 64, tw.TW_TRANSPORT_PEER)
        for q in range(2):
            comm.buffer(q, 0, (2, 2), dt).fill_(1.0)
        shards = [torch.zeros(1, 2, device="cuda", dtype=dt) for _ in range(2)]
        comm.fused_allreduce_rmsnorm(2, 2, shards, [torch.ones(2, device="cuda")] * 2, eps=0.0, dtype=dt)
        torch.cuda.synchronize()
        for q in range(2):
            assert torch.all(comm.buffer(q, 1, (2, 2), dt) == 1.0)
            assert torch.all(shards[q] == 2.0)
        comm.close()
        comm = tw.Communicator(4, [0] * 4, 3 * 8 * 4, tw.TW_TRANSPORT_PEER)
        for q in range(4):
            comm.buffer(q, 0, (3, 8), dt).fill_(1.0)
        comm.allreduce(3, 8, dt)
        torch.cuda.synchronize()
        assert all(torch.all(comm.buffer(q, 1, (3, 8), dt) == 4.0) for q in range(4))
        for q in range(4):
            comm.buffer(q, 0, (3, 8), dt).fill_(float(q))
        comm.allreduce(3, 8, dt)
        torch.cuda.synchronize()
        assert all(torch.all(comm.buffer(q, 1, (3, 8), dt) == 6.0) for q in range(4))
        comm.close()


def test_k1_barrier_timeout_fault_injection(cuda, monkeypatch):
    """A rank that never arrives must not hang the GPU: the bounded spin raises
    the timeout flag and tw_comm_check reports BarrierTimeout."""
    import torch
    import paper_2505_11329_b200 as tw
    W, T, H = 4, 64, 256
    comm = tw.Communicator(W, [0] * W, T * H * 2, tw.TW_TRANSPORT_PEER)
    shards = [torch.zeros(T // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    w = [torch.ones(H, device="cuda")] * W
    comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=2)
    torch.cuda.synchronize()
    comm.check()  # healthy
    monkeypatch.setenv("TW_FAULT_DROP_ARRIVAL_RANK", "2")
    monkeypatch.setenv("TW_BARRIER_SPIN_LIMIT", "20000")
    comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=2)
    torch.cuda.synchronize()
    with pytest.raises(tw.BarrierTimeout):
        comm.check()
    comm.close()
    monkeypatch.delenv("TW_FAULT_DROP_ARRIVAL_RANK")
    monkeypatch.delenv("TW_BARRIER_SPIN_LIMIT")
    fresh = tw.Communicator(W, [0] * W, T * H * 2, tw.TW_TRANSPORT_PEER)
    fresh.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=2)
    torch.cuda.synchronize()
    fresh.check()  # a recreated communicator is healthy again
    fresh.close()


def test_k3_allreduce_baseline(cuda, orc):
    import torch
    import paper_2505_11329_b200 as tw
    W, T, H = 8, 100, 1024
    inputs, _, _ = group_inputs(3, W, T, H)
    comm = tw.Communicator(W, [0] * W, T * H * 4, tw.TW_TRANSPORT_PEER)
    for r in range(W):
        comm.buffer(r, 0, (T, H), torch.float32).copy_(torch.from_numpy(inputs[r]))
    comm.allreduce(T, H, torch.float32, sm_budget=4)
    torch.cuda.synchronize()
    want = orc.all_reduce(list(inputs))
    for r in range(W):
        assert np.array_equal(comm.buffer(r, 1, (T, H), torch.float32).cpu().numpy(), want)
    comm.close()


def test_k1_full_size_llama_boundary_property(cuda, orc):
    """C2 shape (N=8, T=1024, H=8192, bf16) on simulated ranks: the output is
    the RMSNorm of the gathered residual (size-independent property) and a row
    sample matches the oracle."""
    import torch
    import paper_2505_11329_b200 as tw
    W, T, H = 8, 1024, 8192
    comm = tw.Communicator(W, [0] * W, T * H * 2, tw.TW_TRANSPORT_PEER)
    g = torch.Generator(device="cuda").manual_seed(1)
    parts = [(torch.rand(T, H, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(W)]
    res_full = (torch.rand(T, H, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w = torch.rand(H, device="cuda", generator=g) + 0.5
    ranges = tw.token_shard_map(T, W)
    for r in range(W):
        comm.buffer(r, 0, (T, H), torch.bfloat16).copy_(parts[r])
    shards = [res_full[b:e].clone() for b, e in ranges]
    comm.fused_allreduce_rmsnorm(T, H, shards, [w] * W, sm_budget=8, gather_residual=True)
    torch.cuda.synchronize()
    comm.check()
    summed = sum(p.float() for p in parts)
    want_res = (summed + res_full.float()).to(torch.bfloat16)
    assert torch.equal(torch.cat(shards), want_res)
    rb = want_res.float()
    want = rb * torch.rsqrt((rb * rb).mean(1, keepdim=True) + 1e-5) * w
    for r in range(W):
        out = comm.buffer(r, 1, (T, H), torch.bfloat16).float()
        rel = ((out - want).abs() / torch.maximum(want.abs(), want.pow(2).mean(1, keepdim=True).sqrt())).max()
        assert rel.item() <= 2e-2
        assert torch.equal(comm.buffer(r, 2, (T, H), torch.bfloat16), want_res)
    # rows are independent: the oracle on a row sample (as its own T' problem)
    rows = list(range(0, T, 131))
    ins = np.stack([p[rows].float().cpu().numpy() for p in parts])
    res_rows = res_full[rows].float().cpu().numpy()
    sub = orc.token_shard_map(len(rows), W)
    o, new = orc.fused_allreduce_rmsnorm(list(ins), [res_rows[b:e] for b, e in sub], w.cpu().numpy(), sub)
    assert np.array_equal(bf16_round(np.concatenate(new)), want_res[rows].float().cpu().numpy())
    assert_bf16_close(comm.buffer(0, 1, (T, H), torch.bfloat16)[rows].float().cpu().numpy(), o)
    comm.close()


@pytest.mark.skipif("__import__('torch').cuda.device_count() < 2")
@pytest.mark.parametrize("dtype_name", ["float32", "bfloat16"])
def test_k1_nvls_multi_gpu(cuda, orc, dtype_name):
    import torch
    import paper_2505_11329_b200 as tw
    n = min(torch.cuda.device_count(), 8)
    dtype = getattr(torch, dtype_name)
    T, H = 257, 8192 if dtype == torch.bfloat16 else 1024
    comm = tw.Communicator(n, list(range(n)), T * H * 4, tw.TW_TRANSPORT_NVLS)
    inputs, residual, weight = group_inputs(21, n, T, H)
    ranges = tw.token_shard_map(T, n)
    inputs, residual, want_out, want_res = oracle_case(orc, inputs, residual, weight, ranges, dtype == torch.bfloat16)
    shards, weights = [], []
    for r in range(n):
        comm.buffer(r, 0, (T, H), dtype).copy_(torch.from_numpy(inputs[r]).to(dtype))
        b, e = ranges[r]
        shards.append(torch.from_numpy(np.ascontiguousarray(residual[b:e])).to(f"cuda:{r}", dtype))
        weights.append(torch.from_numpy(weight).to(f"cuda:{r}"))
    comm.fused_allreduce_rmsnorm(T, H, shards, weights, sm_budget=8, gather_residual=True,
                                 streams=[torch.cuda.current_stream(r) for r in range(n)])
    for r in range(n):
        torch.cuda.synchronize(r)
    comm.check()
    for r in range(n):
        out = comm.buffer(r, 1, (T, H), dtype).float().cpu().numpy()
        if dtype == torch.float32:
            assert_abs_close(out, want_out, 1e-5)
        else:
            assert_bf16_close(out, want_out)
    comm.close()
