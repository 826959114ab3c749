"""K1 over NVLS -- the north_star kernel (tw_nvls.cuh) -- vs the oracle
(weavesim::fused_allreduce_rmsnorm, proj/src/collectives.cpp:157-182).

Two halves:

* NVLS_SIM (one GPU, always run): the NVLS kernels themselves on simulated
  ranks sharing the device, with each multimem instruction spelled as
  per-rank loads / stores / reductions (MmSim).  Row partition, the
  ld_reduce pipeline at every depth, barrier phases and device-resident
  generations, G = 2 and the fences are the same instantiated code as on an
  NVSwitch box.
* NVLS hardware (>= 2 GPUs with multicast, skipped otherwise): the C2 shapes
  (N = 2/4/8, T = 1024-8192, H = 8192, G = 1/2, bf16 and fp32), repeated
  launches, graph replay, the timeout path and a multi-process (one process
  per GPU) run.

Numerics.  An NVLS reduction of bf16 partials returns bf16 (multimem.ld_reduce
.acc::f32.bf16x2 accumulates in fp32 and rounds once), so the kernel's
r' = RNE(RNE(sum) + res): MmSim reproduces that exactly (rank-ascending fp32
sum), which the tests check bitwise against a numpy model; against the fp32
oracle both r' and the output meet north_star's 2e-2 relative bar (row-rms
guarded).  fp32: MmSim's sum is the reference's rank-ascending order, so the
residual is bitwise and the output <= 1e-5; on hardware the switch's order is
unspecified, so <= 1e-5 for both."""
import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest

from tests.conftest import ROOT
from tests.helpers import assert_abs_close, assert_bf16_close, bf16_round, group_inputs

pytestmark = pytest.mark.gpu


def nvls_model_residual(inputs, residual_rows):
    """r' of the NVLS kernel on bf16 data: RNE(RNE(rank-ascending fp32 sum) + res)."""
    acc = np.zeros(inputs.shape[1:], np.float32)
    for q in range(inputs.shape[0]):
        acc = (acc + inputs[q]).astype(np.float32)
    return acc, lambda rows, res: bf16_round(bf16_round(acc[rows]) + res)


def make_comm(W, nbytes, transport=None):
    import paper_2505_11329_b200 as tw
    t = tw.TW_TRANSPORT_NVLS_SIM if transport is None else transport
    devices = [0] * W if t == tw.TW_TRANSPORT_NVLS_SIM else list(range(W))
    return tw.Communicator(W, devices, max(nbytes, 1), t)


def run_nvls(comm, inputs, residual, weight, dtype, ranges, gather=False, sm_budget=4, depth=0, reps=1):
    import torch
    W, T, H = inputs.shape
    dev = lambda r: comm.devices[r]  # noqa: E731
    for r in range(W):
        comm.buffer(r, 0, (T, H), dtype).copy_(torch.from_numpy(inputs[r]).to(dtype))
        comm.buffer(r, 1, (T, H), dtype).fill_(float("nan"))
        if gather:
            comm.buffer(r, 2, (T, H), dtype).fill_(float("nan"))
    weights = [torch.from_numpy(weight).to(f"cuda:{dev(r)}") for r in range(W)]
    for _ in range(reps):
        shards = [torch.from_numpy(np.ascontiguousarray(residual[b:e])).to(f"cuda:{dev(r)}", dtype)
                  for r, (b, e) in enumerate(ranges)]
        comm.fused_allreduce_rmsnorm(T, H, shards, weights, shard_ranges=ranges, sm_budget=sm_budget,
                                     gather_residual=gather, dtype=dtype, nvls_depth=depth)
        for d in set(comm.devices):
            torch.cuda.synchronize(d)
    comm.check()
    outs = [comm.buffer(r, 1, (T, H), dtype).float().cpu().numpy() for r in range(W)]
    res = [s.float().cpu().numpy() for s in shards]
    gathered = [comm.buffer(r, 2, (T, H), dtype).float().cpu().numpy() for r in range(W)] if gather else None
    return outs, res, gathered


def check_case(orc, inputs, residual, weight, ranges, dtype, outs, res, gathered, exact_sum=True):
    """Compare one run with the oracle (and, for bf16, the NVLS rounding model)."""
    import torch
    bf16 = dtype == torch.bfloat16
    shards = [residual[b:e] for b, e in ranges]
    want_out, want_res = orc.fused_allreduce_rmsnorm(list(inputs), shards, weight, ranges)
    W = len(ranges)
    H = inputs.shape[2]
    if bf16:
        _, model = nvls_model_residual(inputs, residual)
        full_model = []
        for r, (b, e) in enumerate(ranges):
            got = res[r].reshape(e - b, H)
            if exact_sum:
                assert np.array_equal(got, model(slice(b, e), residual[b:e])), f"rank {r}: r' != RNE(RNE(sum)+res)"
            assert_bf16_close(got, want_res[r].reshape(e - b, H), what=f"rank {r} residual vs oracle")
            full_model.append(got)
        for r in range(W):
            assert_bf16_close(outs[r], want_out, what=f"rank {r} output")
            assert np.array_equal(outs[r], outs[0]), "replicated output must be identical on every rank"
        if gathered is not None:
            full = np.concatenate(full_model)
            for r in range(W):
                assert np.array_equal(gathered[r], full), f"rank {r} gathered residual"
    else:
        for r, (b, e) in enumerate(ranges):
            got = res[r].reshape(e - b, H)
            if exact_sum:
                assert np.array_equal(got, want_res[r].reshape(e - b, H)), f"rank {r} residual must be bitwise"
            else:
                assert_abs_close(got, want_res[r].reshape(e - b, H), 1e-5, f"rank {r} residual")
        for r in range(W):
            assert_abs_close(outs[r], want_out, 1e-5, f"rank {r} output")
            assert np.array_equal(outs[r], outs[0])
        if gathered is not None:
            full = np.concatenate([r_.reshape(-1, H) for r_ in res])
            for r in range(W):
                assert np.array_equal(gathered[r], full)


def bf16_inputs(seed, W, T, H):
    inputs, residual, weight = group_inputs(seed, W, T, H)
    return bf16_round(inputs), bf16_round(residual), weight


# ---- NVLS_SIM: the NVLS kernels on one GPU --------------------------------------------------------

@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("T,H", [(1, 16), (3, 64), (17, 1024), (40, 8), (256, 8192), (33, 4096)])
@pytest.mark.parametrize("depth", [1, 2, 3])
def test_nvls_sim_fp32(cuda, orc, world, T, H, depth):
    import torch
    import paper_2505_11329_b200 as tw
    inputs, residual, weight = group_inputs(31 * world + T + H + depth, world, T, H)
    ranges = tw.token_shard_map(T, world)
    comm = make_comm(world, T * H * 4)
    outs, res, _ = run_nvls(comm, inputs, residual, weight, torch.float32, ranges, depth=depth)
    comm.close()
    check_case(orc, inputs, residual, weight, ranges, torch.float32, outs, res, None)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("T,H", [(1, 16), (17, 64), (40, 1024), (128, 8192), (64, 6144), (37, 16384)])
@pytest.mark.parametrize("depth", [1, 2, 3])
def test_nvls_sim_bf16(cuda, orc, world, T, H, depth):
    import torch
    import paper_2505_11329_b200 as tw
    inputs, residual, weight = bf16_inputs(5 * world + 3 * T + H + depth, world, T, H)
    ranges = tw.token_shard_map(T, world)
    comm = make_comm(world, T * H * 2)
    outs, res, _ = run_nvls(comm, inputs, residual, weight, torch.bfloat16, ranges, depth=depth)
    comm.close()
    check_case(orc, inputs, residual, weight, ranges, torch.bfloat16, outs, res, None)


@pytest.mark.parametrize("dtype_name", ["float32", "bfloat16"])
@pytest.mark.parametrize("W,H", [(2, 8192), (4, 256), (8, 8192)])
def test_nvls_sim_gather_residual(cuda, orc, dtype_name, W, H):
    """G = 2 (north_star): r' multicast to every rank's RESIDUAL buffer."""
    import torch
    import paper_2505_11329_b200 as tw
    dtype = getattr(torch, dtype_name)
    T = 45
    inputs, residual, weight = (bf16_inputs if dtype == torch.bfloat16 else group_inputs)(9 + W, W, T, H)
    ranges = tw.token_shard_map(T, W)
    comm = make_comm(W, T * H * 4)
    outs, res, gathered = run_nvls(comm, inputs, residual, weight, dtype, ranges, gather=True, sm_budget=3)
    comm.close()
    check_case(orc, inputs, residual, weight, ranges, dtype, outs, res, gathered)


def test_nvls_sim_golden_fixtures(cuda, golden):
    """The reference's own outputs (tests/golden, generated from oracle/_ref)."""
    import torch
    meta, arrays = golden
    cases = [c for c in meta["fused"] if c["H"] % 4 == 0]  # the NVLS kernels move 16-byte vectors
    assert len(cases) >= 36
    for case in cases:
        inputs, residual, weight = group_inputs(case["seed"], case["world"], case["T"], case["H"])
        ranges = [tuple(r) for r in case["ranges"]]
        comm = make_comm(case["world"], case["T"] * case["H"] * 4)
        outs, res, _ = run_nvls(comm, inputs, residual, weight, torch.float32, ranges)
        comm.close()
        assert_abs_close(outs[0], arrays[f"fused_{case['id']}_out"], 1e-5)
        assert np.array_equal(np.concatenate([x.reshape(-1, case["H"]) for x in res]),
                              arrays[f"fused_{case['id']}_res"])


def test_nvls_sim_uneven_and_empty_shards(cuda, orc):
    """Custom shard maps with empty ranges (T < N)."""
    import torch
    for W, T, ranges in [(8, 3, None), (4, 10, [(0, 7), (7, 7), (7, 9), (9, 10)]), (2, 9, [(0, 0), (0, 9)])]:
        inputs, residual, weight = group_inputs(T + W, W, T, 64)
        if ranges is None:
            ranges = orc.token_shard_map(T, W)
        comm = make_comm(W, T * 64 * 4)
        outs, res, _ = run_nvls(comm, inputs, residual, weight, torch.float32, ranges)
        comm.close()
        check_case(orc, inputs, residual, weight, ranges, torch.float32, outs, res, None)


def test_nvls_sim_repeated_launches_budgets_depths(cuda, orc):
    """Barrier generations stay consistent across many launches on one
    communicator while SM budget, depth, shape and G change (no reset)."""
    import torch
    import paper_2505_11329_b200 as tw
    W, H = 8, 1024
    comm = make_comm(W, 300 * H * 2)
    plan = [(1, 1, 1), (256, 2, 2), (17, 4, 3), (300, 8, 2), (64, 16, 1), (5, 3, 3), (200, 12, 2)] * 3
    for it, (T, budget, depth) in enumerate(plan):
        inputs, residual, weight = bf16_inputs(it, W, T, H)
        ranges = tw.token_shard_map(T, W)
        outs, res, g = run_nvls(comm, inputs, residual, weight, torch.bfloat16, ranges, gather=bool(it & 1),
                                sm_budget=budget, depth=depth)
        check_case(orc, inputs, residual, weight, ranges, torch.bfloat16, outs, res, g)
    comm.close()


def test_nvls_sim_graph_replay(cuda, orc):
    """K1 captured once in a CUDA graph and replayed with new inputs each time:
    the barrier generation lives on the device, so no host epoch goes stale."""
    import torch
    import paper_2505_11329_b200 as tw
    W, T, H = 4, 96, 2048
    comm = make_comm(W, T * H * 2)
    ranges = tw.token_shard_map(T, W)
    shards = [torch.zeros(e - b, H, device="cuda", dtype=torch.bfloat16) for b, e in ranges]
    wt = torch.ones(H, device="cuda")
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):  # warm-up launch (first-use setup outside the capture)
        comm.fused_allreduce_rmsnorm(T, H, shards, [wt] * W, sm_budget=4, gather_residual=True)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        comm.fused_allreduce_rmsnorm(T, H, shards, [wt] * W, sm_budget=4, gather_residual=True)
    for it in range(6):
        inputs, residual, weight = bf16_inputs(100 + it, W, T, H)
        weight = np.ones(H, np.float32)
        for r in range(W):
            comm.buffer(r, 0, (T, H), torch.bfloat16).copy_(torch.from_numpy(inputs[r]).bfloat16())
            comm.buffer(r, 1, (T, H), torch.bfloat16).fill_(float("nan"))
        for r, (b, e) in enumerate(ranges):
            shards[r].copy_(torch.from_numpy(residual[b:e]).bfloat16())
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        comm.check()
        outs = [comm.buffer(r, 1, (T, H), torch.bfloat16).float().cpu().numpy() for r in range(W)]
        gathered = [comm.buffer(r, 2, (T, H), torch.bfloat16).float().cpu().numpy() for r in range(W)]
        check_case(orc, inputs, residual, weight, ranges, torch.bfloat16, outs,
                   [s.float().cpu().numpy() for s in shards], gathered)
    comm.close()


@pytest.mark.parametrize("env", [{"TW_NVLS_ALIAS_FENCE": "1"}, {"TW_FORCE_SYS_SCOPE": "1"},
                                 {"TW_NVLS_ALIAS_FENCE": "1", "TW_FORCE_SYS_SCOPE": "1"}])
def test_nvls_sim_barrier_variants(cuda, env):
    """The barrier options read once per process (the optional proxy-alias
    fence at exit; system-scope fences for co-located ranks): parity and
    repeated launches in a fresh process with each set."""
    code = textwrap.dedent("""
        import sys
        sys.path.insert(0, ".")
        import numpy as np, torch
        import paper_2505_11329_b200 as tw, oracle
        from tests.test_nvls_gpu import make_comm, run_nvls, check_case, bf16_inputs
        orc = oracle.Oracle()
        for W, T, H in ((2, 33, 1024), (8, 128, 8192), (4, 7, 64)):
            comm = make_comm(W, T * H * 2)
            for it in range(3):
                inputs, residual, weight = bf16_inputs(it + W, W, T, H)
                ranges = tw.token_shard_map(T, W)
                outs, res, g = run_nvls(comm, inputs, residual, weight, torch.bfloat16, ranges, gather=bool(it & 1),
                                        sm_budget=4)
                check_case(orc, inputs, residual, weight, ranges, torch.bfloat16, outs, res, g)
            comm.close()
        print("OK")
    """)
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, **env))
    assert p.returncode == 0 and "OK" in p.stdout, p.stdout[-2000:] + p.stderr[-3000:]


def test_nvls_sim_barrier_timeout(cuda, monkeypatch):
    """A rank that never arrives: the bounded spin raises the timeout flag and
    tw_comm_check reports BarrierTimeout (no GPU hang); a fresh communicator
    is healthy."""
    import torch
    import paper_2505_11329_b200 as tw
    W, T, H = 4, 64, 256
    comm = make_comm(W, T * H * 2)
    shards = [torch.zeros(T // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    w = [torch.ones(H, device="cuda")] * W
    comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=2)
    torch.cuda.synchronize()
    comm.check()
    monkeypatch.setenv("TW_FAULT_DROP_ARRIVAL_RANK", "1")
    monkeypatch.setenv("TW_BARRIER_SPIN_LIMIT", "20000")
    comm.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=2)
    torch.cuda.synchronize()
    with pytest.raises(tw.BarrierTimeout):
        comm.check()
    comm.close()
    monkeypatch.delenv("TW_FAULT_DROP_ARRIVAL_RANK")
    monkeypatch.delenv("TW_BARRIER_SPIN_LIMIT")
    fresh = make_comm(W, T * H * 2)
    fresh.fused_allreduce_rmsnorm(T, H, shards, w, sm_budget=2)
    torch.cuda.synchronize()
    fresh.check()
    fresh.close()


def test_nvls_sim_unsupported_shapes(cuda):
    """The NVLS kernels need 16-byte vectors (H % 8 bf16 / H % 4 fp32) like the
    hardware path; the transport is for co-located ranks only."""
    import torch
    import paper_2505_11329_b200 as tw
    W, T, H = 2, 4, 12
    comm = make_comm(W, T * H * 2)
    shards = [torch.zeros(2, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    with pytest.raises(tw.Unsupported):
        comm.fused_allreduce_rmsnorm(T, H, shards, [torch.ones(H, device="cuda")] * W)
    comm.close()
    if torch.cuda.device_count() < 2:
        with pytest.raises(tw.TwError):
            tw.Communicator(2, [0, 1], 1024, tw.TW_TRANSPORT_NVLS_SIM)


def test_nvls_sim_k3_allreduce(cuda, orc):
    """K3 over the NVLS kernels: SPEC.md:104-105 known answers and the oracle."""
    import torch
    for dt in (torch.float32, torch.bfloat16):
        comm = make_comm(4, 3 * 8 * 4)
        for q in range(4):
            comm.buffer(q, 0, (3, 8), dt).fill_(float(q))
        comm.allreduce(3, 8, dt)
        torch.cuda.synchronize()
        assert all(torch.all(comm.buffer(q, 1, (3, 8), dt) == 6.0) for q in range(4))
        comm.close()
    W, T, H = 8, 100, 1024
    inputs, _, _ = group_inputs(3, W, T, H)
    comm = make_comm(W, T * H * 4)
    for r in range(W):
        comm.buffer(r, 0, (T, H), torch.float32).copy_(torch.from_numpy(inputs[r]))
    comm.allreduce(T, H, torch.float32, sm_budget=4)
    torch.cuda.synchronize()
    want = orc.all_reduce(list(inputs))
    for r in range(W):
        assert np.array_equal(comm.buffer(r, 1, (T, H), torch.float32).cpu().numpy(), want)
    comm.close()


@pytest.mark.parametrize("T", [1024, 8192])
def test_nvls_sim_c2_full_size(cuda, orc, T):
    """C2 (Llama-3.3-70B boundary: N = 8, H = 8192, bf16, G = 2) at full size:
    r' bitwise against the NVLS rounding model over all rows, the output is the
    RMSNorm of the gathered r' (size-independent), and a row sample matches
    the oracle."""
    import torch
    import paper_2505_11329_b200 as tw
    W, H = 8, 8192
    comm = make_comm(W, T * H * 2)
    g = torch.Generator(device="cuda").manual_seed(T)
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
    acc = torch.zeros(T, H, device="cuda")
    for p in parts:
        acc = acc + p.float()
    want_res = (acc.to(torch.bfloat16).float() + res_full.float()).to(torch.bfloat16)
    assert torch.equal(torch.cat(shards), want_res)
    rb = want_res.float()
    want = rb * torch.rsqrt((rb * rb).mean(1, keepdim=True) + 1e-5) * w
    for r in range(W):
        out = comm.buffer(r, 1, (T, H), torch.bfloat16).float()
        rel = ((out - want).abs() / torch.maximum(want.abs(), want.pow(2).mean(1, keepdim=True).sqrt())).max()
        assert rel.item() <= 2e-2
        assert torch.equal(comm.buffer(r, 2, (T, H), torch.bfloat16), want_res)
    rows = list(range(0, T, 257))
    ins = np.stack([p[rows].float().cpu().numpy() for p in parts])
    res_rows = res_full[rows].float().cpu().numpy()
    sub = orc.token_shard_map(len(rows), W)
    o, new = orc.fused_allreduce_rmsnorm(list(ins), [res_rows[b:e] for b, e in sub], w.cpu().numpy(), sub)
    assert_bf16_close(np.concatenate(new), want_res[rows].float().cpu().numpy(), what="r' vs oracle")
    assert_bf16_close(comm.buffer(0, 1, (T, H), torch.bfloat16)[rows].float().cpu().numpy(), o)
    comm.close()


# ---- NVLS hardware: >= 2 NVSwitch-attached GPUs ---------------------------------------------------

def _nvls_world_sizes():
    try:
        import torch
        n = torch.cuda.device_count()
    except Exception:
        return []
    return [w for w in (2, 4, 8) if w <= n]


def _require_nvls(n):
    import paper_2505_11329_b200 as tw
    try:
        comm = tw.Communicator(n, list(range(n)), 1 << 21, tw.TW_TRANSPORT_NVLS)
    except tw.Unsupported as exc:
        pytest.skip(f"NVLS unavailable on this box: {exc}")
    comm.close()


multi_gpu = pytest.mark.skipif("__import__('torch').cuda.device_count() < 2",
                               reason="NVLS needs >= 2 NVSwitch-attached GPUs (these run automatically when visible)")


@multi_gpu
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("T", [1024, 2048, 4096, 8192])
@pytest.mark.parametrize("G", [1, 2])
def test_nvls_hw_c2_bf16(cuda, orc, world, T, G):
    """C2/C3 shapes on real NVLS: r' and the output within 2e-2 of the oracle
    (sampled rows) and the output equal to the RMSNorm of the gathered r'
    (all rows); replicated outputs identical on every rank."""
    import torch
    import paper_2505_11329_b200 as tw
    if world > torch.cuda.device_count():
        pytest.skip(f"{world} GPUs not visible")
    _require_nvls(world)
    H = 8192
    comm = make_comm(world, T * H * 2, tw.TW_TRANSPORT_NVLS)
    ranges = tw.token_shard_map(T, world)
    g = torch.Generator().manual_seed(T + world)
    parts = [(torch.rand(T, H, generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(world)]
    res_full = (torch.rand(T, H, generator=g) * 2 - 1).to(torch.bfloat16)
    w = torch.rand(H, generator=g) + 0.5
    for r in range(world):
        comm.buffer(r, 0, (T, H), torch.bfloat16).copy_(parts[r].to(f"cuda:{r}"))
    shards = [res_full[b:e].to(f"cuda:{r}") for r, (b, e) in enumerate(ranges)]
    comm.fused_allreduce_rmsnorm(T, H, shards, [w.to(f"cuda:{r}") for r in range(world)], sm_budget=8,
                                 gather_residual=G == 2, streams=[torch.cuda.current_stream(r) for r in range(world)])
    for r in range(world):
        torch.cuda.synchronize(r)
    comm.check()
    got_res = torch.cat([s.cpu() for s in shards]).float()
    summed = sum(p.float() for p in parts)
    want_res = summed + res_full.float()
    rms = want_res.pow(2).mean(1, keepdim=True).sqrt()
    assert ((got_res - want_res).abs() <= 2e-2 * torch.maximum(want_res.abs(), rms)).all()
    want = got_res * torch.rsqrt((got_res * got_res).mean(1, keepdim=True) + 1e-5) * w
    out0 = comm.buffer(0, 1, (T, H), torch.bfloat16).cpu()
    for r in range(world):
        out = comm.buffer(r, 1, (T, H), torch.bfloat16).cpu()
        assert torch.equal(out, out0)
        if G == 2:
            assert torch.equal(comm.buffer(r, 2, (T, H), torch.bfloat16).cpu().float(), got_res)
    wr = want.pow(2).mean(1, keepdim=True).sqrt()
    assert ((out0.float() - want).abs() <= 2e-2 * torch.maximum(want.abs(), wr)).all()
    rows = list(range(0, T, 509))
    ins = np.stack([p[rows].float().numpy() for p in parts])
    sub = orc.token_shard_map(len(rows), world)
    o, _ = orc.fused_allreduce_rmsnorm(list(ins), [res_full[rows].float().numpy()[b:e] for b, e in sub],
                                       w.numpy(), sub)
    assert_bf16_close(out0[rows].float().numpy(), o)
    comm.close()


@multi_gpu
@pytest.mark.parametrize("dtype_name", ["float32", "bfloat16"])
@pytest.mark.parametrize("depth", [1, 2, 3])
def test_nvls_hw_parity_small(cuda, orc, dtype_name, depth):
    """Acceptance-grid style shapes on every visible GPU (fp32 <= 1e-5)."""
    import torch
    import paper_2505_11329_b200 as tw
    n = _nvls_world_sizes()[-1]
    _require_nvls(n)
    dtype = getattr(torch, dtype_name)
    for T, H in [(1, 16), (3, 64), (17, 1024), (257, 8192), (64, 6144)]:
        gen = bf16_inputs if dtype == torch.bfloat16 else group_inputs
        inputs, residual, weight = gen(T + H + depth, n, T, H)
        ranges = tw.token_shard_map(T, n)
        comm = make_comm(n, T * H * 4, tw.TW_TRANSPORT_NVLS)
        outs, res, g = run_nvls(comm, inputs, residual, weight, dtype, ranges, gather=True, sm_budget=8,
                                depth=depth, reps=2)
        comm.close()
        check_case(orc, inputs, residual, weight, ranges, dtype, outs, res, g, exact_sum=False)


@multi_gpu
def test_nvls_hw_repeated_and_graph(cuda, orc):
    """Many launches with changing budgets, then graph replay, on real NVLS."""
    import torch
    import paper_2505_11329_b200 as tw
    n = _nvls_world_sizes()[-1]
    _require_nvls(n)
    H = 1024
    comm = make_comm(n, 300 * H * 2, tw.TW_TRANSPORT_NVLS)
    for it, (T, budget) in enumerate([(1, 1), (256, 2), (17, 4), (300, 8), (64, 16), (5, 3)] * 2):
        inputs, residual, weight = bf16_inputs(it, n, T, H)
        ranges = tw.token_shard_map(T, n)
        outs, res, g = run_nvls(comm, inputs, residual, weight, torch.bfloat16, ranges, gather=bool(it & 1),
                                sm_budget=budget)
        check_case(orc, inputs, residual, weight, ranges, torch.bfloat16, outs, res, g, exact_sum=False)
    T = 128
    ranges = tw.token_shard_map(T, n)
    shards = [torch.zeros(e - b, H, device=f"cuda:{r}", dtype=torch.bfloat16) for r, (b, e) in enumerate(ranges)]
    ws = [torch.ones(H, device=f"cuda:{r}") for r in range(n)]
    streams = [torch.cuda.Stream(device=r) for r in range(n)]
    comm.fused_allreduce_rmsnorm(T, H, shards, ws, sm_budget=4, streams=streams)
    for r in range(n):
        torch.cuda.synchronize(r)
    # one graph per device: the _group call launches every rank on its own
    # stream, so every stream is put under capture around one call
    graphs = [torch.cuda.CUDAGraph() for _ in range(n)]
    ctxs = [torch.cuda.graph(graphs[r], stream=streams[r], capture_error_mode="thread_local") for r in range(n)]
    # capture: enter every device's capture, launch the group once, exit
    for c in ctxs:
        c.__enter__()
    try:
        comm.fused_allreduce_rmsnorm(T, H, shards, ws, sm_budget=4, streams=streams)
    finally:
        for c in reversed(ctxs):
            c.__exit__(None, None, None)
    for it in range(4):
        inputs, residual, _ = bf16_inputs(50 + it, n, T, H)
        for r in range(n):
            comm.buffer(r, 0, (T, H), torch.bfloat16).copy_(torch.from_numpy(inputs[r]).bfloat16())
        for r, (b, e) in enumerate(ranges):
            shards[r].copy_(torch.from_numpy(residual[b:e]).bfloat16())
        for r in range(n):
            torch.cuda.synchronize(r)
        for gr in graphs:
            gr.replay()
        for r in range(n):
            torch.cuda.synchronize(r)
        comm.check()
        outs = [comm.buffer(r, 1, (T, H), torch.bfloat16).float().cpu().numpy() for r in range(n)]
        check_case(orc, inputs, residual, np.ones(H, np.float32), ranges, torch.bfloat16, outs,
                   [s.float().cpu().numpy() for s in shards], None, exact_sum=False)
    comm.close()


@multi_gpu
def test_nvls_hw_barrier_timeout(cuda, monkeypatch):
    import torch
    import paper_2505_11329_b200 as tw
    n = _nvls_world_sizes()[-1]
    _require_nvls(n)
    T, H = 64, 256
    comm = make_comm(n, T * H * 2, tw.TW_TRANSPORT_NVLS)
    ranges = tw.token_shard_map(T, n)
    shards = [torch.zeros(e - b, H, device=f"cuda:{r}", dtype=torch.bfloat16) for r, (b, e) in enumerate(ranges)]
    ws = [torch.ones(H, device=f"cuda:{r}") for r in range(n)]
    monkeypatch.setenv("TW_FAULT_DROP_ARRIVAL_RANK", "1")
    monkeypatch.setenv("TW_BARRIER_SPIN_LIMIT", "20000")
    comm.fused_allreduce_rmsnorm(T, H, shards, ws, sm_budget=2,
                                 streams=[torch.cuda.current_stream(r) for r in range(n)])
    for r in range(n):
        torch.cuda.synchronize(r)
    with pytest.raises(tw.BarrierTimeout):
        comm.check()
    comm.close()


MP_WORKER = textwrap.dedent("""
    import ctypes, json, sys
    sys.path.insert(0, {root!r})
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2505_11329_b200 as tw
    from paper_2505_11329_b200 import _lib
    from tools.bench_tp import rendezvous_id
    from tests.helpers import group_inputs, bf16_round
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    T, H = {T}, {H}
    torch.cuda.set_device(rank)
    rid = rendezvous_id(dist)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib.tw_comm_create_mp(world, rank, rank, T * H * 2, rid.encode(), _lib.TW_TRANSPORT_NVLS,
                                          ctypes.byref(h)))
    inputs, residual, weight = group_inputs(7, world, T, H)
    inputs, residual = bf16_round(inputs), bf16_round(residual)
    p = ctypes.c_void_p()
    _lib.check(_lib.lib.tw_comm_buffer(h, rank, _lib.TW_BUF_INPUT, ctypes.byref(p)))
    buf = torch.as_tensor(tw._DevBuf(p.value, (T * H,), "<i2"), device="cuda").view(torch.bfloat16).view(T, H)
    buf.copy_(torch.from_numpy(inputs[rank]).bfloat16())
    ranges = tw.token_shard_map(T, world)
    b, e = ranges[rank]
    shard = torch.from_numpy(np.ascontiguousarray(residual[b:e])).cuda().bfloat16()
    wt = torch.from_numpy(weight).cuda()
    flat = (ctypes.c_int64 * (2 * world))(*[v for rg in ranges for v in rg])
    for _ in range(3):
        shard.copy_(torch.from_numpy(np.ascontiguousarray(residual[b:e])).bfloat16())
        torch.cuda.synchronize()
        dist.barrier()
        _lib.check(_lib.lib.tw_fused_allreduce_rmsnorm(h, T, H, 0, flat, shard.data_ptr(), wt.data_ptr(), 1e-5,
                                                       _lib.TW_BF16, 8, _lib.TW_GATHER_RESIDUAL, None))
        torch.cuda.synchronize()
    _lib.check(_lib.lib.tw_comm_check(h))
    _lib.check(_lib.lib.tw_comm_buffer(h, rank, _lib.TW_BUF_OUTPUT, ctypes.byref(p)))
    out = torch.as_tensor(tw._DevBuf(p.value, (T * H,), "<i2"), device="cuda").view(torch.bfloat16).view(T, H)
    np.save({outdir!r} + f"/out{{rank}}.npy", out.float().cpu().numpy())
    np.save({outdir!r} + f"/res{{rank}}.npy", shard.float().cpu().numpy())
    print(json.dumps({{"rank": rank, "ok": True}}), flush=True)
    dist.barrier()
    _lib.lib.tw_comm_destroy(h)
    dist.destroy_process_group()
""")


@multi_gpu
def test_nvls_hw_multi_process(cuda, orc, tmp_path):
    """One process per GPU (torchrun style): rank 0 creates the multicast
    object and shares it by POSIX fd; every rank runs K1 over NVLS."""
    n = _nvls_world_sizes()[-1]
    _require_nvls(n)
    T, H = 300, 4096
    script = tmp_path / "w.py"
    script.write_text(MP_WORKER.format(root=ROOT, T=T, H=H, outdir=str(tmp_path)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for rank in range(n):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(n),
                   TW_BARRIER_SPIN_LIMIT=str(1 << 28))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=600)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
    inputs, residual, weight = group_inputs(7, n, T, H)
    inputs, residual = bf16_round(inputs), bf16_round(residual)
    ranges = orc.token_shard_map(T, n)
    want_out, want_res = orc.fused_allreduce_rmsnorm(list(inputs), [residual[b:e] for b, e in ranges], weight)
    for r in range(n):
        assert_bf16_close(np.load(tmp_path / f"out{r}.npy"), want_out)
        assert_bf16_close(np.load(tmp_path / f"res{r}.npy"), want_res[r], what="r'")
