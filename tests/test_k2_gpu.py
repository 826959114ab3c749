"""K2 -- TP=1 fused residual-add + RMSNorm on the GPU vs the oracle
(weavesim::rmsnorm_residual, proj/src/numerics.cpp:30-64).

Tolerances (north_star): fp32 storage -- residual_out bitwise (same fp32 add),
output <= 1e-5 absolute; bf16 storage -- residual_out bitwise equal to the
RNE-rounded oracle r', output within 2e-2 relative (row-rms guarded)."""
import numpy as np
import pytest

from tests.helpers import assert_abs_close, assert_bf16_close, bf16_round, norm_inputs

pytestmark = pytest.mark.gpu


def run_k2(inp, res, w, dtype, eps=1e-5, sm_budget=0, inplace=False):
    import torch
    import paper_2505_11329_b200 as tw
    ti = torch.from_numpy(inp).to("cuda", dtype)
    tr = torch.from_numpy(res).to("cuda", dtype)
    tw_ = torch.from_numpy(w).to("cuda", torch.float32)
    out, rout = tw.rmsnorm_residual(ti, tr, tw_, eps, residual_out=tr if inplace else None, sm_budget=sm_budget)
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), rout.float().cpu().numpy()


@pytest.mark.parametrize("T,H", [(1, 8), (5, 16), (17, 33), (64, 128), (3, 1024), (33, 4096), (64, 8192),
                                 (7, 12), (9, 24), (2, 16384), (1000, 4096)])
def test_k2_fp32_matches_oracle(cuda, orc, T, H):
    inp, res, w = norm_inputs(11 + T * 7 + H, T, H)
    want_out, want_res = orc.rmsnorm_residual(inp, res, w)
    import torch
    out, rout = run_k2(inp, res, w, torch.float32)
    assert np.array_equal(rout, want_res), "r' must be the same fp32 add"
    assert_abs_close(out, want_out, 1e-5)


# (2048, 6144) and (1500, 8192): many rows per CTA, so the two-row-group TMA
# engine wraps its smem ring and alternates groups (the default below 48 rows/SM).
@pytest.mark.parametrize("T,H", [(1, 8), (5, 16), (17, 33), (64, 128), (64, 8192), (7, 24), (256, 8192),
                                 (4, 6144), (3, 16384), (2048, 6144), (1500, 8192)])
def test_k2_bf16_matches_oracle(cuda, orc, T, H):
    import torch
    inp, res, w = norm_inputs(5 + T + H, T, H)
    inp, res = bf16_round(inp), bf16_round(res)
    want_out, want_res = orc.rmsnorm_residual(inp, res, w)
    out, rout = run_k2(inp, res, w, torch.bfloat16)
    assert np.array_equal(rout, bf16_round(want_res)), "bf16 r' must be RNE(fp32 r')"
    assert_bf16_close(out, want_out)


def _bf16_rounding_edge_pairs(seed, T, H):
    """bf16 (x, r) pairs that stress r' = RNE(x + r): every exponent gap 0..24
    (the smaller operand's bits beyond, at and below bf16's half ulp), exact
    ties onto even and odd mantissas in both signs, cancellation to +-0,
    subnormals (down to 2^-133), and the normal/subnormal boundary."""
    rng = np.random.default_rng(seed)
    n = T * H
    sign = lambda: np.where(rng.random(n) < 0.5, -1.0, 1.0)  # noqa: E731
    mant = lambda: 1.0 + rng.integers(0, 128, n) / 128.0  # noqa: E731  (8 significant bits: exact in bf16)
    e1 = rng.integers(-20, 12, n)
    gap = rng.integers(0, 25, n)
    x = sign() * mant() * np.exp2(e1)
    r = sign() * mant() * np.exp2(e1 - gap)
    kind = rng.integers(0, 6, n)
    half_ulp = np.exp2(e1 - 8)  # x in [2^e1, 2^(e1+1)): bf16 ulp 2^(e1-7)
    r = np.where(kind == 1, np.sign(r) * half_ulp, r)  # exact ties (either sign)
    r = np.where(kind == 2, -x, r)  # cancellation
    sub = np.exp2(rng.integers(-133, -120, n).astype(np.float64)) * mant()
    x = np.where(kind == 3, sign() * sub, x)  # subnormal / boundary operands
    r = np.where(kind == 3, sign() * np.exp2(rng.integers(-133, -118, n).astype(np.float64)), r)
    r = np.where(kind == 4, sign() * half_ulp * 3, r)  # 1.5 ulp: rounds away from the tie
    x32 = bf16_round(x.astype(np.float32)).reshape(T, H)
    r32 = bf16_round(r.astype(np.float32)).reshape(T, H)
    return x32, r32


def test_k2_bf16_rounding_edges_matches_oracle(cuda, orc):
    """r' bitwise = RNE(fp32 x + r) on crafted tie / gap / subnormal pairs (the
    two-group engine forms r' with add.rn.bf16x2, the one-group engine with an
    fp32 add and an RNE pack; the every-engine test re-runs this per engine)."""
    import torch
    for T in (64, 1500):  # two row groups, and many rows per CTA
        x, r = _bf16_rounding_edge_pairs(91 + T, T, 8192)
        w = np.random.default_rng(T).uniform(0.5, 1.5, 8192).astype(np.float32)
        want_out, want_res = orc.rmsnorm_residual(x, r, w)
        out, rout = run_k2(x, r, w, torch.bfloat16)
        assert np.array_equal(rout.view(np.uint32), bf16_round(want_res).view(np.uint32)), \
            "bf16 r' must be RNE(fp32 x + r), signed zeros included"
        assert_bf16_close(out, want_out)


def test_k2_in_place_residual(cuda, orc):
    import torch
    inp, res, w = norm_inputs(3, 40, 8192)
    inp, res = bf16_round(inp), bf16_round(res)
    want_out, want_res = orc.rmsnorm_residual(inp, res, w)
    out, rout = run_k2(inp, res, w, torch.bfloat16, inplace=True)
    assert np.array_equal(rout, bf16_round(want_res))
    assert_bf16_close(out, want_out)


def test_k2_unaligned_pointers_take_the_scalar_path(cuda, orc):
    import torch
    import paper_2505_11329_b200 as tw
    T, H = 6, 64
    inp, res, w = norm_inputs(17, T, H)
    want_out, want_res = orc.rmsnorm_residual(inp, res, w)
    big_i = torch.zeros(T * H + 1, device="cuda")
    big_r = torch.zeros(T * H + 1, device="cuda")
    ti = big_i[1:].view(T, H)
    tr = big_r[1:].view(T, H)
    ti.copy_(torch.from_numpy(inp))
    tr.copy_(torch.from_numpy(res))
    out, rout = tw.rmsnorm_residual(ti, tr, torch.from_numpy(w).cuda())
    assert np.array_equal(rout.cpu().numpy(), want_res)
    assert_abs_close(out.cpu().numpy(), want_out, 1e-5)


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("T,H,chunk", [(100, 8192, 7), (1, 64, 0), (513, 4096, 64), (2048, 8192, 0), (37, 33, 5)])
def test_k2_host_buffers_pipeline(cuda, orc, T, H, chunk, pinned):
    """tw_rmsnorm_residual_host (chunked H2D | K2 | D2H) == the oracle."""
    import torch
    import paper_2505_11329_b200 as tw
    inp, res, w = norm_inputs(T + H + chunk, T, H)
    inp, res = bf16_round(inp), bf16_round(res)
    want_out, want_res = orc.rmsnorm_residual(inp, res, w)
    hi = torch.from_numpy(inp).bfloat16()
    hr = torch.from_numpy(res).bfloat16()
    if pinned:
        hi, hr = hi.pin_memory(), hr.pin_memory()
    out, rout = tw.rmsnorm_residual_host(hi, hr, torch.from_numpy(w), chunk_rows=chunk)
    torch.cuda.synchronize()
    assert np.array_equal(rout.float().numpy(), bf16_round(want_res))
    assert_bf16_close(out.float().numpy(), want_out)


def test_k2_host_pipeline_calls_on_different_streams(cuda, orc):
    """Back-to-back host-buffer calls on two caller streams share one device
    staging context: the second call's weight upload and staging slots wait
    for the first call's kernels and copies, so both results are
    right even though nothing orders the two caller streams."""
    import torch
    import paper_2505_11329_b200 as tw
    T, H = 3000, 8192
    outs = []
    cases = []
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for k in range(2):
        inp, res, w = norm_inputs(900 + k, T, H)
        inp, res = bf16_round(inp), bf16_round(res)
        w = w * (1.0 + k)  # different weights: a race on the shared weight buffer shows
        cases.append(orc.rmsnorm_residual(inp, res, w))
        hi = torch.from_numpy(inp).bfloat16().pin_memory()
        hr = torch.from_numpy(res).bfloat16().pin_memory()
        ho = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
        hro = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
        outs.append((ho, hro, hi, hr))
        tw.rmsnorm_residual_host(hi, hr, torch.from_numpy(w), residual_out=hro, out=ho, stream=streams[k])
    torch.cuda.synchronize()
    for k in range(2):
        want_out, want_res = cases[k]
        ho, hro = outs[k][0], outs[k][1]
        assert np.array_equal(hro.float().numpy(), bf16_round(want_res)), k
        assert_bf16_close(ho.float().numpy(), want_out, what=f"call {k}")


@pytest.mark.parametrize("dtype_name", ["float32", "bfloat16"])
@pytest.mark.parametrize("T,H", [(1, 64), (37, 33), (513, 4096), (1100, 8192), (4096, 8192)])
def test_k2_host_sync_pageable(cuda, orc, T, H, dtype_name):
    """tw_rmsnorm_residual_host_sync on PAGEABLE numpy memory (pinned-ring
    staging by host threads, chunks wrapping the ring several times) == the
    oracle: fp32 residual bitwise / output <= 1e-5, bf16 as elsewhere."""
    import ctypes
    import paper_2505_11329_b200 as tw
    from paper_2505_11329_b200 import _lib
    inp, res, w = norm_inputs(3 * T + H, T, H)
    bf = dtype_name == "bfloat16"
    if bf:
        inp, res = bf16_round(inp), bf16_round(res)
    want_out, want_res = orc.rmsnorm_residual(inp, res, w)
    if bf:
        hi = (inp.view(np.uint32) >> 16).astype(np.uint16)
        hr = (res.view(np.uint32) >> 16).astype(np.uint16)
        ho, hro = np.empty_like(hi), np.empty_like(hi)
    else:
        hi, hr = np.ascontiguousarray(inp), np.ascontiguousarray(res)
        ho, hro = np.empty_like(hi), np.empty_like(hi)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    tw.check(_lib.lib.tw_rmsnorm_residual_host_sync(p(hi), p(hr), p(hro), p(ho), p(w), T, H, 1e-5,
                                                   tw.TW_BF16 if bf else tw.TW_F32, _lib.TW_HOST_CHECK_FINITE))
    if bf:
        up = lambda a: (a.astype(np.uint32) << 16).view(np.float32)  # noqa: E731
        assert np.array_equal(up(hro), bf16_round(want_res))
        assert_bf16_close(up(ho), want_out)
    else:
        assert np.array_equal(hro, want_res)
        assert_abs_close(ho, want_out, 1e-5)
    # a NaN anywhere (here: the residual's last chunk) -> NumericError
    bad = hr.copy()
    bad.reshape(-1)[-1] = 0x7FC0 if bf else np.float32("nan")
    with pytest.raises(tw.NumericError):
        tw.check(_lib.lib.tw_rmsnorm_residual_host_sync(p(hi), p(bad), p(hro), p(ho), p(w), T, H, 1e-5,
                                                       tw.TW_BF16 if bf else tw.TW_F32, _lib.TW_HOST_CHECK_FINITE))
    # without the flag the call does not scan
    tw.check(_lib.lib.tw_rmsnorm_residual_host_sync(p(hi), p(hr), p(hro), p(ho), p(w), T, H, 1e-5,
                                                   tw.TW_BF16 if bf else tw.TW_F32, 0))


@pytest.mark.parametrize("dtype_name", ["float32", "bfloat16"])
@pytest.mark.parametrize("T,H", [(37, 33), (1100, 8192)])
def test_k2_host_sync_gated(cuda, orc, T, H, dtype_name):
    """tw_rmsnorm_residual_host_sync_gated: two row gates advanced by a host
    thread in small uneven steps (as the drop-in's fill threads do) -- the
    results land only behind the gates and equal the oracle's; gates already
    at T behave like the ungated call."""
    import ctypes
    import threading
    import time
    import paper_2505_11329_b200 as tw
    from paper_2505_11329_b200 import _lib
    inp, res, w = norm_inputs(5 * T + H, T, H)
    bf = dtype_name == "bfloat16"
    if bf:
        inp, res = bf16_round(inp), bf16_round(res)
        hi = (inp.view(np.uint32) >> 16).astype(np.uint16)
        hr = (res.view(np.uint32) >> 16).astype(np.uint16)
    else:
        hi, hr = np.ascontiguousarray(inp), np.ascontiguousarray(res)
    want_out, want_res = orc.rmsnorm_residual(inp, res, w)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    code = tw.TW_BF16 if bf else tw.TW_F32
    for threaded in (True, False):
        ho, hro = np.zeros_like(hi), np.zeros_like(hi)
        gates = (ctypes.c_int64 * 2)(0, 0) if threaded else (ctypes.c_int64 * 2)(T, T)
        seen = []

        def advance():
            for t in list(range(0, T, max(1, T // 7))) + [T]:
                seen.append(int(np.count_nonzero(hro.reshape(T, -1).any(axis=1))))  # rows written so far
                gates[0] = t
                time.sleep(0.002)
                gates[1] = t
                time.sleep(0.002)

        th = threading.Thread(target=advance) if threaded else None
        if th:
            th.start()
        tw.check(_lib.lib.tw_rmsnorm_residual_host_sync_gated(p(hi), p(hr), p(hro), p(ho), p(w), T, H, 1e-5, code,
                                                              _lib.TW_HOST_CHECK_FINITE, gates, 2))
        if th:
            th.join()
            steps = list(range(0, T, max(1, T // 7)))
            # before gate step k was published, no row at or beyond step k-1's value had been written
            for k, rows in enumerate(seen[1:], start=1):
                assert rows <= steps[k - 1] if k - 1 < len(steps) else True, (k, rows)
        if bf:
            up = lambda a: (a.astype(np.uint32) << 16).view(np.float32)  # noqa: E731
            assert np.array_equal(up(hro), bf16_round(want_res))
            assert_bf16_close(up(ho), want_out)
        else:
            assert np.array_equal(hro, want_res)
            assert_abs_close(ho, want_out, 1e-5)


@pytest.mark.parametrize("engine,pipeline,groups,lookahead",
                         [("rows", "1", "1", "0"), ("rows", "0", "1", "0"), ("bulk", "0", "1", "0"),
                          ("tma", "0", "1", "0"), ("tma", "0", "2", "0"), ("flat", "0", "1", "0"),
                          ("tma", "0", "1", "1"), ("tma", "0", "2", "2"), ("tma", "0", "2", "3"),
                          ("tma", "0", "1", "0/256"), ("tma", "0", "1", "0/512")])
def test_k2_every_engine_matches_oracle(cuda, engine, pipeline, groups, lookahead):
    """Every K2 engine (and the software-pipelined row loop that the NVLS K1
    path uses), the TMA engine's one- and two-group row math (scalar / packed
    bf16x2 + f32x2) and its load lookahead (rows in flight per SM) against the
    oracle: the parity tests above re-run in a subprocess with the knobs forced
    (they are read once per process)."""
    import os
    import subprocess
    import sys
    lookahead, _, tpr = lookahead.partition("/")  # "0/256": lookahead 0, 256 threads per row group
    env = dict(os.environ, TW_K2_ENGINE=engine, TW_ROWS_PIPELINE=pipeline, TW_K2_GROUPS=groups,
               TW_K2_LOOKAHEAD=lookahead)
    if tpr:
        env["TW_K2_TPR"] = tpr
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", __file__, "-k",
                        "matches_oracle and not every_engine or in_place or full_size or host_buffers "
                        "or sm_budget or under_budget"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert " passed" in p.stdout


def test_k2_known_answer_single_token(cuda):
    """T=1, H=1: in 3, res 1, w 2, eps 0 -> out 2, res 4 (exact)."""
    import torch
    import paper_2505_11329_b200 as tw
    for dt in (torch.float32, torch.bfloat16):
        x = torch.tensor([[3.0]], device="cuda", dtype=dt)
        r = torch.tensor([[1.0]], device="cuda", dtype=dt)
        out, rout = tw.rmsnorm_residual(x, r, torch.tensor([2.0], device="cuda"), eps=0.0)
        assert out.item() == 2.0 and rout.item() == 4.0


def test_k2_zero_input_normalizes_to_zero(cuda):
    import torch
    import paper_2505_11329_b200 as tw
    z = torch.zeros(3, 8, device="cuda")
    out, rout = tw.rmsnorm_residual(z, z, torch.ones(8, device="cuda"))
    assert torch.all(out == 0) and torch.all(rout == 0)


def test_k2_row_locality(cuda):
    """proj/tests/test_numerics.cpp:100-115: scaling one row leaves the others unchanged."""
    import torch
    import paper_2505_11329_b200 as tw
    x = torch.randn(4, 16, device="cuda")
    r = torch.zeros(4, 16, device="cuda")
    w = torch.ones(16, device="cuda")
    base, _ = tw.rmsnorm_residual(x, r, w)
    x2 = x.clone()
    x2[2] *= 8
    changed, _ = tw.rmsnorm_residual(x2, r, w)
    keep = [0, 1, 3]
    assert torch.equal(base[keep], changed[keep])


def test_k2_errors(cuda):
    import torch
    import paper_2505_11329_b200 as tw
    a = torch.zeros(2, 8, device="cuda")
    b = torch.zeros(3, 8, device="cuda")
    with pytest.raises(tw.DimensionError):
        tw.rmsnorm_residual(a, b, torch.ones(8, device="cuda"))
    with pytest.raises(tw.DimensionError):
        tw.rmsnorm_residual(a, a, torch.ones(7, device="cuda"))
    with pytest.raises(tw.NumericError):
        tw.rmsnorm_residual(a, a, torch.ones(8, device="cuda"), eps=-1.0)
    out, rout = tw.rmsnorm_residual(a[:0], a[:0], torch.ones(8, device="cuda"))
    assert out.shape == (0, 8)


def test_k2_sm_budget_does_not_change_results(cuda):
    import torch
    import paper_2505_11329_b200 as tw
    x = torch.randn(300, 8192, device="cuda", dtype=torch.bfloat16)
    r = torch.randn(300, 8192, device="cuda", dtype=torch.bfloat16)
    w = torch.rand(8192, device="cuda") + 0.5
    ref_out, ref_res = tw.rmsnorm_residual(x, r, w)
    for budget in (1, 2, 8, 16, 64, 65, 148):
        # r' is bitwise identical; the output may differ by the row-sum order
        # if an engine other than the default is chosen (one bf16 ulp at most)
        o, rr = tw.rmsnorm_residual(x, r, w, sm_budget=budget)
        assert torch.equal(rr, ref_res)
        assert (o.float() - ref_out.float()).abs().max().item() <= 2 ** -7 * ref_out.float().abs().max().item()


@pytest.mark.parametrize("H,dtype_name", [(10240, "float32"), (20480, "bfloat16")])
def test_k2_two_stage_ring_under_budget(cuda, orc, H, dtype_name):
    """40 KB rows leave room for a two-stage ring only: with a small SM budget
    each CTA walks many rows, and the row-group count must stay below the ring
    depth (a group frees its stage one row late)."""
    import torch
    T = 96
    inp, res, w = norm_inputs(5 + H, T, H)
    want_out, want_res = orc.rmsnorm_residual(bf16_round(inp), bf16_round(res), w) \
        if dtype_name == "bfloat16" else orc.rmsnorm_residual(inp, res, w)
    for budget in (2, 4):
        if dtype_name == "bfloat16":
            out, rout = run_k2(bf16_round(inp), bf16_round(res), w, torch.bfloat16, sm_budget=budget)
            assert np.array_equal(rout, bf16_round(want_res))
            assert_bf16_close(out, want_out)
        else:
            out, rout = run_k2(inp, res, w, torch.float32, sm_budget=budget)
            assert np.array_equal(rout, want_res)
            assert_abs_close(out, want_out, 1e-5)


def test_k2_full_size_vs_torch_fp32_and_sampled_oracle(cuda, orc):
    """Bench shape (8192 x 8192 bf16): torch fp32 restatement over every row,
    and the C oracle on a sample of rows."""
    import torch
    import paper_2505_11329_b200 as tw
    T, H = 8192, 8192
    g = torch.Generator(device="cuda").manual_seed(0)
    x = (torch.rand(T, H, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    r = (torch.rand(T, H, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w = torch.rand(H, device="cuda", generator=g) + 0.5
    out, rout = tw.rmsnorm_residual(x, r, w)
    rp = x.float() + r.float()
    assert torch.equal(rout, rp.to(torch.bfloat16))
    rb = rout.float()
    want = rb * torch.rsqrt((rb * rb).mean(dim=1, keepdim=True) + 1e-5) * w
    assert_bf16_close(out[::97].float().cpu().numpy(), want[::97].cpu().numpy())
    err = ((out.float() - want).abs() / torch.maximum(want.abs(), want.pow(2).mean(1, keepdim=True).sqrt())).max()
    assert err.item() <= 2e-2
    rows = torch.arange(0, T, 509, device="cuda")
    o2, r2 = orc.rmsnorm_residual(x[rows].float().cpu().numpy(), r[rows].float().cpu().numpy(), w.cpu().numpy())
    assert np.array_equal(rout[rows].float().cpu().numpy(), bf16_round(r2))
    assert_bf16_close(out[rows].float().cpu().numpy(), o2)
