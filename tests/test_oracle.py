"""The oracle (C restatement) pinned against the reference and its golden
vectors.  CPU only."""
import numpy as np
import pytest

from tests.helpers import group_inputs, norm_inputs


def test_kat_single_token_worked_example(orc):
    # T=1, H=1: in 3, res 1, w 2, eps 0 -> out 2, res 4
    out, rout = orc.rmsnorm_residual(np.array([[3.0]]), np.array([[1.0]]), np.array([2.0]), eps=0.0)
    assert out[0, 0] == 2.0 and rout[0, 0] == 4.0


def test_kat_two_rank_ones(orc):
    # N=2, T=2, H=2, inputs ones, residual 0, w 1, eps 0 -> out 1, res 2
    inputs = [np.ones((2, 2), np.float32)] * 2
    ranges = orc.token_shard_map(2, 2)
    shards = [np.zeros((e - b, 2), np.float32) for b, e in ranges]
    out, new = orc.fused_allreduce_rmsnorm(inputs, shards, np.ones(2, np.float32), eps=0.0)
    assert np.all(out == 1.0)
    assert all(np.all(s == 2.0) for s in new)


def test_kat_shard_maps(orc):
    # SPEC.md:95-97
    assert orc.token_shard_map(8, 4) == [(0, 2), (2, 4), (4, 6), (6, 8)]
    assert orc.token_shard_map(10, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert orc.token_shard_map(3, 8) == [(0, 1), (1, 2), (2, 3)] + [(3, 3)] * 5


def test_kat_allreduce(orc):
    # SPEC.md:104-105
    assert np.all(orc.all_reduce([np.ones((3, 4), np.float32)] * 4) == 4.0)
    assert np.all(orc.all_reduce([np.full((3, 4), r, np.float32) for r in range(4)]) == 6.0)


def test_kat_zero_input_zero_output(orc):
    # proj/tests/test_numerics.cpp:91-98
    z = np.zeros((3, 8), np.float32)
    out, _ = orc.rmsnorm_residual(z, z, np.ones(8, np.float32))
    assert np.all(out == 0.0)


def test_shard_map_balance_and_errors(orc):
    # proj/tests/test_collectives.cpp:40-70
    for T in (0, 1, 7, 8, 100, 1023):
        for W in (2, 3, 4, 8):
            m = orc.token_shard_map(T, W)
            assert orc.shard_map_validate(m, T) == 0
            assert all(T // W <= e - b <= T // W + 1 for b, e in m)
    m = orc.token_shard_map(16, 4)
    assert orc.shard_map_validate(m, 17) == 4
    bad = [list(r) for r in m]
    bad[2][0] -= 1
    assert orc.shard_map_validate(bad, 16) == 4
    bad = [list(r) for r in m]
    bad[1][0] += 1
    assert orc.shard_map_validate(bad, 16) == 4
    with pytest.raises(Exception):
        orc.token_shard_map(16, 1)


def test_oracle_matches_golden_fused(orc, golden):
    meta, arrays = golden
    for case in meta["fused"]:
        inputs, residual, weight = group_inputs(case["seed"], case["world"], case["T"], case["H"])
        ranges = [tuple(r) for r in case["ranges"]]
        assert orc.token_shard_map(case["T"], case["world"]) == ranges
        shards = [residual[b:e] for b, e in ranges]
        out, new = orc.fused_allreduce_rmsnorm(list(inputs), shards, weight)
        i = case["id"]
        # bit-exact: same fp32 operation order as proj/src/collectives.cpp:134-153
        assert np.array_equal(out.view(np.uint32), arrays[f"fused_{i}_out"].view(np.uint32)), case
        assert np.array_equal(np.concatenate(new), arrays[f"fused_{i}_res"]), case
        assert np.array_equal(orc.all_reduce(list(inputs)), arrays[f"fused_{i}_ar"]), case


def test_oracle_matches_golden_norm(orc, golden):
    meta, arrays = golden
    for case in meta["norm"]:
        inp, res, w = norm_inputs(case["seed"], case["T"], case["H"])
        out, rout = orc.rmsnorm_residual(inp, res, w)
        assert np.array_equal(out, arrays[f"norm_{case['id']}_out"])
        assert np.array_equal(rout, arrays[f"norm_{case['id']}_res"])


def test_oracle_matches_golden_plans(orc, golden):
    meta, _ = golden
    for p in meta["plans"]:
        got = orc.make_split_plan(p["T"], p["threshold"], p["num_sms"], p["tile_tokens"], p["cta_columns"])
        assert got == (p["prefix"], p["suffix"], p["offset"], p["mode"]), p


def test_appendix_a_plans(golden):
    # SURVEY.md Appendix A (probed from the reference)
    meta, _ = golden
    plans = {(p["profile"], p["model"], p["T"]): (p["prefix"], p["suffix"], p["offset"], p["mode"])
             for p in meta["plans"]}
    assert plans[("b200", "llama-70b", 4096)] == (1152, 2944, -896, 2)
    assert plans[("b200", "llama-70b", 6144)] == (2944, 3200, -128, 2)
    assert plans[("b200", "llama-70b", 8192)] == (4096, 4096, 0, 2)
    assert plans[("b200", "llama-70b", 512)] == (512, 0, 0, 1)
    assert plans[("b200", "mixtral-8x22b", 2048)] == (2048, 0, 0, 1)


def test_worked_example_300_ctas(orc):
    # proj/tests/acceptance.cpp:90-105 (tile 128, 4 columns, 132 SMs, T=9600)
    T = 9600
    prefix = T // 2 + orc.smart_offset_analytic(T, 132, 128, 4)
    wc = orc.L.orc_wave_count
    cc = orc.L.orc_cta_count
    assert wc(cc(T, 128, 4), 132) == 3
    assert wc(cc(prefix, 128, 4), 132) + wc(cc(T - prefix, 128, 4), 132) == 3
    assert cc(prefix, 128, 4) == 132


def test_sequence_boundaries(orc):
    # proj/tests/test_splitter.cpp:128-150
    assert orc.place_sequence_boundaries([30, 40, 30], 100, 55) == [30, 25, 0]


def test_oracle_matches_reference_acceptance_draws(orc, ref):
    """Restatement == reference on the acceptance generator (mt19937_64 draws,
    proj/tests/acceptance.cpp:41-66), a slice of its N x T x H x seed grid."""
    for world in (2, 4, 8):
        for T in (1, 3, 17, 256):
            for H in (16, 64, 1024):
                for i in range(2):
                    inputs, residual, weight = ref.fill_group(ref.acceptance_seed(world, T, H, i), world, T, H)
                    ranges = orc.token_shard_map(T, world)
                    shards = [residual[b:e] for b, e in ranges]
                    o1, s1 = orc.fused_allreduce_rmsnorm(list(inputs), shards, weight)
                    o2, s2 = ref.fused_allreduce_rmsnorm(list(inputs), shards, weight)
                    assert np.array_equal(o1.view(np.uint32), o2.view(np.uint32))
                    assert all(np.array_equal(a, b) for a, b in zip(s1, s2))


def test_oracle_matches_reference_split_planner(orc, ref):
    for T in list(range(0, 20000, 97)) + [4096, 6144, 9600]:
        for sms, tile, cols in ((148, 128, 32), (132, 128, 32), (132, 128, 4)):
            assert orc.smart_offset_analytic(T, sms, tile, cols) == ref.smart_offset_analytic(T, sms, tile, cols)


def test_measured_calibration_table_feeds_reference_calibrate(ref):
    """profiles/microbench_b200_measured.json parses with the
    reference's CalibrationTable reader and calibrates: the measured K2 series
    gives a smaller RMSNorm intercept and a higher effective HBM bandwidth
    than the paper's table."""
    import os
    from tests.conftest import ROOT
    path = os.path.join(ROOT, "profiles", "microbench_b200_measured.json")
    if not os.path.exists(path):
        pytest.skip("no measured table committed")
    ours = ref.calibrate_file(path)
    paper = ref.calibrate_file("/root/reference/proj/data/microbench_b200.json") if os.path.exists(
        "/root/reference/proj/data/microbench_b200.json") else None
    assert ours["rmsnorm_slope_us_per_token"] > 0 and ours["hbm_bandwidth_effective"] > 0
    if paper:
        assert ours["rmsnorm_intercept_us"] < paper["rmsnorm_intercept_us"]
        assert ours["hbm_bandwidth_effective"] > paper["hbm_bandwidth_effective"]


def test_oracle_error_codes_match_reference(orc, ref):
    x = np.ones((2, 4), np.float32)
    w = np.ones(4, np.float32)
    bad = x.copy()
    bad[1, 2] = np.nan
    from oracle import StatusError
    for lib in (orc, ref):
        with pytest.raises(StatusError) as e:
            lib.rmsnorm_residual(bad, x, w)
        assert e.value.code == 2
        with pytest.raises(StatusError) as e:
            lib.rmsnorm_residual(x, x, w, eps=-1.0)
        assert e.value.code == 2
