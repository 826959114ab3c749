"""Request traces and chunked-prefill batch formation (§8f row 4).

The product (libweavesim_b200.so through tw_workload.h) against the reference
itself (oracle/_ref: proj/src/workloads.cpp compiled unmodified), the C
restatement (oracle/tw_oracle.c) and the committed golden batches; the
reference's own cases (proj/tests/test_workloads.cpp) restated.  Integer
work: every comparison is exact.
"""
import os
import random

import pytest

from paper_2505_11329_b200 import weave
from paper_2505_11329_b200._lib import ConfigError, ParseError


def _tuples(batches):
    return [(t, d, kv, [tuple(s) for s in sl]) for t, d, kv, sl in batches]


def test_golden_batches(golden, orc):
    meta, _ = golden
    assert len(meta["batches"]) >= 10
    for case in meta["batches"]:
        reqs = [tuple(r) for r in case["requests"]]
        want = _tuples(case["batches"])
        assert weave.form_batches(reqs, case["chunk_size"]) == want, case["name"]
        assert orc.form_batches(reqs, case["chunk_size"]) == want, case["name"]


def test_random_traces_match_reference(ref, orc):
    rng = random.Random(2505)
    for _ in range(300):
        n = rng.randint(0, 24)
        reqs = [(rng.randint(1, 600), rng.randint(0, 40), rng.choice([0.0, 0.0, 0.5, 1.0, 3.0])) for _ in range(n)]
        chunk = rng.choice([1, 2, 7, 64, 256, 1000, 5000])
        want = ref.form_batches(reqs, chunk)
        assert weave.form_batches(reqs, chunk) == want, (reqs, chunk)
        assert orc.form_batches(reqs, chunk) == want, (reqs, chunk)


def test_conservation():
    """test_workloads.cpp:56-70."""
    batches = weave.form_batches(weave.synth_trace(16, 1000, 37), 512)
    prefill = decode = 0
    for total, d, _, slices in batches:
        s = sum(x[2] for x in slices)
        assert total == s + d
        prefill += s
        decode += d
    assert prefill == 16 * 1000 and decode == 16 * 37


def test_budget_after_decode_priority():
    """test_workloads.cpp:72-80."""
    for total, d, _, slices in weave.form_batches(weave.synth_trace(8, 4096, 64), 1024):
        assert sum(x[2] for x in slices) <= 1024
        assert total <= 1024 + d


def test_fcfs_and_decode_only_tail():
    """test_workloads.cpp:82-98."""
    b = weave.form_batches(weave.synth_trace(4, 100, 5), 250)
    assert [s[0] for s in b[0][3]] == [0, 1, 2] and b[0][3][2][2] == 50 and b[0][1] == 0
    assert b[1][1] == 2
    assert b[-1][3] == []


def test_arrival_ties_stable():
    """test_workloads.cpp:100-106."""
    b = weave.form_batches([(100, 0, 2.0), (100, 0, 0.0), (100, 0, 2.0)], 100)
    assert [x[3][0][0] for x in b] == [1, 0, 2]


def test_kv_context():
    """test_workloads.cpp:108-119."""
    b = weave.form_batches(weave.synth_trace(1, 300, 3), 100)
    assert [x[2] for x in b] == [0, 100, 200, 300, 301, 302]


def test_bad_arguments():
    """test_workloads.cpp:121-125."""
    with pytest.raises(ConfigError):
        weave.form_batches([], 0)
    for args in ((0, 100, 10), (4, 0, 10), (4, 10, -1)):
        with pytest.raises(ConfigError):
            weave.synth_trace(*args)
    assert weave.form_batches([], 16) == []


def test_trace_round_trip(tmp_path):
    """test_workloads.cpp:14-26."""
    reqs = [(100, 10, 0.0), (2048, 128, 0.5), (1, 0, 1.25)]
    p = str(tmp_path / "t.jsonl")
    weave.save_trace(reqs, p)
    assert weave.load_trace(p) == reqs


def test_save_trace_text_matches_reference(golden, tmp_path):
    """save_trace writes the reference's bytes (nlohmann dump: sorted keys,
    arrival_s only when > 0, shortest round-trip floats)."""
    meta, _ = golden
    p = str(tmp_path / "t.jsonl")
    weave.save_trace([tuple(r) for r in meta["trace_text"]["requests"]], p)
    assert open(p).read() == meta["trace_text"]["text"]


BAD_TRACES = {
    "not json": 'not json',
    "missing output": '{"prompt_tokens": 10}',
    "zero prompt": '{"prompt_tokens": 0, "output_tokens": 2}',
    "negative output": '{"prompt_tokens": 3, "output_tokens": -1}',
    "negative arrival": '{"prompt_tokens": 3, "output_tokens": 1, "arrival_s": -0.5}',
    "array": '[1, 2, 3]',
    "trailing": '{"prompt_tokens": 3, "output_tokens": 1} x',
    "unterminated": '{"prompt_tokens": 3, "output_tokens": 1',
}


@pytest.mark.parametrize("name", sorted(BAD_TRACES))
def test_parse_errors_name_the_line(name, tmp_path, ref):
    """test_workloads.cpp:28-54: ParseError naming the offending line; the
    reference rejects the same files."""
    p = str(tmp_path / "bad.jsonl")
    with open(p, "w") as f:
        f.write('{"prompt_tokens": 10, "output_tokens": 2}\n\n' + BAD_TRACES[name] + "\n")
    with pytest.raises(ParseError, match="line 3"):
        weave.load_trace(p)
    import oracle
    with pytest.raises(oracle.StatusError):
        ref.load_trace(p)


def test_missing_trace_file():
    with pytest.raises(ParseError):
        weave.load_trace("/nonexistent/missing_trace.jsonl")


def test_load_accepts_what_reference_accepts(tmp_path, ref):
    lines = ['{"output_tokens": 5, "prompt_tokens": 7}',
             '  {"prompt_tokens": 1, "output_tokens": 0, "arrival_s": 2.5, "extra": [1, {"a": null}], "s": "x\\"y"}',
             '{"prompt_tokens": 4.9, "output_tokens": 2, "arrival_s": 1e-3}',
             '{"prompt_tokens": 12, "output_tokens": 3, "arrival_s": 0}']
    p = str(tmp_path / "ok.jsonl")
    with open(p, "w") as f:
        f.write("\n".join(lines) + "\n   \n")
    assert weave.load_trace(p) == ref.load_trace(p)
    # and the reference reads what the drop-in writes
    q = str(tmp_path / "rt.jsonl")
    reqs = [(9, 1, 0.0), (3, 3, 0.1), (5, 0, 7.0)]
    weave.save_trace(reqs, q)
    assert ref.load_trace(q) == reqs


def test_throughput_predictions_fixture(golden):
    """The reference's modeled throughput for the measured workloads
    (tools/throughput_bench.py prints it beside the measurement)."""
    meta, _ = golden
    for row in meta["throughput_pred"]:
        assert row["nocomm"]["tokens_per_sec"] >= row["multimem"]["tokens_per_sec"]
        reqs = [(p, o, 0.0) for p, o in row["requests"]]
        assert row["tokenweave"]["iterations"] == len(weave.form_batches(reqs, row["chunk_size"]))
        assert row["tokenweave"]["total_tokens"] == sum(p + o for p, o in row["requests"])


def test_cli_throughput_workloads_pinned(golden, ref):
    """The fixture's fixed-2048x128 / chatlike requests are the ones the
    reference CLI's `throughput` command simulates (proj/src/commands.cpp:
    432-480): the reference's own CSV, re-derived from the fixture rows."""
    meta, _ = golden
    csv = ref.cmd_throughput_csv("llama-70b", "b200", 2048, 42)
    assert csv == meta["cli_throughput_csv"]
    rows = {(ln.split(",")[0], ln.split(",")[1]): ln.split(",") for ln in csv.strip().splitlines()[1:]}
    for case in meta["throughput_pred"][:2]:
        for mode in ("default", "multimem", "nocomm", "fuseonly", "tokenweave"):
            got = case[mode]
            want = rows[(case["name"], mode)]
            assert f"{got['tokens_per_sec']:.2f}" == want[2] and got["iterations"] == int(want[3])


@pytest.mark.gpu
def test_measured_throughput_accounting():
    """test_workloads.cpp:127-139 on the measured runner: totals, iteration
    count = form_batches, per-iteration latencies sum to total_seconds."""
    reqs = weave.synth_trace(4, 512, 3)
    r = weave.LayerRunner("llama-70b", tp=8, max_tokens=2048)
    try:
        for mode in ("fuseonly", "tokenweave", "unfused", "nocomm"):
            res = r.throughput(reqs, 1024, mode, num_layers=2, layers_measured=1)
            assert res["total_tokens"] == 4 * (512 + 3)
            assert res["iterations"] == len(weave.form_batches(reqs, 1024)) == len(res["iteration_latencies"])
            assert abs(sum(res["iteration_latencies"]) - res["total_seconds"]) <= 1e-9 * res["total_seconds"] + 1e-12
            assert res["tokens_per_sec"] == pytest.approx(res["total_tokens"] / res["total_seconds"], rel=1e-12)
            assert all(x > 0 for x in res["iteration_latencies"])
    finally:
        r.close()


@pytest.mark.gpu
def test_prior_context_attention_costs_time():
    """A decode batch attending 256K cached tokens is slower than the same
    batch without context (the KV stream is real HBM traffic)."""
    r = weave.LayerRunner("llama-70b", tp=8, max_tokens=1024)
    try:
        base = min(r.run_batch(64, 0, "fuseonly", layers=4) for _ in range(3))
        ctx = min(r.run_batch(64, 262144, "fuseonly", layers=4) for _ in range(3))
        assert ctx > base, (base, ctx)
        # weave mode splits the context between the halves and still runs
        assert r.run_batch(1024, 65536, "tokenweave", prefix=512, layers=2) > 0
    finally:
        r.close()
