"""Generate tests/golden/ fixtures from the reference itself (oracle/_ref).

Run here (needs /root/reference to build oracle/_ref):
    make ref && python tests/golden/make_golden.py

Inputs are drawn with numpy's PCG64 (portable) from the recorded seed, so only
the reference's OUTPUTS are stored.  The fixtures pin the C restatement
(oracle/tw_oracle.c) on hosts where the reference sources are absent.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402  (test infrastructure)


def group_inputs(seed: int, world: int, T: int, H: int):
    """Portable draw: rank inputs U(-1,1), residual U(-1,1), weight U(0.5,1.5)
    -- the distributions of proj/tests/acceptance.cpp:59-66."""
    rng = np.random.default_rng(seed)
    inputs = rng.uniform(-1.0, 1.0, (world, T, H)).astype(np.float32)
    residual = rng.uniform(-1.0, 1.0, (T, H)).astype(np.float32)
    weight = rng.uniform(0.5, 1.5, (H,)).astype(np.float32)
    return inputs, residual, weight


def norm_inputs(seed: int, T: int, H: int):
    """proj/tests/test_numerics.cpp:14-19,62-72: inputs U(-2,2), weight U(0.5,1.5)."""
    rng = np.random.default_rng(seed)
    inp = rng.uniform(-2.0, 2.0, (T, H)).astype(np.float32)
    res = rng.uniform(-2.0, 2.0, (T, H)).astype(np.float32)
    weight = rng.uniform(0.5, 1.5, (H,)).astype(np.float32)
    return inp, res, weight


FUSED_CASES = [(w, t, h) for w in (2, 4, 8) for t in (1, 3, 17, 40) for h in (16, 24, 33, 64)]
NORM_CASES = [(1, 8), (5, 16), (17, 33), (64, 128)]
PLAN_CASES = [("b200", "llama-70b", t) for t in (256, 512, 1024, 2048, 4096, 6144, 8192, 16384)] + \
             [("b200", "mixtral-8x22b", t) for t in (1024, 2048, 4096, 8192)] + \
             [("h100", "llama-70b", t) for t in (1024, 2048, 4096, 8192, 16384)]



def synth(count, prompt, output):
    """synth_trace (proj/src/workloads.cpp:56-66) as (prompt, output, arrival) tuples."""
    return [(prompt, output, 0.0)] * count


def mixed_trace(seed: int, n: int, max_prompt: int, max_output: int):
    """Portable mixed-length trace with arrival-time ties (numpy PCG64)."""
    rng = np.random.default_rng(seed)
    return [(int(rng.integers(1, max_prompt + 1)), int(rng.integers(0, max_output + 1)),
             float(rng.choice([0.0, 0.25, 0.5, 1.0]))) for _ in range(n)]


# form_batches cases: proj/tests/test_workloads.cpp:56-132 plus mixed traces.
BATCH_CASES = [
    ("conservation", synth(16, 1000, 37), 512),        # test_workloads.cpp:56-70
    ("budget", synth(8, 4096, 64), 1024),               # :72-80
    ("fcfs", synth(4, 100, 5), 250),                    # :82-98
    ("arrival_ties", [(100, 0, 2.0), (100, 0, 0.0), (100, 0, 2.0)], 100),  # :100-106
    ("kv_context", synth(1, 300, 3), 100),              # :108-119
    ("decode_over_budget", synth(12, 50, 40), 8),
    ("no_output", [(7, 0, 0.0), (3, 0, 0.0)], 4),
    ("empty", [], 16),
    ("mixed_a", mixed_trace(11, 40, 3000, 200), 2048),
    ("mixed_b", mixed_trace(12, 64, 700, 50), 333),
    ("mixed_c", mixed_trace(13, 25, 9000, 16), 8192),
]

# Serving workloads of tools/throughput_bench.py: (name, model, requests, chunk).
# The first two are the reference CLI's own `throughput` defaults
# (proj/src/commands.cpp:432-446: synth_trace(64, 2048, 128) and
# chatlike_trace(96, seed 42), chunk 2048 = RunConfig's default); chatlike
# requests come from the reference (restated in oracle/ref_capi.cpp, pinned
# against the CLI's CSV), so they are stored in the fixture.
def throughput_cases(ref):
    chat = ref.chatlike_trace(96, 42)
    return [
        ("fixed-2048x128", "llama-70b", synth(64, 2048, 128), 2048),
        ("chatlike", "llama-70b", chat, 2048),
        ("fixed-2048x128-chunk8192", "llama-70b", synth(64, 2048, 128), 8192),
        ("mixtral-fixed-2048x128-chunk8192", "mixtral-8x22b", synth(64, 2048, 128), 8192),
    ]


def main() -> None:
    ref = oracle.RefLib()
    arrays = {}
    meta = {"fused": [], "norm": [], "plans": [], "layer_latency_s": []}
    for i, (w, t, h) in enumerate(FUSED_CASES):
        seed = 1000 + i
        inputs, residual, weight = group_inputs(seed, w, t, h)
        ranges = ref.token_shard_map(t, w)
        shards = [residual[b:e] for b, e in ranges]
        out, new_shards = ref.fused_allreduce_rmsnorm(list(inputs), shards, weight)
        out_p, shards_p = ref.fused_allreduce_rmsnorm(list(inputs), shards, weight, parallel=True)
        assert np.array_equal(out, out_p) and all(np.array_equal(a, b) for a, b in zip(new_shards, shards_p))
        arrays[f"fused_{i}_out"] = out
        arrays[f"fused_{i}_res"] = np.concatenate(new_shards, axis=0) if t else np.zeros((0, h), np.float32)
        arrays[f"fused_{i}_ar"] = ref.all_reduce(list(inputs))
        meta["fused"].append({"id": i, "seed": seed, "world": w, "T": t, "H": h, "ranges": ranges})
    for i, (t, h) in enumerate(NORM_CASES):
        seed = 7 + i
        inp, res, weight = norm_inputs(seed, t, h)
        out, rout = ref.rmsnorm_residual(inp, res, weight)
        arrays[f"norm_{i}_out"] = out
        arrays[f"norm_{i}_res"] = rout
        meta["norm"].append({"id": i, "seed": seed, "T": t, "H": h})
    for prof, model, t in PLAN_CASES:
        plan, geom = ref.make_split_plan(prof, model, t)
        meta["plans"].append({"profile": prof, "model": model, "T": t, "prefix": plan[0], "suffix": plan[1],
                              "offset": plan[2], "mode": plan[3], "num_sms": geom[0], "tile_tokens": geom[1],
                              "cta_columns": geom[2], "threshold": geom[3]})
    for model, toks in (("llama-70b", (1024, 2048, 4096, 8192)), ("mixtral-8x22b", (1024, 2048, 4096, 8192)),
                        ("qwen-72b", (256, 512, 1024, 2048, 4096, 8192, 16384))):
        for t in toks:
            row = {"model": model, "T": t}
            for mode in ("multimem", "fuseonly", "tokenweave", "nocomm"):
                row[mode] = ref.layer_latency("b200", model, t, mode)
            meta["layer_latency_s"].append(row)
    meta["batches"] = []
    for name, reqs, chunk in BATCH_CASES:
        meta["batches"].append({"name": name, "requests": [list(r) for r in reqs], "chunk_size": chunk,
                                "batches": [[t, d, kv, [list(x) for x in sl]]
                                            for t, d, kv, sl in ref.form_batches(reqs, chunk)]})
    # save_trace text of the reference (byte-exact drop-in check).
    import tempfile
    trace = [(100, 10, 0.0), (2048, 128, 0.5), (1, 0, 1.25), (5, 3, 1e-7), (9, 9, 3.0), (4, 1, 123456.789)]
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "t.jsonl")
        ref.save_trace(trace, path)
        meta["trace_text"] = {"requests": [list(r) for r in trace], "text": open(path).read()}
    meta["throughput_pred"] = []
    for name, model, reqs, chunk in throughput_cases(ref):
        row = {"name": name, "model": model, "chunk_size": chunk, "requests": [[p, o] for p, o, _ in reqs]}
        for mode in ("default", "multimem", "fuseonly", "tokenweave", "nocomm"):
            row[mode] = ref.simulate_throughput("b200", model, mode, reqs, chunk)
        meta["throughput_pred"].append(row)
    meta["cli_throughput_csv"] = ref.cmd_throughput_csv("llama-70b", "b200", 2048, 42)
    # Timeline JSON schema fixture (modeled values; the measured C++ timeline
    # must produce the same keys, vocabularies and DAG edges per layer)
    meta["timeline_json"] = {m: ref.timeline_json("b200", "llama-70b", 8192, m) for m in ("tokenweave", "fuseonly")}
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(f"wrote {len(arrays)} arrays, {len(meta['plans'])} plans")


if __name__ == "__main__":
    main()
