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
    for model in ("llama-70b", "mixtral-8x22b"):
        for t in (1024, 2048, 4096, 8192):
            row = {"model": model, "T": t}
            for mode in ("multimem", "fuseonly", "tokenweave", "nocomm"):
                row[mode] = ref.layer_latency("b200", model, t, mode)
            meta["layer_latency_s"].append(row)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(f"wrote {len(arrays)} arrays, {len(meta['plans'])} plans")


if __name__ == "__main__":
    main()
