"""The drop-in C++ API: the reference's own test cases (restated in
tests/cpp/test_dropin.cpp) compiled against libweavesim_b200.so."""
import os
import subprocess

import pytest

from tests.conftest import ROOT

BIN = os.path.join(ROOT, "build", "tests", "test_dropin")


def ensure_built():
    subprocess.run(["make", "-C", ROOT, "-s", "cpptests"], check=True, capture_output=True)
    assert os.path.exists(BIN)


def run(mode):
    ensure_built()
    p = subprocess.run([BIN, mode], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    return p.stdout


def test_dropin_host_cases():
    out = run("host")
    assert "0 failed" in out


@pytest.mark.gpu
def test_dropin_gpu_cases():
    out = run("gpu")
    assert "0 failed" in out
    print(out)


@pytest.mark.gpu
def test_dropin_acceptance_check1_full_grid():
    """proj/tests/acceptance.cpp check 1 on the drop-in: 2250 instances,
    fused vs unfused chain <= 1e-5, < 60 s."""
    out = run("acceptance")
    assert "instances=2250" in out and "0 failed" in out, out
    print(out)


@pytest.mark.gpu
def test_dropin_iteration_timeline_matches_reference_schema(tmp_path, golden):
    """weavesim::iteration_timeline (measured, one layer) writes the
    reference's Timeline JSON schema (proj/src/scheduler.cpp:301-317): the same
    keys, vocabularies and -- per layer -- the same event sequence and
    dependency edges as the reference's modeled timeline."""
    import json
    ensure_built()
    p = subprocess.run([BIN, "timeline", str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    meta, _ = golden
    for mode, n_layer in (("tokenweave", 8), ("fuseonly", 4)):
        ours = json.loads((tmp_path / f"timeline_{mode}.json").read_text())
        ref = json.loads(meta["timeline_json"][mode])
        assert set(ours) == set(ref) and ours["iteration_latency"] > 0
        assert len(ours["events"]) == n_layer
        for e, r in zip(ours["events"], ref["events"][:n_layer]):
            assert set(e) == set(r)
            assert (e["id"], e["op"], e["split"], e["stream"], e["depends_on"]) == \
                   (r["id"], r["op"], r["split"], r["stream"], r["depends_on"])
            assert 0 <= e["start"] <= e["end"]
