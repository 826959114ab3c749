"""bench.py's reference arm on CPU: the reference's own code only -- the
process never maps the product libraries (so the driver's reference-vs-ours
ratio compares two independent arms)."""
import json
import os
import subprocess
import sys

import pytest

from tests.conftest import ROOT

PROBE = r"""
import json, os, sys
root = os.path.realpath(os.getcwd())
sys.argv = ["bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1", "--tokens", "256",
            "--hidden", "512", "--gpus", GPUS]
sys.path.insert(0, ".")
import bench
rc = bench.main()
maps = open("/proc/self/maps").read()
libs = sorted({ln.split()[-1] for ln in maps.splitlines()
               if ln.endswith(".so") and (root in os.path.realpath(ln.split()[-1]) or "libtw" in ln)})
print(json.dumps({"rc": rc, "libs": libs, "pkg": [m for m in sys.modules if m.startswith("paper_2505")]}))
"""


@pytest.mark.parametrize("gpus", ["1", "4"])
def test_reference_arm_loads_only_the_reference(gpus):
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libweavesim_ref.so")):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    p = subprocess.run([sys.executable, "-c", PROBE.replace("GPUS", repr(gpus))], cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(ln) for ln in p.stdout.splitlines() if ln.startswith("{")]
    line, probe = lines[0], lines[-1]
    assert line["impl"] == "reference" and line["n_gpus"] == int(gpus) and line["value"] > 0
    assert line["dtype"] == "f32" and line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["value"] == line["value"] and len(line["step_ms"]) == 2
    assert probe["rc"] == 0 and probe["pkg"] == []
    assert not any("libtw" in lib or "libweavesim_b200" in lib for lib in probe["libs"]), probe["libs"]
    assert any("oracle/_ref" in lib for lib in probe["libs"]), probe["libs"]
