"""weave_repeat_check without importing torch: which cuBLAS the layer runner
binds depends on whether torch (and its bundled libcublas) loaded first."""
import sys

sys.path.insert(0, '.')
from paper_2505_11329_b200 import weave  # noqa: E402

T = 8192
r = weave.LayerRunner("llama-70b", tp=8, max_tokens=T)
for rep in range(2):
    print("notorch", rep, {m: round(r.run(T, m, layers=6), 1) for m in ("unfused", "fuseonly", "nocomm")},
          {b: round(r.run(T, "tokenweave", prefix=4096, boundary_sms=b, layers=6), 1) for b in (16, 32, 64)},
          flush=True)
with open("/proc/self/maps") as f:
    print(sorted({l.split()[-1] for l in f if "cublas" in l}))
