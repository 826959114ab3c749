"""One weaved layer and one fuse-only layer (Llama TP=8 shapes, T=8192) for an
ncu launch list: which cuBLAS kernels this box's heuristics pick."""
import sys

sys.path.insert(0, '.')
from paper_2505_11329_b200 import weave  # noqa: E402

r = weave.LayerRunner("llama-70b", tp=8, max_tokens=8192)
print("weave", r.run(8192, "tokenweave", prefix=4096, boundary_sms=64, layers=1))
print("fuseonly", r.run(8192, "fuseonly", layers=1))
