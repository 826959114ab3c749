"""Per-op timeline of one weaved layer (Llama TP=8 shapes, T=8192) at several
boundary budgets -- for comparing how boxes schedule the two streams."""
import sys

sys.path.insert(0, '.')
from paper_2505_11329_b200 import weave  # noqa: E402

r = weave.LayerRunner("llama-70b", tp=8, max_tokens=8192)
for b in (16, 64):
    us = r.run(8192, "tokenweave", prefix=4096, boundary_sms=b, layers=4)
    ev = r.trace()
    t0 = min(e["start_us"] for e in ev)
    print(f"budget {b}: {us:.1f} us/layer")
    for e in ev:
        print(f"  {e['op']:14s} {e['split']:7s} {e['stream']:8s} {e['start_us'] - t0:8.1f} {e['end_us'] - t0:8.1f} "
              f"({e['end_us'] - e['start_us']:.1f})")
us = r.run(8192, "fuseonly", layers=4)
ev = r.trace()
t0 = min(e["start_us"] for e in ev)
print(f"fuseonly: {us:.1f}")
for e in ev:
    print(f"  {e['op']:14s} {e['split']:7s} {e['stream']:8s} {e['start_us'] - t0:8.1f} {e['end_us'] - t0:8.1f} "
          f"({e['end_us'] - e['start_us']:.1f})")
