"""A/B microbenchmark of the two K2 engines (bulk pipeline vs row engine)."""
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(H=8192, tokens=(1024, 2048, 4096, 8192, 16384), reps=30):
    import torch
    import paper_2505_11329_b200 as tw
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {}
    for T in tokens:
        x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
        w = torch.ones(H, device="cuda")
        o, ro = torch.empty_like(x), torch.empty_like(x)
        for _ in range(3):
            tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o)
        ts = []
        for i in range(reps):
            flush.fill_(i)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        us = 1e3 * statistics.median(ts)
        out[T] = (round(us, 2), round(4 * T * H * 2 / us / 1e3, 1))
    return out


def H_label():
    return os.environ.get("TW_K2_ENGINE", "tma") + " H=" + sys.argv[2]


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        print(H_label(), run(H=int(sys.argv[2])))
    else:
        for H in (8192, 4096, 6144):
            for eng in ("tma", "bulk", "rows", "flat"):
                env = dict(os.environ, TW_K2_ENGINE=eng)
                subprocess.run([sys.executable, __file__, "child", str(H)], env=env, check=True)
