"""Tiny batches: fixed cost of each K2 engine (bench methodology)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    if len(sys.argv) > 1:
        from bench import L2Flush, k2_timed
        flush = L2Flush("cuda:0")
        out = {}
        for T in (4, 64, 256, 512, 1024):
            ts, _ = k2_timed(T, 8192, 50, 5, flush)
            out[T] = round(1e3 * sum(ts) / len(ts), 2)
        print(os.environ["TW_K2_ENGINE"], out, flush=True)
    else:
        for eng in ("tma", "bulk", "rows", "flat"):
            subprocess.run([sys.executable, __file__, "x"], env=dict(os.environ, TW_K2_ENGINE=eng), check=True)
