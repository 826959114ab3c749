"""Per-step CUDA-event times of bench.py's K2 timed loop (T = H = 8192 bf16,
50 steps): shows whether any step is an outlier."""
import sys
sys.path.insert(0, '.')
import bench
times, _ = bench.k2_timed(8192, 8192, 50, 5, bench.L2Flush("cuda:0"))
print([round(1e3 * t, 1) for t in times])
