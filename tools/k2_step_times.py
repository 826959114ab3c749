import sys
sys.path.insert(0, '.')
import bench
times, _ = bench.k2_timed(8192, 8192, 50, 5, bench.L2Flush("cuda:0"))
print([round(1e3 * t, 1) for t in times])
