"""e2e (pinned host buffers through tw_rmsnorm_residual_host) per chunk size,
T = H = 8192 bf16, interleaved reps: the chunk-size choice behind the C-ABI's
8 MiB default.  python tools/e2e_chunk_sweep.py [reps]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_11329_b200 as tw  # noqa: E402  (loads the toolkit cuBLAS before torch)
import torch  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    T = H = 8192
    hx = torch.rand(T, H, dtype=torch.bfloat16).pin_memory()
    hr = torch.rand(T, H, dtype=torch.bfloat16).pin_memory()
    hw = torch.ones(H, dtype=torch.float32)
    ho = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
    hro = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
    stream = torch.cuda.Stream()
    res = {}
    for _ in range(reps):
        for rows in (128, 256, 512, 1024, 2048):  # 2 / 4 / 8 / 16 / 32 MiB per tensor per chunk
            for _ in range(2):
                tw.rmsnorm_residual_host(hx, hr, hw, 1e-5, residual_out=hro, out=ho, chunk_rows=rows, stream=stream)
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
            ev[0].record(stream)
            for i in range(10):
                tw.rmsnorm_residual_host(hx, hr, hw, 1e-5, residual_out=hro, out=ho, chunk_rows=rows, stream=stream)
                ev[i + 1].record(stream)
            torch.cuda.synchronize()
            per = [1e3 * ev[i].elapsed_time(ev[i + 1]) for i in range(10)]
            res.setdefault(str(rows), []).append(round(statistics.median(per), 1))
    print(json.dumps({"what": "e2e us per step (median of 10) per chunk_rows, T=H=8192 bf16", "us": res}))


if __name__ == "__main__":
    main()
