"""K2 at the short batches of configs[2] (T = 1024 / 2048, H = 8192 bf16):
flushed and back-to-back (steady-state) CUDA-event times, beside a plain
device copy of the same byte count (torch copy_ of input->output and
residual->residual_out), the practical floor for this many bytes at this size.

    python tools/k2_small_t.py [time|profile T]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_11329_b200 as tw  # noqa: E402

H = 8192


def bufs(T):
    import torch
    x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
    r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
    w = torch.rand(H, device="cuda") + 0.5
    return x, r, w, torch.empty_like(x), torch.empty_like(x)


def timed(fn, flush, reps=50):
    import torch
    for _ in range(5):
        if flush is not None:
            flush.fill_(1)
        fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        if flush is not None:
            flush.fill_(i & 0x7F)
            flush.view(torch.float32).sum()  # read back: L2 left holding clean lines (bench.py's L2Flush)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(1e3 * s.elapsed_time(e))
    return statistics.median(ts)


def back_to_back(fn, n=200):
    import torch
    for _ in range(5):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return 1e3 * s.elapsed_time(e) / n


def main():
    import torch
    mode = sys.argv[1] if len(sys.argv) > 1 else "time"
    if mode == "profile":
        T = int(sys.argv[2])
        x, r, w, o, ro = bufs(T)
        for _ in range(3):
            tw.rmsnorm_residual(x, r, w, 1e-5, residual_out=ro, out=o)
        torch.cuda.synchronize()
        return
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    sizes = [int(t) for t in os.environ.get("K2_SIZES", "512,1024,2048,4096,8192").split(",")]
    for T in sizes:
        x, r, w, o, ro = bufs(T)
        k2 = lambda: tw.rmsnorm_residual(x, r, w, 1e-5, residual_out=ro, out=o)  # noqa: E731

        def cp():
            o.copy_(x)
            ro.copy_(r)
        alg = 4 * T * H * 2
        k = timed(k2, flush)
        c = timed(cp, flush)
        kb = back_to_back(k2)
        res[T] = {"k2_flushed_us": round(k, 2), "k2_b2b_us": round(kb, 2), "copy2_flushed_us": round(c, 2),
                  "k2_GBps": round(alg / k / 1e3, 1), "copy2_GBps": round(alg / c / 1e3, 1),
                  "k2_b2b_GBps": round(alg / kb / 1e3, 1)}
        print(T, res[T], flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
