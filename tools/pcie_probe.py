"""PCIe copy-engine concurrency on the box: H2D / D2H with 1 or 2 streams, and both directions at once."""
import torch

N = 256 << 20
h = [torch.empty(N, dtype=torch.uint8).pin_memory() for _ in range(4)]
d = [torch.empty(N, dtype=torch.uint8, device="cuda") for _ in range(4)]
ss = [torch.cuda.Stream() for _ in range(4)]


def run(ops, reps=5):
    for _ in range(2):
        for s, fn in ops:
            with torch.cuda.stream(s):
                fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in ss:
        s.wait_event(a)
    for _ in range(reps):
        for s, fn in ops:
            with torch.cuda.stream(s):
                fn()
    for s in ss:
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


t = run([(ss[0], lambda: d[0].copy_(h[0], non_blocking=True))])
print("H2D 1 stream GB/s", round(N / t / 1e9, 1))
t = run([(ss[0], lambda: d[0].copy_(h[0], non_blocking=True)), (ss[1], lambda: d[1].copy_(h[1], non_blocking=True))])
print("H2D 2 streams GB/s (total)", round(2 * N / t / 1e9, 1))
t = run([(ss[0], lambda: h[2].copy_(d[2], non_blocking=True))])
print("D2H 1 stream GB/s", round(N / t / 1e9, 1))
t = run([(ss[0], lambda: h[2].copy_(d[2], non_blocking=True)), (ss[1], lambda: h[3].copy_(d[3], non_blocking=True))])
print("D2H 2 streams GB/s (total)", round(2 * N / t / 1e9, 1))
t = run([(ss[0], lambda: d[0].copy_(h[0], non_blocking=True)), (ss[1], lambda: h[2].copy_(d[2], non_blocking=True))])
print("H2D+D2H concurrent GB/s (each)", round(N / t / 1e9, 1))
t = run([(ss[0], lambda: d[0].copy_(h[0], non_blocking=True)), (ss[1], lambda: d[1].copy_(h[1], non_blocking=True)),
         (ss[2], lambda: h[2].copy_(d[2], non_blocking=True)), (ss[3], lambda: h[3].copy_(d[3], non_blocking=True))])
print("2xH2D+2xD2H concurrent GB/s (per direction)", round(2 * N / t / 1e9, 1))
