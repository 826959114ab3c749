"""How the L2-flush method changes K2 timings (write flush / read flush / none)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(H=8192, reps=30):
    import torch
    import paper_2505_11329_b200 as tw
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sink = torch.empty(1, device="cuda")
    for T in (1024, 2048, 4096, 8192, 16384):
        sets = []
        for _ in range(3):
            x = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
            r = torch.randn(T, H, device="cuda", dtype=torch.bfloat16)
            sets.append((x, r, torch.empty_like(x), torch.empty_like(x)))
        w = torch.ones(H, device="cuda")
        res = {}
        for mode in ("write", "write+read", "none", "copy_ref"):
            ts = []
            for i in range(reps + 3):
                x, r, o, ro = sets[i % 3]
                if mode == "write":
                    flush.fill_(i)
                elif mode == "write+read":
                    flush.fill_(i)
                    sink.copy_(flush.view(torch.float32).sum())
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                if mode == "copy_ref":
                    o.copy_(x)
                else:
                    tw.rmsnorm_residual(x, r, w, residual_out=ro, out=o)
                e.record()
                if mode != "none":
                    torch.cuda.synchronize()
                ts.append((s, e))
            torch.cuda.synchronize()
            vals = [s.elapsed_time(e) for s, e in ts[3:]]
            us = 1e3 * statistics.median(vals)
            nb = (4 if mode != "copy_ref" else 2) * T * H * 2
            res[mode] = (round(us, 2), round(nb / us / 1e3, 1))
        print(T, res, flush=True)


if __name__ == "__main__":
    main()
