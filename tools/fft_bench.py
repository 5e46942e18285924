"""Microbenchmark of the batched Bluestein FFT kernel (pfft_kernel) through sfft_stage_pfft: n lines of
length p (the C3 iteration-1 shape by default), median of several calls.  The stage call also computes
the prime's tables (one CTA) -- small against thousands of lines."""
import sys
import time

import torch

import paper_1606_07407_b200 as S
import workloads as W


def main():
    c = W.CONFIGS["c3"]
    plan = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks)
    shapes = [(5003, 5100), (2503, 2100), (1009, 2600), (503, 5000)]
    if len(sys.argv) > 1:
        shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
    g = torch.Generator(device="cuda").manual_seed(0)
    lib = S.lib()
    prof = getattr(lib, "sfft_debug_fft_prof", None) if hasattr(lib, "sfft_debug_fft_prof") else None
    import ctypes
    buf = (ctypes.c_ulonglong * 8)()
    for p, n in shapes:
        x = torch.randn((n, p, 2), dtype=torch.float64, device="cuda", generator=g)
        xc = torch.view_as_complex(x)
        ts = []
        for _ in range(7):
            torch.cuda.synchronize()
            t = time.perf_counter()
            S.sfft_stage_pfft(plan, xc)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        ms = sorted(ts)[3] * 1e3
        if prof is not None:
            prof(buf, 1)                       # reset after the timing runs
            S.sfft_stage_pfft(plan, xc)
            torch.cuda.synchronize()
            prof(buf, 1)
            names = ["load", "dif", "mid", "dit", "epilogue"]
            tot = sum(buf[i] for i in range(5)) or 1
            print("   phases (cycles/CTA): " + ", ".join(f"{names[i]} {buf[i] / n:.0f} ({100 * buf[i] / tot:.0f}%)"
                                                       for i in range(5)))
        print(f"p={p:5d} lines={n:5d}: {ms:.3f} ms  {ms * 1e3 / n * 148:.1f} us/line/SM  "
              f"{32.0 * p * n / (ms / 1e3) / 1e9:.0f} GB/s (32 B/sample)", flush=True)


if __name__ == "__main__":
    main()
