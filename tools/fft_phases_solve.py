"""Phase cycle counters of pfft_kernel (SFFT_FFT_PROF tuning build, SFFT_LIB_PATH) over one batched execute of a
BASELINE config: load | DIF | mid | DIT | epilogue (fused select / test), cycles summed over all CTAs."""
import ctypes
import sys

import torch

import paper_1606_07407_b200 as S
import workloads as W


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    c = W.CONFIGS[name]
    w, a = W.make_batch(c, list(range(c.trials if c.trials <= 100 else 100)))
    plan = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=w.shape[0], table_cache_slots=1024, max_iter=max_iter)
    wt, at = torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda()
    S.solve(plan, wt, at)
    buf = (ctypes.c_ulonglong * 8)()
    S.lib().sfft_debug_fft_prof(buf, 1)
    r = S.solve(plan, wt, at)
    torch.cuda.synchronize()
    S.lib().sfft_debug_fft_prof(buf, 1)
    names = ["load", "dif", "mid", "dit", "select(line0)", "wait(line n)", "test(line n)"]
    tot = sum(buf[i] for i in range(7)) or 1
    print(name, "max_iter", max_iter, "iterations", r.report.iterations, "| " + ", ".join(f"{names[i]} {100 * buf[i] / tot:.0f}%" for i in range(7)),
          f"| total {tot / 1e6:.1f} Mcycles")


if __name__ == "__main__":
    main()
