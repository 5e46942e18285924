"""NEXT #1: replay of the paper's own experiment on the GPU path.

PAPER.md:422-426 (Sec. 5): d in {100, 1000}, d1 = 5 (d2 = 20 / 200), N = 20, k = 2^0 .. 2^10,
eps = 1/(2 N^d1), c = 5, |a_j| = 1 with uniform phase, 100 trials per (d, k).  Reported per (d, k):
exact-recovery rate, average l2 error (SPEC S:79 matched/unmatched formula) and its square (the
paper's "below 2^-52" most plausibly plots a squared norm, reading notes), average
samples (Fig. 5), and GPU time per solve (our analogue of the CPU TICKS of Fig. 6).

    python tools/paper_replay.py [--trials 100] [--ks 0-10] [--ds 100,1000] [--out profiles/r01_paper_replay.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402


def l2_error(w_true, a_true, w_rec, a_rec):
    """sqrt(sum_matched |a - a^|^2 + sum_unmatched |a|^2 + sum_spurious |a^|^2)."""
    t = {tuple(r): a for r, a in zip(w_true.tolist(), a_true)}
    g = {tuple(r): a for r, a in zip(w_rec.tolist(), a_rec)}
    s = 0.0
    for key, a in t.items():
        s += abs(a - g[key]) ** 2 if key in g else abs(a) ** 2
    for key, a in g.items():
        if key not in t:
            s += abs(a) ** 2
    return float(np.sqrt(s))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=100)
    ap.add_argument("--ks", default="0-10")
    ap.add_argument("--ds", default="100,1000")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_paper_replay.json"))
    args = ap.parse_args()
    import torch
    import paper_1606_07407_b200 as S

    lo, hi = (int(x) for x in args.ks.split("-"))
    rows = []
    for d in (int(x) for x in args.ds.split(",")):
        for e in range(lo, hi + 1):
            k = 2 ** e
            c = W.paper_config(d, k, trials=args.trials)
            w, a = W.make_batch(c, range(args.trials))
            plan = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=args.trials, profile=True)
            wd, ad = torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda()
            S.solve(plan, wd, ad)                      # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = S.solve(plan, wd, ad)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            gw, ga, gn = res.freqs.cpu().numpy(), res.coeffs.cpu().numpy(), res.count.cpu().numpy()
            exact, l2 = 0, []
            for i in range(args.trials):
                n = int(gn[i])
                ws, as_ = W.canonical_sort(w[i], a[i])
                exact += int(n == k and np.array_equal(gw[i, :n], ws))
                l2.append(l2_error(w[i], a[i], gw[i, :n], ga[i, :n]))
            rep = res.report
            row = {"d": d, "k": k, "trials": args.trials, "exact_rate": exact / args.trials,
                   "l2_mean": float(np.mean(l2)), "l2_max": float(np.max(l2)),
                   "l2_sq_mean": float(np.mean(np.square(l2))),
                   "log2_l2_sq_mean": float(np.log2(max(np.mean(np.square(l2)), 1e-300))),
                   "samples_mean": rep.samples_used / args.trials, "iterations": rep.iterations,
                   "gpu_ms_per_batch": dt * 1e3, "gpu_us_per_solve": dt * 1e6 / args.trials,
                   "expsum_ms": rep.ms_expsum, "fft_ms": rep.ms_fft, "decode_ms": rep.ms_decode}
            rows.append(row)
            print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"workload": "PAPER.md:422 (N=20, d1=5, eps=1/(2 N^5), c=5, |a|=1), seeded synthetic",
               "rows": rows}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
