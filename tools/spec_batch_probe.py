"""Batched throughput with multi-prime speculation (R26): ms per 100-signal execute at G = 1, 2, 4 (unprofiled plans,
L2 flushed between executes, CUDA events) -- debugging aid, not a bench line."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1606_07407_b200 as S
import workloads as W

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in sys.argv[1:] or ["c5", "c3", "c4", "c2"]:
    c = W.CONFIGS[name]
    T = 1024 if name == "c2" else 100
    w, a = W.make_batch(c, range(T))
    wd, ad = torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda()
    for G in (1, 2, 3, 4):
        plan = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=T, spec_primes=G)
        sig = S.sfft_signal_expsum(plan, wd, ad)
        outs = (torch.empty((T, c.k, c.d), dtype=torch.int32, device="cuda"),
                torch.empty((T, c.k, 2), dtype=torch.float64, device="cuda"),
                torch.empty((T,), dtype=torch.int32, device="cuda"), torch.empty((T,), dtype=torch.int32, device="cuda"))
        for _ in range(3):
            r = S.sfft_execute(plan, sig, outs)
        ts = []
        for _ in range(6):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = S.sfft_execute(plan, sig, outs)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ok = all(np.array_equal(outs[0][i].cpu().numpy(), W.canonical_sort(w[i], a[i])[0]) for i in range(T))
        print(name, "G", G, "ms %.3f" % sorted(ts)[len(ts) // 2], "iters", r.report.iterations,
              "samples", r.report.samples_used, "exact", ok, flush=True)
        del plan, sig, outs
