"""Single-signal latency breakdown (SFFT_DEBUG per-iteration events on stderr) -- debugging aid."""
import os, sys, time
import torch
sys.path.insert(0, ".")
import paper_1606_07407_b200 as S
import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
c = W.CONFIGS[name]
w, a = W.make_batch(c, range(1))
for prof in (False, True):
    plan = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=1, profile=prof)
    wd, ad = torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda()
    sig = S.sfft_signal_expsum(plan, wd, ad)
    outs = (torch.empty((1, c.k, c.d), dtype=torch.int32, device="cuda"),
            torch.empty((1, c.k, 2), dtype=torch.float64, device="cuda"),
            torch.empty((1,), dtype=torch.int32, device="cuda"), torch.empty((1,), dtype=torch.int32, device="cuda"))
    for _ in range(3):
        r = S.sfft_execute(plan, sig, outs)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = S.sfft_execute(plan, sig, outs); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(name, "profile" if prof else "plain", "median %.3f ms min %.3f iters %d launches %d" %
          (ts[len(ts) // 2], ts[0], r.report.iterations, r.report.kernel_launches), flush=True)
