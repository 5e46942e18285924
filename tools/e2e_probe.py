"""Where does the host-buffer pipeline's time go?  Per-solve device time (profiled plan, rep.ms_total) and wall
time of: device executes, sfft_solve_host per step, sfft_solve_host_batches (debugging aid, not a bench)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1606_07407_b200 as S
import workloads as W

prof = bool(int(__import__("os").environ.get("PROBE_PROF", "1")))
for name in sys.argv[1:] or ["c2", "c3"]:
    c = W.CONFIGS[name]
    T = 1024 if name == "c2" else 100
    nb = 10
    w, a = W.make_batch(c, range(T))
    plan = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=T, profile=prof)
    wd, ad = torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda()
    sig = S.sfft_signal_expsum(plan, wd, ad)
    outs = (torch.empty((T, c.k, c.d), dtype=torch.int32, device="cuda"),
            torch.empty((T, c.k, 2), dtype=torch.float64, device="cuda"),
            torch.empty((T,), dtype=torch.int32, device="cuda"), torch.empty((T,), dtype=torch.int32, device="cuda"))
    for _ in range(3):
        S.sfft_execute(plan, sig, outs)
    torch.cuda.synchronize()
    t = time.perf_counter(); tots = []
    for _ in range(nb):
        r = S.sfft_execute(plan, sig, outs); tots.append(r.report.ms_total)
    torch.cuda.synchronize()
    print(name, "device  wall/step %.3f ms, ms_total %s" % ((time.perf_counter() - t) * 1e3 / nb, np.round(tots, 3)))
    wh, ah = torch.from_numpy(w).pin_memory(), torch.from_numpy(a).pin_memory()
    ho = (torch.empty((T, c.k, c.d), dtype=torch.int32).pin_memory(),
          torch.empty((T, c.k, 2), dtype=torch.float64).pin_memory(),
          torch.empty((T,), dtype=torch.int32).pin_memory(), torch.empty((T,), dtype=torch.int32).pin_memory())
    S.sfft_solve_host(plan, wh, ah, ho)
    t = time.perf_counter(); tots = []
    for _ in range(nb):
        r = S.sfft_solve_host(plan, wh, ah, ho); tots.append(r.report.ms_total)
    print(name, "serial  wall/step %.3f ms, ms_total %s" % ((time.perf_counter() - t) * 1e3 / nb, np.round(tots, 3)))
    wb = wh.unsqueeze(0).expand(nb, *wh.shape).contiguous().pin_memory()
    ab = ah.unsqueeze(0).expand(nb, *ah.shape).contiguous().pin_memory()
    bo = (torch.empty((nb, T, c.k, c.d), dtype=torch.int32).pin_memory(),
          torch.empty((nb, T, c.k, 2), dtype=torch.float64).pin_memory(),
          torch.empty((nb, T), dtype=torch.int32).pin_memory(), torch.empty((nb, T), dtype=torch.int32).pin_memory())
    S.sfft_solve_host_batches(plan, wb[:2], ab[:2], tuple(o[:2] for o in bo))
    for rep in range(3):
        t = time.perf_counter()
        rc, of, oc, on, os_, reps = S.sfft_solve_host_batches(plan, wb, ab, bo)
        print(name, "batches wall/step %.3f ms, ms_total %s" % ((time.perf_counter() - t) * 1e3 / nb,
                                                             np.round([r.ms_total for r in reps], 3)))
