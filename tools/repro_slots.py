"""Largest batch a plan runs (C2 shape): debugging aid for the table-assignment shared-memory bound."""
import sys, torch
sys.path.insert(0, ".")
import paper_1606_07407_b200 as S, workloads as W
c = W.CONFIGS["c2"]
for T in [int(x) for x in (sys.argv[1:] or ["1024", "1536", "2048", "3072", "4096", "6144", "8192"])]:
    w, a = W.make_batch(c, [t % 1024 for t in range(T)])
    try:
        plan = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=T)
        r = S.solve(plan, torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda())
        print(T, "ok", r.status, flush=True)
    except Exception as e:
        print(T, "ERR", e, flush=True)
