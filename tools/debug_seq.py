import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_07407_b200 as S, workloads as W
for name, tag, n in [("c2", "p", 16), ("c2", "a", 16), ("c4", "p", 4), ("c4", "a", 1), ("c3", "p", 4), ("c3", "a", 1), ("c5", "p", 4)]:
    c = W.CONFIGS[name]
    blocks = c.blocks if tag == "p" else c.alt_blocks
    w, a = W.make_batch(c, range(n))
    plan = S.sfft_plan(c.d, c.N, c.k, blocks=blocks, batch=n)
    try:
        res = S.solve(plan, torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda())
        print(name, tag, "ok", res.status, res.count.tolist()[:4], flush=True)
    except Exception as e:
        print(name, tag, "ERR", e, flush=True)
        break
