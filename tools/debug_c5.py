import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_07407_b200 as S, workloads as W
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
c = W.CONFIGS[name]
w, a = W.make_batch(c, range(n))
plan = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=n, profile=True)
try:
    res = S.solve(plan, torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda())
    print("ok", res.status, res.count.tolist())
except Exception as e:
    print("ERR", e)
