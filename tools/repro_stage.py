import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch, oracle as O, workloads as W
import paper_1606_07407_b200 as S
c = W.CONFIGS["c2"]
order = [((1, 1, 1), 101, 2), ((2, 1), 503, 1)] if len(sys.argv) > 1 else [((2, 1), 503, 1), ((1, 1, 1), 101, 2)]
for blocks, p, m in order:
    w, a = W.make_signal(c, 2)
    P = O.params_for(c, blocks=blocks); E, _, _ = O.prepare(P); v = O.project(P, w)
    try:
        plan = S.sfft_plan(c.d, c.N, c.k, blocks=blocks, expsum_path=1)
        print("plan ok", blocks, flush=True)
        got = S.sfft_stage_expsum(plan, torch.from_numpy(np.ascontiguousarray(v.T)).cuda(), torch.from_numpy(a).cuda(), p, m)
        torch.cuda.synchronize(); print("ok", blocks, flush=True)
    except Exception as ex:
        print("ERR", blocks, ex, flush=True)
