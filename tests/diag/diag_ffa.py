"""Diagnostic (GPU box): forced-false-accept workloads, GPU vs oracle per seed -- solo (batch 1) and batched --
first divergent iteration of the (p, accepted) trace.  Usage: python tests/diag/diag_ffa.py [ci] [extra] [path]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1606_07407_b200 as S  # noqa: E402
import workloads as W  # noqa: E402
from test_oracle_pins import FFA_CASES, FFA_PARAMS, ffa_config  # noqa: E402

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 0
extra = int(sys.argv[2]) if len(sys.argv) > 2 else 0
path = int(sys.argv[3]) if len(sys.argv) > 3 else 1
(d, N, k, blocks), _ = FFA_CASES[ci]
c = ffa_config(d, N, k, blocks)
kw = dict(FFA_PARAMS, extra_checks=extra)
P = O.params_for(c, **kw)
trials = list(range(40))
w, a = W.make_batch(c, trials)
planB = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=40, expsum_path=path, **kw)
resB = S.solve(planB, torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda())
plan1 = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=1, expsum_path=path, **kw)
nbad = 0
for t in trials:
    ref = O.solve(P, w[t], a[t])
    r1 = S.solve(plan1, torch.from_numpy(w[t:t + 1]).cuda(), torch.from_numpy(a[t:t + 1]).cuda())
    rep = r1.report
    n = min(len(ref.trace), 64, rep.n_iter_logged)
    gp = [rep.primes[i] for i in range(n)]
    ga = [rep.accepted[i] for i in range(n)]
    div = next((i for i in range(n) if gp[i] != ref.trace[i, 1] or ga[i] != ref.trace[i, 4]), None)
    s1, sb = int(r1.per_status[0]), int(resB.per_status[t])
    c1, cb = int(r1.count[0]), int(resB.count[t])
    same_b = (s1 == sb and c1 == cb and np.array_equal(r1.freqs[0, :c1].cpu().numpy(), resB.freqs[t, :cb].cpu().numpy()))
    okr = s1 == ref.status and (ref.status == O.ECORRUPT or (c1 == ref.w.shape[0] and np.array_equal(
        r1.freqs[0, :c1].cpu().numpy(), ref.w)))
    if div is not None or not okr or not same_b:
        nbad += 1
        print(f"seed {t}: oracle st={ref.status} n={ref.w.shape[0]} it={ref.iterations} | gpu solo st={s1} n={c1} "
              f"it={rep.iterations} | batch st={sb} n={cb} same_as_solo={same_b} | first trace divergence {div}")
        if div is not None:
            lo = max(0, div - 1)
            print("   oracle (i,p,m,ncand,na,nonempty,acc,pruned):", ref.trace[lo:div + 2].tolist())
            print("   gpu (p,na):", list(zip(gp[lo:div + 2], ga[lo:div + 2])))
print(f"ci={ci} extra={extra} path={path}: {nbad} of {len(trials)} seeds differ")
