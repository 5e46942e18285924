"""Diagnostic (GPU box): registry after t iterations, GPU vs oracle, for one forced-false-accept seed.
Usage: python tests/diag/diag_ffa2.py ci extra path seed t0 t1"""
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

ci, extra, path, seed, t0, t1 = (int(x) for x in sys.argv[1:7])
(d, N, k, blocks), _ = FFA_CASES[ci]
c = ffa_config(d, N, k, blocks)
w, a = W.make_signal(c, seed)
print(f"== ci={ci} extra={extra} path={path} seed={seed}")
for t in range(t0, t1 + 1):
    kw = dict(FFA_PARAMS, extra_checks=extra, max_iter=t)
    st, rv, ra = O.solve_raw(O.params_for(c, **kw), w, a)
    plan = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=1, expsum_path=path, **kw)
    res = S.solve(plan, torch.from_numpy(w[None]).cuda(), torch.from_numpy(a[None]).cuda())
    n = int(res.count[0])
    ga = res.coeffs[0, :n].cpu().numpy()
    gw = res.freqs[0, :n].cpu().numpy()
    key = lambda z: (round(z.real, 9), round(z.imag, 9))
    so = sorted(ra, key=key)
    sg = sorted(ga, key=key)
    print(f"t={t}: oracle |R|={len(ra)} st={st} | gpu |R|={n} st={int(res.per_status[0])} "
          f"p={[res.report.primes[i] for i in range(t)][-3:]} acc={[res.report.accepted[i] for i in range(t)][-3:]}")
    oset = {key(z) for z in so}
    gset = {key(z) for z in sg}
    only_o = [z for z in so if key(z) not in gset]
    only_g = [(z, gw[i].tolist()) for i, z in enumerate(ga) if key(z) not in oset]
    if only_o or only_g:
        print("   only oracle:", [(z, rv[list(ra).index(z)].tolist()) for z in only_o])
        print("   only gpu   :", only_g)
