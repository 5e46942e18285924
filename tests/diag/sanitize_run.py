"""Small solves for compute-sanitizer runs (memcheck / racecheck / synccheck / initcheck, one tool per GPU call):
C1 (both partitions), two C2 signals, the reduced C3-like workload of smoke() (int8 tcgen05 exp-sum), a
forced-false-accept workload (accumulate / prune / cap paths) and one line-shard group solve; each checked
against the oracle's frequency sets."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1606_07407_b200 as S  # noqa: E402
import workloads as W  # noqa: E402


def run(c, trials, blocks=None, **kw):
    blocks = blocks or c.blocks
    w, a = W.make_batch(c, trials)
    plan = S.sfft_plan(c.d, c.N, c.k, blocks=blocks, batch=len(trials), **kw)
    res = S.solve(plan, torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda())
    torch.cuda.synchronize()
    okw = {k: v for k, v in kw.items() if k in ("tol", "round_tol", "extra_checks", "max_iter")}
    for i in range(len(trials)):
        ref = O.solve(O.params_for(c, blocks=blocks, **okw), w[i], a[i])
        n = int(res.count[i])
        assert int(res.per_status[i]) == ref.status, (c.name, i)
        if ref.status != O.ECORRUPT:
            assert np.array_equal(res.freqs[i, :n].cpu().numpy(), ref.w), (c.name, i)
    print("ok", c.name, blocks, kw, flush=True)


def main():
    torch.cuda.set_device(0)
    c1, c2 = W.CONFIGS["c1"], W.CONFIGS["c2"]
    run(c1, list(range(4)))
    run(c1, list(range(4)), blocks=c1.alt_blocks)
    run(c2, [0, 1])
    c3s = W.custom_config(16, 65536, 60, (2,) * 8, cfg=90, rho="uniform1_10")
    run(c3s, [0, 1])
    ffa = W.custom_config(3, 32, 30, (1, 1, 1), cfg=81, rho="uniform1_10")
    run(ffa, [13, 28], tol=0.5, round_tol=0.5, extra_checks=0, max_iter=60)
    # line shards (group executor on one device)
    w, a = W.make_batch(c3s, [0])
    plans = [S.sfft_plan(c3s.d, c3s.N, c3s.k, blocks=c3s.blocks, batch=1, line_shards=2, line_rank=g) for g in (0, 1)]
    wt, at = torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda()
    res = S.sfft_execute_group(plans, [S.sfft_signal_expsum(p, wt, at) for p in plans])
    ref = O.solve(O.params_for(c3s), w[0], a[0])
    assert np.array_equal(res.freqs[0, :int(res.count[0])].cpu().numpy(), ref.w)
    print("ok line shards", flush=True)
    print("sanitize run ok")


if __name__ == "__main__":
    main()
