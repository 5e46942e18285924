import torch, sys
sys.path.insert(0, '.')
import paper_1606_07407_b200 as S, workloads as W
for name in sys.argv[1:]:
    c = W.CONFIGS[name]
    w, a = W.make_batch(c, range(100))
    plan = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=100, profile=True)
    sig = S.sfft_signal_expsum(plan, torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda())
    for i in range(3):
        r = S.sfft_execute(plan, sig)
    torch.cuda.synchronize()
    print(name, 'DONE', flush=True)
