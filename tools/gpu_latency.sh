cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2lat}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
cat > /tmp/lat.py <<'PY'
import torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_1606_07407_b200 as S, workloads as W
for name in ("c3", "c5"):
    c = W.CONFIGS[name]
    w, a = W.make_batch(c, [0])
    plan = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=1, profile=True)
    sig = S.sfft_signal_expsum(plan, torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda())
    for i in range(3):
        r = S.sfft_execute(plan, sig)
    torch.cuda.synchronize()
    rep = r.report
    print(name, "iters", rep.iterations, "ms_total", rep.ms_total, "expsum", rep.ms_expsum, "fft", rep.ms_fft, "decode", rep.ms_decode, "other", rep.ms_other, flush=True)
PY
SFFT_DEBUG=1 timeout 300 python /tmp/lat.py > gpurun_out/${TAG}.log 2>&1
