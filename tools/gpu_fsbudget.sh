# fused-sampling budget sweep (SFFT_FS_BUDGET): single-solve latency and short bench lines
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r3m}
for b in 0 1000 2500 5000 10000; do
  for c in c3 c5 c4; do echo "budget $b $(SFFT_FS_BUDGET=$b timeout 300 python tools/latency_probe.py $c 2>/dev/null | grep plain)"; done
  for c in c5 c4 c3; do
    SFFT_FS_BUDGET=$b timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('budget $b $c', round(d['ms_per_step'],3), d['verified_exact_recovery'])"
  done
done > gpurun_out/${TAG}_fsbudget.log 2>&1
