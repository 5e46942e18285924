cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2e2e}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for ch in 1 2 3 4; do
  for c in c3 c2; do
  SFFT_HOST_CHUNKS=$ch timeout 600 python bench.py --config $c --steps 3 --e2e-steps 5 --no-cpu-baseline --latency-steps 0 --fp64-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('chunks $ch $c', round(d['value']/1e6,2), 'device M/s; e2e', round(d['e2e']['value']/1e6,2), d['verified_exact_recovery'])" >> gpurun_out/${TAG}.log 2>&1
  done
done
timeout 600 python -m pytest tests -m gpu -q -k "solve_host or bench_launch" > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
