# A/B of environment settings (ENVS, '|' separated; 'none' = defaults) on bench configs (CONFIGS)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2env}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
IFS='|' read -ra EV <<< "${ENVS:-none}"
for round in 1 2; do
for c in ${CONFIGS:-c5 c3}; do
for e in "${EV[@]}"; do
  if [ "$e" = "none" ]; then pre=""; else pre="env $e"; fi
  $pre timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$round','$c','[$e]', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items() if isinstance(v, float)}, d['verified_exact_recovery'])" >> gpurun_out/${TAG}.log 2>&1
done; done; done
