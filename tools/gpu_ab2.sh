# A/B of two in-tree libraries (LIBS) on bench configs (CONFIGS), alternating, 2 rounds
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2ab}
for round in 1 2; do
for c in ${CONFIGS:-c5 c3}; do
for lib in ${LIBS:-libsfft_base.so libsfft.so}; do
  SFFT_LIB_PATH=paper_1606_07407_b200/$lib timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$round','$c','$lib', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items() if isinstance(v, float)}, d['verified_exact_recovery'])" >> gpurun_out/${TAG}.log 2>&1
done; done; done
