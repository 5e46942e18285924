# build, the exp-sum/decode stage tests, then short bench lines (C3, C5, C4) without the extra legs
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2q}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-stage_expsum or full_size}" > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for c in ${CONFIGS:-c3 c5 c4}; do
  timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
python - <<PY > gpurun_out/${TAG}_summary.txt
import json,glob
for f in sorted(glob.glob("gpurun_out/${TAG}_bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']/1e6,3), 'M/s', round(d['ms_per_step'],3), 'ms', 'frac', round(d['roofline']['frac'],3), 'kms', {k: round(v,3) for k,v in d['kernel_ms_per_step'].items() if isinstance(v, float)}, 'exact', d['verified_exact_recovery'])
    except Exception as e: print(f, 'ERR', e)
PY
