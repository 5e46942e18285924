# host-buffer e2e: the batch-pipeline test, then bench lines with the e2e legs only
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-solve_host or binding_validates}" > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for c in ${CONFIGS:-c3 c2 c5}; do
  timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --e2e-steps ${E2E:-10} --latency-steps 0 --fp64-steps 0 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
python - <<PY > gpurun_out/${TAG}_summary.txt
import json,glob
for f in sorted(glob.glob("gpurun_out/${TAG}_bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        e=d['e2e']
        print(f, round(d['value']/1e6,3), 'M/s', round(d['ms_per_step'],3), 'ms', 'e2e', round(e['value']/1e6,3), 'serial', round(e['serial_value']/1e6,3), 'exact', d['verified_exact_recovery'])
    except Exception as ex: print(f, 'ERR', ex)
PY
