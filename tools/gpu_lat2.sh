cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r3a}
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-forced_false or accumulate or prune or e2e_vs_oracle or cap}" > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for c in c3 c5 c4; do SFFT_DEBUG=1 timeout 300 python tools/latency_probe.py $c > gpurun_out/${TAG}_lat_$c.log 2>&1; done
for c in ${CONFIGS:-c3 c4}; do
  timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
