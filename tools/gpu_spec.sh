# multi-prime speculation: GPU tests, then bench lines with the single-solve latency legs (G = 1, 2, 4)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r4a}
timeout 1200 python -m pytest tests -m gpu -x -q -k "${TESTK:-speculation or config1 or full_size or forced_false}" > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for c in ${CONFIGS:-c3 c5 c4}; do
  timeout 900 python bench.py --config $c --steps 5 --no-cpu-baseline --e2e-steps 0 --latency-steps 10 --fp64-steps 0 --spec-primes 2 4 8 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
