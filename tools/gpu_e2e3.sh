cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2w}
for c in c2 c3; do
BENCH_E2E_DEBUG=4 timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --latency-steps 0 --fp64-steps 0 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 300 python tools/e2e_probe.py c2 > gpurun_out/${TAG}_probe.log 2>&1
