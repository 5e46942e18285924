cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r4h}
for c in ${CONFIGS:-c3 c5}; do
SFFT_DEBUG=1 timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0 > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err
done
