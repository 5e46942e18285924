cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2h}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
for c in c3 c5; do
SFFT_I8_PROF=1 timeout 300 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0 2>&1 | grep -E "i8prof" > gpurun_out/${TAG}_i8prof_$c.log
done
