# ncu --set full of the first C launches of kernel KREGEX in a short bench run (CONFIG)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2k}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CMD="python bench.py --config ${CONFIG:-c3} --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-2} -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
