# ncu launch list of the headline bench command (no extra legs) and one full capture of its top kernels
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r5l}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0 --spec-steps 0"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
if [ -n "$FULL" ]; then
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0 --spec-steps 0"
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:pfft|expsum_i8' -c 2 -o gpurun_out/${TAG}_full $CMD1 > gpurun_out/${TAG}_ncu_full.log 2>&1
fi
echo done
