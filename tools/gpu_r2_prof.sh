# bench lines of every config + the ncu launch list and one full capture of the top kernels (C3)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2e}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_gpuinfo.txt 2>&1
lscpu > gpurun_out/${TAG}_lscpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err
for c in c5 c4 c2 c1; do
  timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --latency-steps 5 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0"
timeout 300 $CMD1 > gpurun_out/${TAG}_plain1.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:pfft|expsum_i8' -c 2 -o gpurun_out/${TAG}_full $CMD1 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
