nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_fp64.csv &
SMI=$!
./tools/fp64_peak > gpurun_out/fp64_peak.log 2>&1
kill $SMI
nproc >> gpurun_out/fp64_peak.log; lscpu | grep 'Model name' >> gpurun_out/fp64_peak.log
cat gpurun_out/fp64_peak.log
