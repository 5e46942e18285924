#!/bin/bash
mkdir -p gpurun_out
for dbg in 0 1 2; do
  echo "== dbg $dbg"; SFFT_I8_DBG=$dbg SFFT_DEBUG=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 2>&1 | grep "\[sfft\]" | head -3
done
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
timeout 300 $CMD > gpurun_out/plain_i8.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:expsum_i8 -s 0 -c 1 -o gpurun_out/i8_full $CMD > gpurun_out/ncu_i8.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_i8.log
