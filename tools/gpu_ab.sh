#!/bin/bash
# A/B of library builds on the bench (C3 by default): ms/step, kernel split, exact recovery
mkdir -p gpurun_out
for lib in ${LIBS:-libsfft.so}; do
  for cfg in ${CFGS:-c3}; do
    SFFT_LIB_PATH=paper_1606_07407_b200/$lib timeout 300 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 \
      --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0 ${BENCH_ARGS} 2>/dev/null | tail -1 > gpurun_out/ab_${lib}_${cfg}.json
    python tools/bench_line.py gpurun_out/ab_${lib}_${cfg}.json $cfg "$lib${AB_LABEL:+ $AB_LABEL}"
  done
done
