#!/bin/bash
mkdir -p gpurun_out
for S in ${SHAPES}; do
  echo "== $S" >> gpurun_out/iters.log
  SFFT_DEBUG=1 SFFT_EXPSUM=$S timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 2>&1 | grep "\[sfft\]" | tail -6 >> gpurun_out/iters.log
done
cat gpurun_out/iters.log
