#!/bin/bash
# full ncu capture of the first (iteration-1, largest) exp-sum launch of a short bench, per shape
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
for S in ${SHAPES}; do
  SFFT_EXPSUM=$S timeout 300 $CMD > gpurun_out/plain_$S.log 2>&1 && \
  SFFT_EXPSUM=$S timeout 900 ncu --set full --clock-control none --import-source on -k regex:expsum -s 0 -c 1 -o gpurun_out/ncu_${TAG}_$S $CMD > gpurun_out/ncu_${TAG}_$S.log 2>&1
  echo "$S rc=$?"
done
