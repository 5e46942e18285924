#!/bin/bash
# full ncu capture of the first exp-sum launch for SFFT_EXPSUM=$SHAPE
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
SFFT_EXPSUM=$SHAPE timeout 300 $CMD > gpurun_out/plain_v.log 2>&1 && \
SFFT_EXPSUM=$SHAPE timeout 900 ncu --set full --clock-control none --import-source on -k regex:expsum -s 0 -c 1 -o gpurun_out/ncu_${TAG} $CMD > gpurun_out/ncu_${TAG}.log 2>&1
echo "rc=$?"
