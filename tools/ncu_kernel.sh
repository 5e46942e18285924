#!/bin/bash
# full ncu capture of one launch of the kernel matching $KREGEX in a short bench run
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 ${BENCH_ARGS}"
timeout 300 $CMD > gpurun_out/plain_k.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${SKIP:-0} -c 1 -o gpurun_out/ncu_${TAG} $CMD > gpurun_out/ncu_${TAG}.log 2>&1
echo "rc=$?"
