#!/bin/bash
# bench + launch list + one full ncu capture of the exp-sum kernel (each ncu only after its plain run exited 0)
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${TAG}.log
tail -2 gpurun_out/bench_${TAG}.log
if [ -n "$NCU" ]; then
  CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 --latency-steps 0"
  timeout 300 $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
  echo "launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-expsum_i8} -s 0 -c 1 -o gpurun_out/expsum_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
  echo "full rc=$?"
fi
