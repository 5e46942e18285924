#!/bin/bash
# exp-sum shape sweep on the bench workload (tuning only)
mkdir -p gpurun_out
for S in ${SHAPES}; do
  echo "== $S" >> gpurun_out/sweep.log
  SFFT_EXPSUM=$S timeout 300 python bench.py --steps 10 --warmup 2 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS} 2>&1 | tail -1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); r=l['roofline']
print('value %.4g ms/step %.2f expsum %.2f TF frac %.3f kernels %s ok %s' % (l['value'], l['ms_per_step'], r['achieved'], r['frac'], {k: round(v,2) for k,v in l['kernel_ms_per_step'].items()}, l['verified_exact_recovery']))" >> gpurun_out/sweep.log 2>&1
done
cat gpurun_out/sweep.log
