#!/bin/bash
# bench every config (tuning / evidence); CONFIGS="c1 c2 ..." SHAPES per config via env SHAPES_<cfg>
mkdir -p gpurun_out
for C in ${CONFIGS}; do
  var="SHAPES_${C}"; SH="${!var:-default}"
  for S in $SH; do
    echo "== $C $S" >> gpurun_out/configs.log
    SFFT_EXPSUM=$S timeout 600 python bench.py --config $C --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); r=l['roofline']
print('value %.4g ms/step %.3f expsum %.2f TF frac %.3f kernels %s ok %s e2e %.4g' % (l['value'], l['ms_per_step'], r['achieved'], r['frac'], {k: round(v,3) for k,v in l['kernel_ms_per_step'].items()}, l['verified_exact_recovery'], l['e2e']['value']))" >> gpurun_out/configs.log 2>&1
  done
done
cat gpurun_out/configs.log
