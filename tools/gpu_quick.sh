#!/bin/bash
# quick loop: i8 parity (stage + full size), then per-iteration timings of the c3 bench (both paths optional)
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "stage_expsum or full_size" --timeout 300 > gpurun_out/q_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/q_tests.log
tail -4 gpurun_out/q_tests.log
for cfg in ${CFGS:-c3}; do
  echo "== $cfg"; SFFT_DEBUG=1 timeout 300 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/q_$cfg.log 2>&1
  grep "\[sfft\]" gpurun_out/q_$cfg.log | tail -${ITERS:-4}
  tail -1 gpurun_out/q_$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['verified_exact_recovery'], d['kernel_ms_per_step'])"
done
