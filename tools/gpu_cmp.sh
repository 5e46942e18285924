#!/bin/bash
# GPU tests + bench of both exp-sum paths + per-iteration timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 400 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
for path in 2 1; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 --expsum-path $path > gpurun_out/bench_p$path.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_p$path.log
  SFFT_DEBUG=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --expsum-path $path 2>&1 | grep "\[sfft\]" | tail -8 > gpurun_out/iters_p$path.log
  tail -2 gpurun_out/bench_p$path.log | cut -c1-600; cat gpurun_out/iters_p$path.log
done
for cfg in c2 c4 c5; do
  for path in 2 1; do
    echo "== $cfg path $path"; timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --expsum-path $path 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['verified_exact_recovery'], d['kernel_ms_per_step'])"
  done
done
