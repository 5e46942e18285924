#!/bin/bash
# FFT kernel A/B: libraries x radix plans (SFFT_FFT_PLAN) on tools/fft_bench.py
mkdir -p gpurun_out
for lib in ${LIBS:-libsfft.so}; do
  IFS='|' read -ra PL <<< "${PLANLIST:-default}"
  for plan in "${PL[@]}"; do
    if [ "$plan" = "default" ]; then unset SFFT_FFT_PLAN; else export SFFT_FFT_PLAN="$plan"; fi
    echo "== $lib plan=$plan"
    PYTHONPATH=. SFFT_LIB_PATH=paper_1606_07407_b200/$lib timeout 300 python tools/fft_bench.py ${SHAPES} 2>&1 | tail -6
  done
done
