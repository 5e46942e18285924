#!/bin/bash
# FFT variants: radix cap (SFFT_FFT_RMAX) x big-CTA threads (tuning build libsfft_t512.so)
for lib in paper_1606_07407_b200/libsfft.so paper_1606_07407_b200/libsfft_t512.so; do
  for rmax in 24 16; do
    echo "== $lib rmax $rmax"
    SFFT_LIB_PATH=$PWD/$lib SFFT_FFT_RMAX=$rmax SFFT_DEBUG=1 timeout 200 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 2>&1 | grep "\[sfft\]" | sed -n 7,9p
  done
done
