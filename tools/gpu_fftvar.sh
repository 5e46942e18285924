for cfg in "" "SFFT_FFT_BIGM=20000" "SFFT_FFT_TCAP=256"; do
  echo "== $cfg"
  env $cfg PYTHONPATH=. python tools/fft_bench.py 2>&1 | grep "^p="
  env $cfg CFGS="c3 c5 c4" bash tools/gpu_ab.sh
done
