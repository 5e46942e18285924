# warp-local FFT passes: stage FFT timings (default, knobs, radix plans), parity tests, short bench lines
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r5wl}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
L=gpurun_out/${TAG}.log
SH=${SHAPES:-"5003x5100 2503x10200 1009x20000"}
echo "== default" > $L
PYTHONPATH=. timeout 300 python tools/fft_bench.py $SH >> $L 2>&1
for kn in ${KNOBS:-SFFT_FFT_NO_WL SFFT_FFT_NO_WLPLAN}; do
  echo "== $kn" >> $L
  env $kn=1 PYTHONPATH=. timeout 300 python tools/fft_bench.py $SH >> $L 2>&1
done
for pl in ${PLANS}; do
  echo "== plan $pl" >> $L
  SFFT_FFT_PLAN="$pl" PYTHONPATH=. timeout 300 python tools/fft_bench.py $SH >> $L 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-stage_pfft or full_size or max_fft or line_shards_group}" > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
CONFIGS="${CONFIGS:-c3 c5 c4}" bash tools/gpu_quick_bench.sh ${TAG}
