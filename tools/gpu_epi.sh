cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2k}
bash tools/gpu_quick_bench.sh $TAG
python paper_1606_07407_b200/build.py --out=paper_1606_07407_b200/libsfft_prof.so -DSFFT_FFT_PROF > gpurun_out/${TAG}_pbuild.log 2>&1
for c in "c3 1" c3 c5; do
  PYTHONPATH=. SFFT_LIB_PATH=paper_1606_07407_b200/libsfft_prof.so timeout 300 python tools/fft_phases_solve.py $c >> gpurun_out/${TAG}_phases.log 2>&1
done
