# full ncu capture (source-level) of the stage FFT on the C3 iteration-1 shape
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r5fn}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
export PYTHONPATH=.
timeout 300 python tools/fft_bench.py ${SHAPE:-5003x5100} > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pfft -s 2 -c 1 -o gpurun_out/${TAG} python tools/fft_bench.py ${SHAPE:-5003x5100} > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
