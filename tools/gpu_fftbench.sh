cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2fb}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
PYTHONPATH=. timeout 300 python tools/fft_bench.py 5003x5100 2503x10200 2503x5100 1009x20000 503x50000 > gpurun_out/${TAG}.log 2>&1
SFFT_FFT_BIGM=4096 PYTHONPATH=. timeout 300 python tools/fft_bench.py 2503x10200 >> gpurun_out/${TAG}.log 2>&1
SFFT_FFT_TCAP=256 SFFT_FFT_BIGM=4096 PYTHONPATH=. timeout 300 python tools/fft_bench.py 2503x10200 >> gpurun_out/${TAG}.log 2>&1
