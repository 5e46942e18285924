# A/B bench (libsfft_base.so vs libsfft_A.so) + the full GPU suite and smoke on libsfft_A.so (= libsfft.so)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2abf}
CONFIGS="${CONFIGS:-c2 c1 c3}" LIBS="libsfft_base.so libsfft_A.so" bash tools/gpu_ab2.sh ${TAG}
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
