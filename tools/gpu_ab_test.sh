# A/B of libsfft_base.so vs libsfft_A.so (bench) + the GPU tests on libsfft_A.so (as libsfft.so)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2ab}
CONFIGS="${CONFIGS:-c5 c3}" LIBS="libsfft_base.so libsfft_A.so" bash tools/gpu_ab2.sh ${TAG}
timeout 1500 python -m pytest tests -m gpu -x -q -k "${TESTK:-full_size or literal or line_shard or fallback or forced}" > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
