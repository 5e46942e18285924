# full GPU test suite, smoke, then bench lines + ncu evidence (tools/gpu_r2_prof.sh)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2all}
bash tools/gpu_r2_tests.sh ${TAG}
bash tools/gpu_r2_prof.sh ${TAG}
