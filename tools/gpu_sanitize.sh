# one compute-sanitizer tool per GPU call (B200_PROFILING.md): TOOL=memcheck|racecheck|synccheck|initcheck
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2s}; TOOL=${2:-memcheck}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 300 python tests/diag/sanitize_run.py > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool ${TOOL} --error-exitcode 9 python tests/diag/sanitize_run.py > gpurun_out/${TAG}_${TOOL}.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_${TOOL}.log
