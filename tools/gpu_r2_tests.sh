cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q ${2:+-k "$2"} > gpurun_out/${TAG}_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_gputests.log
