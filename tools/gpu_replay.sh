cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2rep}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python tools/paper_replay.py --out gpurun_out/${TAG}_paper_replay.json > gpurun_out/${TAG}_replay.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_replay.log
timeout 900 python -m pytest tests/test_bench_contract.py -m gpu -q > gpurun_out/${TAG}_contract.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_contract.log
