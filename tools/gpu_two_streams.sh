cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/two_streams.py > gpurun_out/${1:-r2ts}.log 2>&1
