cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SFFT_DEBUG=1 timeout 300 python tools/dbg_iters.py c3 c5 > gpurun_out/${1:-r2dbg}.log 2>&1
