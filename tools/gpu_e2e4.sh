cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python tools/e2e_probe2.py c2 c3 > gpurun_out/${1:-r2x}_probe2.log 2>&1
