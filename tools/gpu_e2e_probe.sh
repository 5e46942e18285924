cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2t}
timeout 600 python tools/e2e_probe.py c2 c3 c5 > gpurun_out/${TAG}_e2e_probe.log 2>&1
PROBE_PROF=0 timeout 600 python tools/e2e_probe.py c2 c3 > gpurun_out/${TAG}_e2e_probe_np.log 2>&1
