cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2z}
for c in c3 c5 c4; do SFFT_DEBUG=1 timeout 300 python tools/latency_probe.py $c > gpurun_out/${TAG}_lat_$c.log 2>&1; done
