# ncu of kernel KREGEX inside the single-signal latency probe (CONFIG), launches SKIP..SKIP+COUNT-1
# (NCU_SET="--set full --import-source on" by default; NCU_SET="--metrics gpu__time_duration.sum" for a launch list)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r3b}
CMD="python tools/latency_probe.py ${CONFIG:-c3}"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 1200 ncu ${NCU_SET:---set full --import-source on} --clock-control none -k "regex:${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-2} -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
