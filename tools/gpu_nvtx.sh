# NVTX ranges (SFFT_NVTX=1): parity test, bench A/B against the default, and ncu's NVTX filter as the attached tool
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r7n}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k nvtx > gpurun_out/${TAG}_test.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_test.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0 --spec-steps 0"
for r in 1 2; do
  timeout 300 $B > gpurun_out/${TAG}_off$r.json 2>/dev/null
  SFFT_NVTX=1 timeout 300 $B > gpurun_out/${TAG}_on$r.json 2>/dev/null
done
CMD1="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0 --spec-steps 0"
SFFT_NVTX=1 timeout 300 $CMD1 > gpurun_out/${TAG}_plain1.log 2>&1 && {
  SFFT_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "sfft expsum_i8/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_nvtx_expsum.csv $CMD1 > gpurun_out/${TAG}_ncu1.log 2>&1
  SFFT_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "sfft iteration 2/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_nvtx_iter2.csv $CMD1 > gpurun_out/${TAG}_ncu2.log 2>&1
  SFFT_NVTX=1 timeout 600 ncu --nvtx --print-nvtx-rename kernel --metrics gpu__time_duration.sum --clock-control none --csv -c 40 \
    --log-file gpurun_out/${TAG}_nvtx_rename.csv $CMD1 > gpurun_out/${TAG}_ncu3.log 2>&1
}
tail -2 gpurun_out/${TAG}_test.log
for f in gpurun_out/${TAG}_off1.json gpurun_out/${TAG}_on1.json gpurun_out/${TAG}_off2.json gpurun_out/${TAG}_on2.json; do
  python - "$f" <<'P'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d["ms_per_step"], d["verified_exact_recovery"])
P
done
wc -l gpurun_out/${TAG}_nvtx_*.csv
