#!/bin/bash
# A/B of library builds on the bench (C3 by default): ms/step, kernel split, exact recovery
mkdir -p gpurun_out
for lib in ${LIBS:-libsfft.so}; do
  for cfg in ${CFGS:-c3}; do
    SFFT_LIB_PATH=paper_1606_07407_b200/$lib timeout 300 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 \
      --no-cpu-baseline --e2e-steps 0 ${BENCH_ARGS} 2>/dev/null | tail -1 > gpurun_out/ab_${lib}_${cfg}.json
    python - "$lib" "$cfg" <<'PY'
import json, sys
try:
    d = json.load(open(f"gpurun_out/ab_{sys.argv[1]}_{sys.argv[2]}.json"))
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e); sys.exit()
print(f"{sys.argv[1]:22s} {sys.argv[2]} {d['ms_per_step']:.3f} ms {d['value']/1e6:.3f} M/s",
      "exact" if d["verified_exact_recovery"] else "NOT EXACT",
      {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()}, f"frac {d['roofline']['frac']:.3f}")
PY
  done
done
