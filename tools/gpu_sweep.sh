#!/bin/bash
# every BASELINE config on both exp-sum paths: ms/step, modes/s, exact recovery, kernel split, roofline frac
mkdir -p gpurun_out
for cfg in c1 c2 c3 c4 c5; do
  for path in 0 1; do
    timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 --expsum-path $path 2>/dev/null | tail -1 > gpurun_out/sweep_${cfg}_p${path}.json
    python - "$cfg" "$path" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/sweep_{sys.argv[1]}_p{sys.argv[2]}.json"))
r = d["roofline"]
print(sys.argv[1], "path", sys.argv[2], f"{d['ms_per_step']:.3f} ms", f"{d['value']/1e6:.3f} M modes/s",
      "exact" if d["verified_exact_recovery"] else "NOT EXACT", {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()},
      f"frac {r['frac']:.3f} ({r['bound']})", f"e2e {d['e2e']['value']/1e6:.3f} M")
PY
  done
done
