"""Print one summary row of a bench.py JSON line: config, label, ms/step, kernel split, exact flag."""
import json
import sys

path, cfg, label = sys.argv[1:4]
try:
    d = json.loads(open(path).read().strip().splitlines()[-1])
    k = d["kernel_ms_per_step"]
    print(cfg, label, round(d["ms_per_step"], 3), "ms", {a: round(b, 3) for a, b in k.items() if isinstance(b, float)},
          "exact", d["verified_exact_recovery"])
except Exception as e:  # noqa: BLE001 -- a failed run is reported, not raised
    print(cfg, label, "ERR", e)
