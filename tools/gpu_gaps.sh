#!/bin/bash
# per-iteration breakdown (SFFT_DEBUG event marks) of the last execute of a short bench run, summed
mkdir -p gpurun_out
for c in ${CFGS:-c5 c3 c1}; do
  SFFT_DEBUG=1 timeout 300 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>&1 | grep "\[sfft\] iter" > gpurun_out/gap_$c.log
  python - $c <<'PY'
import re, sys
L = open("gpurun_out/gap_" + sys.argv[1] + ".log").read().splitlines()
idx = max(i for i, l in enumerate(L) if " iter 1 " in l)
L = L[idx:]
tot = [0.0] * 5
for l in L:
    for i, x in enumerate(re.findall(r"(?:setup|prep|expsum|pfft|decode) ([0-9.]+)", l)):
        tot[i] += float(x)
print(sys.argv[1], len(L), "iters; gap+setup %.3f prep %.3f expsum %.3f pfft %.3f decode %.3f (sum %.3f ms)" % (*tot, sum(tot)))
PY
done
