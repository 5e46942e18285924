#!/bin/bash
# per-iteration timings for library variants: VARIANTS="path:shape ..."
mkdir -p gpurun_out
for V in ${VARIANTS}; do
  LIBP=${V%%@*}; S=${V##*@}
  echo "== $LIBP $S" >> gpurun_out/variants.log
  SFFT_LIB_PATH=$LIBP SFFT_DEBUG=1 SFFT_EXPSUM=$S timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 2>&1 | grep "\[sfft\]" | tail -6 >> gpurun_out/variants.log
done
cat gpurun_out/variants.log
