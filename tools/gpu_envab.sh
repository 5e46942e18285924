# solve-level A/B of environment knobs: bench lines per config with and without each knob (interleaved, 2 rounds)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-ab}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
O=gpurun_out/${TAG}.txt; : > $O
for rep in 1 2; do
for c in ${CONFIGS:-c3 c5 c4}; do
  for kn in none ${KNOBS}; do
    if [ "$kn" = none ]; then E="SFFT_AB_NONE=1"; else E="$kn"; fi
    env $E timeout 600 python bench.py --config $c --steps ${STEPS:-10} --no-cpu-baseline --e2e-steps 0 --latency-steps 0 --fp64-steps 0 > gpurun_out/${TAG}_tmp.json 2>/dev/null
    python tools/bench_line.py gpurun_out/${TAG}_tmp.json $c $kn >> $O
  done
done
done
rm -f gpurun_out/${TAG}_tmp.json
