cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1
for ci in 0 1 2; do for ex in 0 1; do for pa in 1 2; do
  timeout 300 python tests/diag/diag_ffa.py $ci $ex $pa >> gpurun_out/r2b_diag.log 2>&1
done; done; done
