cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.log 2>&1
( python tests/diag/diag_ffa2.py 0 0 1 10 4 8
  python tests/diag/diag_ffa2.py 0 0 1 0 11 15
  python tests/diag/diag_ffa2.py 1 0 1 19 1 5
  python tests/diag/diag_ffa2.py 2 0 1 0 4 8 ) > gpurun_out/r2c_diag.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "stage_expsum or cap_binds or stage_decode" > gpurun_out/r2c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_tests.log
