#!/bin/bash
# int8-limb exp-sum bring-up: stage parity, then full-size e2e parity, each under a timeout
mkdir -p gpurun_out
export SFFT_SYNC=${SFFT_SYNC:-1}
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "stage_expsum" --timeout 200 > gpurun_out/i8_stage.log 2>&1; echo "stage rc=$?" >> gpurun_out/i8_stage.log
tail -25 gpurun_out/i8_stage.log
unset SFFT_SYNC
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size" --timeout 400 > gpurun_out/i8_e2e.log 2>&1; echo "e2e rc=$?" >> gpurun_out/i8_e2e.log
tail -25 gpurun_out/i8_e2e.log
