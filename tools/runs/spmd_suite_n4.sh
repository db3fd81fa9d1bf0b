#!/bin/bash
# the SPMD pytest file on a 4-GPU box: the one-rank-per-GPU cases (2 and 4
# ranks; device barriers over NVLink, NCCL arm) that a one-GPU box skips
timeout 900 python -m pytest tests/test_spmd_gpu.py -m gpu -v -k "not one_device" > gpurun_out/sn4_spmd_tests.log 2>&1; echo "rc=$?"
grep -E "PASSED|FAILED|SKIPPED|ERROR" gpurun_out/sn4_spmd_tests.log | sed 's/ *\[.*%\]//' ; tail -1 gpurun_out/sn4_spmd_tests.log
