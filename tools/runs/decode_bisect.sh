#!/bin/bash
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
i=0
for cfg in "MX_PDL_EARLY=0" "MX_GEMM_EARLY=0" "MX_PDL_EARLY=0 MX_GEMM_EARLY=0" "MX_BARRIER=0 MX_PDL_EARLY=0 MX_GEMM_EARLY=0"; do
  i=$((i+1))
  env $cfg timeout 900 $R2 --master-port=$((31950 + i)) tests/spmd_check.py --tp 1 > gpurun_out/db_$i.log 2>&1; echo "$cfg rc=$?"; grep -E "decode regime|FAIL|OK" gpurun_out/db_$i.log | tail -6
done
