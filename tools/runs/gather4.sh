#!/bin/bash
# GEMM1 gathering A with tile::gather4 from three issuing threads (MX_GATHER=1 MX_GATHER4=1)
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gathered" 2>&1 | tail -3
for cfg in "MX_GATHER=0" "MX_GATHER=1 MX_GATHER4=0" "MX_GATHER=1 MX_GATHER4=1"; do
  env $cfg timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/g4_n1.json 2> gpurun_out/g4_n1.err
  python -c "
import json
d=json.load(open('gpurun_out/g4_n1.json')); p=d['phases_us']; print('$cfg', round(d['ms_per_step'],4), 'dispatch', round(p['dispatch'],1), 'gemm1', round(p['gemm1_swiglu'],1), 'gemm2', round(p['gemm2'],1))
" || tail -5 gpurun_out/g4_n1.err
done
