#!/bin/bash
# (experiment: the code it toggles was reverted after this A/B; the numbers are in DESIGN.md §5/§8)
for r in 1 2; do
for h in 0 1; do
  MX_GEMM_L2HINT=$h timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/l2h.json 2> gpurun_out/l2h.err
  python -c "
import json
d=json.load(open('gpurun_out/l2h.json')); p=d['phases_us']; print('r$r L2HINT=$h', round(d['ms_per_step'],4), 'gemm1', round(p['gemm1_swiglu'],1), 'gemm2', round(p['gemm2'],1), 'combine', round(p['combine'],1))
" || tail -5 gpurun_out/l2h.err
done
done
MX_GEMM_L2HINT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemm or swiglu" 2>&1 | tail -1
