#!/bin/bash
# decode GEMM early start (B boxes before the PDL wait, expand/GEMM1 triggers) A/B at 2 GPUs + parity
mkdir -p gpurun_out
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for tp in 1 2; do
  timeout 600 $R2 --master-port=$((31400 + tp)) tests/spmd_check.py --tp $tp > gpurun_out/ea_spmd_tp$tp.log 2>&1; echo "spmd tp$tp rc=$?"; grep -E "OK|FAIL" gpurun_out/ea_spmd_tp$tp.log | tail -1
done
CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do
for e in 0 1; do
  for tp in 1 2; do
    MX_GEMM_EARLY=$e timeout 900 $R2 --master-port=$((31410 + tp + 3*e + 10*r)) tools/decode_sweep.py --tp $tp --out gpurun_out/ea_decode_tp${tp}_e$e.jsonl > gpurun_out/ea_decode_tp${tp}_e$e.log 2>&1
    python -c "
import json
print('r$r tp$tp early$e', [(json.loads(l)['T_global'], round(json.loads(l)['fused_token_us'],1)) for l in open('gpurun_out/ea_decode_tp${tp}_e$e.jsonl')])
"
  done
done
done
