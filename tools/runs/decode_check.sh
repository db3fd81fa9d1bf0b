#!/bin/bash
# decode-regime parity (spmd_check's new section) at 2 GPUs and as processes sharing one GPU
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for tp in 1 2; do
  timeout 900 $R2 --master-port=$((31900 + tp)) tests/spmd_check.py --tp $tp > gpurun_out/dc_spmd_tp$tp.log 2>&1; echo "spmd tp$tp rc=$?"; grep -E "decode regime|OK|FAIL" gpurun_out/dc_spmd_tp$tp.log | tail -4
done
CUDA_VISIBLE_DEVICES=0 timeout 1800 python -m pytest tests/test_spmd_gpu.py -m gpu -x -q -s -k "one_device" 2>&1 | grep -E "decode regime|passed|failed|FAIL|Error" | tail -12
i=0
for cfg in "MX_PDL_EARLY=0" "MX_PDL_EARLY=1"; do
  i=$((i+1))
  env $cfg timeout 600 $R2 --master-port=$((31960 + i)) tools/decode_sweep.py --tp 1 --iters 30 --out gpurun_out/dc_sweep_$i.jsonl > gpurun_out/dc_sweep_$i.log 2>&1
  python -c "
import json
print('n2 ep2 $cfg', [(json.loads(l)['T_global'], round(json.loads(l)['fused_token_us'],1)) for l in open('gpurun_out/dc_sweep_$i.jsonl')])
" || tail -3 gpurun_out/dc_sweep_$i.log
done
