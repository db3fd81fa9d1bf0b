#!/bin/bash
# decode anomaly diagnosis: token-wire fused graph vs env knobs (2 GPUs, EP2)
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
nvidia-smi --query-gpu=index,name,clocks.sm,power.draw --format=csv,noheader
i=0
for cfg in "MX_PDL_EARLY=0" "MX_PDL_EARLY=0 MX_GEMM_EARLY=0" "MX_PDL_EARLY=0 MX_PREFETCH_MB=0" "MX_PDL_EARLY=0 MX_GEMM_EARLY=0 MX_PREFETCH_MB=0" "MX_PDL_EARLY=1" "MX_PDL_EARLY=1 MX_PREFETCH_MB=0"; do
  i=$((i+1))
  env $cfg timeout 600 $R2 --master-port=$((31700 + i)) tools/decode_sweep.py --tp 1 --iters 30 --out gpurun_out/dd_$i.jsonl > gpurun_out/dd_$i.log 2>&1
  python -c "
import json
print('$cfg', [(json.loads(l)['T_global'], round(json.loads(l)['fused_token_us'],1), round(json.loads(l)['fused_slot_us'],1)) for l in open('gpurun_out/dd_$i.jsonl')])
" || tail -3 gpurun_out/dd_$i.log
done
