#!/bin/bash
# decode on a 4-GPU box: early phase triggers (MX_PDL_EARLY) with / without the weight prefetch
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
i=0
for cfg in "MX_PDL_EARLY=0" "MX_PDL_EARLY=1" "MX_PDL_EARLY=0 MX_GEMM_EARLY=0" "MX_PDL_EARLY=1 MX_PREFETCH_MB=64"; do
  i=$((i+1))
  env $cfg timeout 600 $R4 --master-port=$((31800 + i)) tools/decode_sweep.py --iters 30 --out gpurun_out/d4_$i.jsonl > gpurun_out/d4_$i.log 2>&1
  python -c "
import json
print('n4 tp2ep2 $cfg', [(json.loads(l)['T_global'], round(json.loads(l)['fused_token_us'],1)) for l in open('gpurun_out/d4_$i.jsonl')])
" || tail -3 gpurun_out/d4_$i.log
  env $cfg CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R2 --master-port=$((31810 + i)) tools/decode_sweep.py --tp 1 --iters 30 --out gpurun_out/d2_$i.jsonl > gpurun_out/d2_$i.log 2>&1
  python -c "
import json
print('n2 ep2 $cfg', [(json.loads(l)['T_global'], round(json.loads(l)['fused_token_us'],1)) for l in open('gpurun_out/d2_$i.jsonl')])
" || tail -3 gpurun_out/d2_$i.log
done
