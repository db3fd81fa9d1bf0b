#!/bin/bash
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
timeout 900 $R4 --master-port=33501 tools/decode_sweep.py --out gpurun_out/de_n4.jsonl > gpurun_out/de_n4.log 2>&1; echo "n4 rc=$?"
timeout 900 $R4 --master-port=33502 tools/decode_sweep.py --tp 1 --out gpurun_out/de_n4_ep4.jsonl > gpurun_out/de_n4_ep4.log 2>&1; echo "n4 ep4 rc=$?"
export CUDA_VISIBLE_DEVICES=0,1
timeout 900 $R2 --master-port=33503 tools/decode_sweep.py --tp 1 --out gpurun_out/de_n2_ep2.jsonl > gpurun_out/de_n2_ep2.log 2>&1; echo "n2 ep2 rc=$?"
timeout 900 $R2 --master-port=33504 tools/decode_sweep.py --tp 2 --out gpurun_out/de_n2_tp2.jsonl > gpurun_out/de_n2_tp2.log 2>&1; echo "n2 tp2 rc=$?"
for f in de_n4 de_n4_ep4 de_n2_ep2 de_n2_tp2; do
python -c "
import json
print('$f', [(json.loads(l)['T_global'], round(json.loads(l)['fused_token_us'],1), round(json.loads(l)['nccl_us'],1)) for l in open('gpurun_out/$f.jsonl')])
"
done
