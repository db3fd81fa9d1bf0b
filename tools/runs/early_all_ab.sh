#!/bin/bash
# prefill: early start for every grouped GEMM (MX_GEMM_EARLY_ALL=1) vs decode only
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for r in 1 2; do
for e in 0 1; do
  CUDA_VISIBLE_DEVICES=0 MX_GEMM_EARLY_ALL=$e timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/eall_n1_$e.json 2> gpurun_out/eall_n1_$e.err
  MX_GEMM_EARLY_ALL=$e timeout 900 $R2 --master-port=$((31500 + e + 10*r)) bench.py --gpus 2 --steps 30 --warmup 5 > gpurun_out/eall_n2_$e.json 2> gpurun_out/eall_n2_$e.err
  python -c "
import json
for f in ['eall_n1_$e','eall_n2_$e']:
    d=json.load(open('gpurun_out/'+f+'.json')); p=d['phases_us']; print('r$r', f, round(d['ms_per_step'],4), 'gemm1', round(p['gemm1_swiglu'],1), 'gemm2', round(p['gemm2'],1), 'expand', round(p.get('expand',0),1))
"
done
done
