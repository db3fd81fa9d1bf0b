#!/bin/bash
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
for r in 1 2; do
for e in 0 1; do
  MX_GEMM_EARLY_ALL=$e timeout 900 $R4 --master-port=$((32100 + e + 10*r)) bench.py --gpus 4 --steps 30 --warmup 5 > gpurun_out/ea4_$e.json 2> gpurun_out/ea4_$e.err
  MX_GEMM_EARLY_ALL=$e timeout 900 $R4 --master-port=$((32102 + e + 10*r)) bench.py --gpus 4 --steps 30 --warmup 5 --tp 2 > gpurun_out/ea4tp2_$e.json 2> gpurun_out/ea4tp2_$e.err
  python -c "
import json
for f in ['ea4_$e','ea4tp2_$e']:
    d=json.load(open('gpurun_out/'+f+'.json')); print('r$r', f, d['config']['parallelism'], round(d['ms_per_step'],4))
"
done
done
