#!/bin/bash
# config C pre-reduction: bulk (default) vs register kernel (MX_PRB=0)
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for e in -1 0; do
  MX_PRB=$e timeout 1200 $R4 --master-port=$((32800 + e + 2)) bench.py --gpus 4 --steps 10 --warmup 3 --config C > gpurun_out/pc4_$e.json 2> gpurun_out/pc4_$e.err
  CUDA_VISIBLE_DEVICES=0,1 MX_PRB=$e timeout 1200 $R2 --master-port=$((32810 + e + 2)) bench.py --gpus 2 --steps 10 --warmup 3 --config C > gpurun_out/pc2_$e.json 2> gpurun_out/pc2_$e.err
  MX_PRB=$e timeout 900 $R4 --master-port=$((32820 + e + 2)) bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/pb4_$e.json 2> gpurun_out/pb4_$e.err
  python -c "
import json
for f in ['pc4_$e','pc2_$e','pb4_$e']:
    d=json.load(open('gpurun_out/'+f+'.json')); p=d['phases_us']; print('MX_PRB=$e', f, d['config']['parallelism'], round(d['ms_per_step'],4), 'pair_reduce', round(p.get('pair_reduce',0),1), 'combine', round(p.get('combine',0),1))
"
done
