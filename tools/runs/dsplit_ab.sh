#!/bin/bash
# (experiment: the default stays DSPLIT=2; numbers in DESIGN.md §8)
# (experiment) four warps per token in the token dispatch (MX_DSPLIT=4 build) vs two, EP4 / TP2xEP2
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
for r in 1 2; do
 for L in paper_2601_08800_b200/lib/libmixserve_b200.so paper_2601_08800_b200/lib/variants/libmx_dsplit4.so; do
  MIXSERVE_B200_LIB=$L timeout 900 $R4 --master-port=$((33610 + r)) bench.py --gpus 4 --steps 30 --warmup 5 > gpurun_out/ds_b4.json 2> gpurun_out/ds_b4.err
  MIXSERVE_B200_LIB=$L timeout 900 $R4 --master-port=$((33620 + r)) bench.py --gpus 4 --steps 30 --warmup 5 --tp 2 > gpurun_out/ds_b4tp2.json 2> gpurun_out/ds_b4tp2.err
  python -c "
import json
for f in ['ds_b4','ds_b4tp2']:
    d=json.load(open('gpurun_out/'+f+'.json')); print('r$r', '$L'.split('/')[-1], f, d['config']['parallelism'], round(d['ms_per_step'],4), 'dispatch', round(d['phases_us'].get('dispatch',0),1))
"
 done
done
