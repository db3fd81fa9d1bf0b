#!/bin/bash
# token dispatch: remote hosts first vs ascending host order (HEAD variant), interleaved
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
timeout 900 $R4 --master-port=33301 tests/spmd_check.py --tp 1 > gpurun_out/do_spmd.log 2>&1; echo "spmd rc=$?"; grep -E "OK|FAIL" gpurun_out/do_spmd.log | tail -1
for r in 1 2; do
 for L in paper_2601_08800_b200/lib/variants/libmx_head.so paper_2601_08800_b200/lib/libmixserve_b200.so; do
  MIXSERVE_B200_LIB=$L timeout 900 $R4 --master-port=$((33310 + r)) bench.py --gpus 4 --steps 30 --warmup 5 > gpurun_out/do_b4.json 2> gpurun_out/do_b4.err
  MIXSERVE_B200_LIB=$L timeout 900 $R4 --master-port=$((33320 + r)) bench.py --gpus 4 --steps 30 --warmup 5 --tp 2 > gpurun_out/do_b4tp2.json 2> gpurun_out/do_b4tp2.err
  MIXSERVE_B200_LIB=$L CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R2 --master-port=$((33330 + r)) bench.py --gpus 2 --steps 30 --warmup 5 > gpurun_out/do_b2.json 2> gpurun_out/do_b2.err
  python -c "
import json
for f in ['do_b4','do_b4tp2','do_b2']:
    d=json.load(open('gpurun_out/'+f+'.json')); print('r$r', '$L'.split('/')[-1], f, d['config']['parallelism'], round(d['ms_per_step'],4), 'dispatch', round(d['phases_us'].get('dispatch',0),1))
"
 done
done
