#!/bin/bash
# combine side as one persistent kernel (MX_FUSED_COMBINE=1, lean in-kernel exchange barrier) vs three launches
mkdir -p gpurun_out
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
timeout 600 $R4 --master-port=31301 tests/spmd_check.py --tp 1 > gpurun_out/fc_spmd_tp1.log 2>&1; echo "spmd tp1 rc=$?"; grep -E "fused|OK|FAIL" gpurun_out/fc_spmd_tp1.log | tail -3
timeout 600 $R4 --master-port=31302 tests/spmd_check.py --tp 2 > gpurun_out/fc_spmd_tp2.log 2>&1; echo "spmd tp2 rc=$?"; grep -E "fused|OK|FAIL" gpurun_out/fc_spmd_tp2.log | tail -3
for r in 1 2; do
for fc in 0 1; do
  MX_FUSED_COMBINE=$fc timeout 900 $R4 --master-port=$((31310 + fc + 10*r)) bench.py --gpus 4 --steps 30 --warmup 5 > gpurun_out/fc_b4_$fc.json 2> gpurun_out/fc_b4_$fc.err
  MX_FUSED_COMBINE=$fc timeout 900 $R4 --master-port=$((31312 + fc + 10*r)) bench.py --gpus 4 --steps 30 --warmup 5 --tp 2 > gpurun_out/fc_b4tp2_$fc.json 2> gpurun_out/fc_b4tp2_$fc.err
  CUDA_VISIBLE_DEVICES=0,1 MX_FUSED_COMBINE=$fc timeout 900 $R2 --master-port=$((31314 + fc + 10*r)) bench.py --gpus 2 --steps 30 --warmup 5 > gpurun_out/fc_b2_$fc.json 2> gpurun_out/fc_b2_$fc.err
  python -c "
import json
for f in ['fc_b4_$fc','fc_b4tp2_$fc','fc_b2_$fc']:
    d=json.load(open('gpurun_out/'+f+'.json')); print('round $r', f, d['config']['parallelism'], round(d['ms_per_step'],4), 'combine', round(d['phases_us'].get('combine',0),1), 'pair_reduce', round(d['phases_us'].get('pair_reduce',0),1))
"
done
done
