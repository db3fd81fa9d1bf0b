#!/bin/bash
# (experiment: the code it toggles was reverted after this A/B; the numbers are in DESIGN.md §5/§8)
# two producer warps in the bulk pre-reduction: parity (4 GPUs + fused combine path) and A/B vs HEAD
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for tp in 1 2; do
  timeout 900 $R4 --master-port=$((32500 + tp)) tests/spmd_check.py --tp $tp --bench-shape > gpurun_out/p2_spmd_tp$tp.log 2>&1; echo "spmd n4 tp$tp rc=$?"; grep -E "bench shape|fused|OK|FAIL" gpurun_out/p2_spmd_tp$tp.log | tail -3
done
for r in 1 2; do
 for L in paper_2601_08800_b200/lib/variants/libmx_head.so paper_2601_08800_b200/lib/libmixserve_b200.so; do
  MIXSERVE_B200_LIB=$L timeout 900 $R4 --master-port=$((32510 + r)) bench.py --gpus 4 --steps 30 --warmup 5 > gpurun_out/p2_b4.json 2> gpurun_out/p2_b4.err
  MIXSERVE_B200_LIB=$L timeout 900 $R4 --master-port=$((32520 + r)) bench.py --gpus 4 --steps 30 --warmup 5 --tp 2 > gpurun_out/p2_b4tp2.json 2> gpurun_out/p2_b4tp2.err
  MIXSERVE_B200_LIB=$L CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R2 --master-port=$((32530 + r)) bench.py --gpus 2 --steps 30 --warmup 5 > gpurun_out/p2_b2.json 2> gpurun_out/p2_b2.err
  python -c "
import json
for f in ['p2_b4','p2_b4tp2','p2_b2']:
    d=json.load(open('gpurun_out/'+f+'.json')); print('r$r', '$L'.split('/')[-1], f, d['config']['parallelism'], round(d['ms_per_step'],4), 'pair_reduce', round(d['phases_us'].get('pair_reduce',0),1))
"
 done
done
