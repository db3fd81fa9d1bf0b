#!/bin/bash
# (experiment: the code it toggles was reverted after this A/B; the numbers are in DESIGN.md §5/§8)
# bulk pre-reduction: 4-pair batches dealt round-robin over CTAs vs contiguous ranges (HEAD variant)
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
timeout 900 $R4 --master-port=33801 tests/spmd_check.py --tp 1 > gpurun_out/pi_spmd.log 2>&1; echo "spmd n4 tp1 rc=$?"; grep -E "fused|OK|FAIL" gpurun_out/pi_spmd.log | tail -2
for L in paper_2601_08800_b200/lib/variants/libmx_head.so paper_2601_08800_b200/lib/libmixserve_b200.so paper_2601_08800_b200/lib/variants/libmx_head.so paper_2601_08800_b200/lib/libmixserve_b200.so; do
  MIXSERVE_B200_LIB=$L timeout 900 $R4 --master-port=33811 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/pi_b4.json 2> gpurun_out/pi_b4.err
  MIXSERVE_B200_LIB=$L CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R2 --master-port=33812 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/pi_b2.json 2> gpurun_out/pi_b2.err
  python -c "
import json
for f in ['pi_b4','pi_b2']:
    d=json.load(open('gpurun_out/'+f+'.json')); print('$L'.split('/')[-1], f, d['config']['parallelism'], round(d['ms_per_step'],4), 'pair_reduce', round(d['phases_us'].get('pair_reduce',0),1))
"
done
