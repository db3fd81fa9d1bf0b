#!/bin/bash
# the bulk pre-reduction's ring threshold (>= 3 pairs of slots): config C falls back to the register kernel
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
timeout 900 $R4 --master-port=32901 tests/spmd_check.py --tp 2 > gpurun_out/pt_spmd.log 2>&1; echo "spmd n4 tp2 rc=$?"; grep -E "fused|OK|FAIL" gpurun_out/pt_spmd.log | tail -2
timeout 1200 $R4 --master-port=32902 bench.py --gpus 4 --steps 10 --warmup 3 --config C > gpurun_out/pt_c4.json 2> gpurun_out/pt_c4.err; echo "C n4 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 1200 $R2 --master-port=32903 bench.py --gpus 2 --steps 10 --warmup 3 --config C > gpurun_out/pt_c2.json 2> gpurun_out/pt_c2.err; echo "C n2 rc=$?"
timeout 900 $R4 --master-port=32904 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/pt_b4.json 2> gpurun_out/pt_b4.err; echo "B n4 rc=$?"
timeout 900 $R4 --master-port=32905 bench.py --gpus 4 --steps 20 --warmup 5 --tp 2 > gpurun_out/pt_b4_tp2.json 2> gpurun_out/pt_b4_tp2.err; echo "B n4 tp2 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R2 --master-port=32906 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/pt_b2.json 2> gpurun_out/pt_b2.err; echo "B n2 rc=$?"
python -c "
import json
for f in ['pt_c4','pt_c2','pt_b4','pt_b4_tp2','pt_b2']:
    d=json.load(open('gpurun_out/'+f+'.json')); p=d['phases_us']; print(f, d['config']['parallelism'], round(d['ms_per_step'],4), round(d['value']/1e6,3), 'M tok/s', 'pair_reduce', round(p.get('pair_reduce',0),1), 'nccl', round(d.get('nccl_baseline',{}).get('ms_per_step',0) or 0,3))
"
