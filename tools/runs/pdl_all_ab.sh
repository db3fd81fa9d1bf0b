#!/bin/bash
# prefill: every phase kernel triggering its dependents at entry (MX_PDL_EARLY_ALL=1) vs decode only
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
MX_PDL_EARLY_ALL=1 timeout 900 $R4 --master-port=32301 tests/spmd_check.py --tp 1 --bench-shape > gpurun_out/pa_spmd.log 2>&1; echo "spmd rc=$?"; grep -E "bench shape|OK|FAIL" gpurun_out/pa_spmd.log | tail -2
for r in 1 2; do
for e in 0 1; do
  MX_PDL_EARLY_ALL=$e timeout 900 $R4 --master-port=$((32310 + e + 10*r)) bench.py --gpus 4 --steps 30 --warmup 5 > gpurun_out/pa4_$e.json 2> gpurun_out/pa4_$e.err
  MX_PDL_EARLY_ALL=$e timeout 900 $R4 --master-port=$((32312 + e + 10*r)) bench.py --gpus 4 --steps 30 --warmup 5 --tp 2 > gpurun_out/pa4tp2_$e.json 2> gpurun_out/pa4tp2_$e.err
  CUDA_VISIBLE_DEVICES=0,1 MX_PDL_EARLY_ALL=$e timeout 900 $R2 --master-port=$((32314 + e + 10*r)) bench.py --gpus 2 --steps 30 --warmup 5 > gpurun_out/pa2_$e.json 2> gpurun_out/pa2_$e.err
  python -c "
import json
for f in ['pa4_$e','pa4tp2_$e','pa2_$e']:
    d=json.load(open('gpurun_out/'+f+'.json')); print('r$r', f, d['config']['parallelism'], round(d['ms_per_step'],4))
"
done
done
