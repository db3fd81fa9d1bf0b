#!/bin/bash
# lean barrier + column-split warp kernels: SPMD parity, decode sweep and the bench at 2 GPUs
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for tp in 1 2; do
  timeout 600 $R --master-port=$((30160 + tp)) tests/spmd_check.py --tp $tp > gpurun_out/dn2_spmd_tp$tp.log 2>&1; echo "spmd tp$tp rc=$?"; grep -E "OK|FAIL" gpurun_out/dn2_spmd_tp$tp.log | tail -2
done
for tp in 1 2; do
  timeout 900 $R --master-port=$((30170 + tp)) tools/decode_sweep.py --tp $tp --out gpurun_out/dn2_decode_tp$tp.jsonl > gpurun_out/dn2_decode_tp$tp.log 2>&1; echo "decode tp$tp rc=$?"
  python -c "
import json
for l in open('gpurun_out/dn2_decode_tp$tp.jsonl'):
    d=json.loads(l); print(d['T_global'], d['layout'], round(d['fused_token_us'],1), round(d['nccl_us'],1), d.get('token_phases_us'))
"
done
timeout 900 $R --master-port=30181 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/dn2_b2.json 2> gpurun_out/dn2_b2.err; echo "bench B rc=$?"
python tools/summarize_line.py gpurun_out/dn2_b2.json | cut -c1-400
