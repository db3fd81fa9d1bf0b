#!/bin/bash
# refresh after the lean barrier / column split / SiLU changes: SPMD parity at 4 and 2 GPUs,
# decode sweeps, bench lines (default + named) of configs B and C
mkdir -p gpurun_out
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for tp in 1 2 4; do
  timeout 600 $R4 --master-port=$((31060 + tp)) tests/spmd_check.py --tp $tp > gpurun_out/rf_spmd_n4_tp$tp.log 2>&1; echo "spmd n4 tp$tp rc=$?"; grep -E "OK|FAIL" gpurun_out/rf_spmd_n4_tp$tp.log | tail -1
done
timeout 900 $R4 --master-port=31071 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/rf_b4_def.json 2> gpurun_out/rf_b4_def.err; echo "bench B n4 default rc=$?"
timeout 900 $R4 --master-port=31072 bench.py --gpus 4 --steps 20 --warmup 5 --tp 2 > gpurun_out/rf_b4_tp2.json 2> gpurun_out/rf_b4_tp2.err; echo "bench B n4 tp2 rc=$?"
timeout 1200 $R4 --master-port=31073 bench.py --gpus 4 --steps 10 --warmup 3 --config C > gpurun_out/rf_c4.json 2> gpurun_out/rf_c4.err; echo "bench C n4 rc=$?"
timeout 900 $R4 --master-port=31074 tools/decode_sweep.py --out gpurun_out/rf_decode_n4.jsonl > gpurun_out/rf_decode_n4.log 2>&1; echo "decode n4 rc=$?"
timeout 900 $R4 --master-port=31075 tools/decode_sweep.py --tp 1 --out gpurun_out/rf_decode_n4_ep4.jsonl > gpurun_out/rf_decode_n4_ep4.log 2>&1; echo "decode n4 ep4 rc=$?"
export CUDA_VISIBLE_DEVICES=0,1
timeout 900 $R2 --master-port=31081 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/rf_b2_def.json 2> gpurun_out/rf_b2_def.err; echo "bench B n2 default rc=$?"
timeout 900 $R2 --master-port=31082 bench.py --gpus 2 --steps 20 --warmup 5 --tp 2 > gpurun_out/rf_b2_tp2.json 2> gpurun_out/rf_b2_tp2.err; echo "bench B n2 tp2 rc=$?"
timeout 900 $R2 --master-port=31083 tools/decode_sweep.py --tp 1 --out gpurun_out/rf_decode_n2_ep2.jsonl > gpurun_out/rf_decode_n2_ep2.log 2>&1; echo "decode n2 ep2 rc=$?"
unset CUDA_VISIBLE_DEVICES
python tools/summarize_line.py gpurun_out/rf_b4_def.json gpurun_out/rf_b4_tp2.json gpurun_out/rf_c4.json gpurun_out/rf_b2_def.json gpurun_out/rf_b2_tp2.json | cut -c1-300
for f in rf_decode_n4 rf_decode_n4_ep4 rf_decode_n2_ep2; do
python -c "
import json
for l in open('gpurun_out/$f.jsonl'):
    d=json.loads(l); print('$f', d['T_global'], d['layout'], round(d['fused_token_us'],1), round(d['nccl_us'],1))
"
done
