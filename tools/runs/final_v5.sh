#!/bin/bash
# final pass at HEAD: parity at 4 and 2 GPUs, default bench lines of configs B and C, decode at 4 GPUs
mkdir -p gpurun_out
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for tp in 1 2 4; do
  extra=""; [ $tp -ne 4 ] && extra="--bench-shape"
  timeout 900 $R4 --master-port=$((32600 + tp)) tests/spmd_check.py --tp $tp $extra > gpurun_out/f5_spmd_n4_tp$tp.log 2>&1; echo "spmd n4 tp$tp rc=$?"; grep -E "OK|FAIL" gpurun_out/f5_spmd_n4_tp$tp.log | tail -1
done
timeout 900 $R4 --master-port=32611 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/f5_b4.json 2> gpurun_out/f5_b4.err; echo "B n4 rc=$?"
timeout 900 $R4 --master-port=32612 bench.py --gpus 4 --steps 20 --warmup 5 --tp 2 > gpurun_out/f5_b4_tp2.json 2> gpurun_out/f5_b4_tp2.err; echo "B n4 tp2 rc=$?"
timeout 1200 $R4 --master-port=32613 bench.py --gpus 4 --steps 10 --warmup 3 --config C > gpurun_out/f5_c4.json 2> gpurun_out/f5_c4.err; echo "C n4 rc=$?"
timeout 900 $R4 --master-port=32614 tools/decode_sweep.py --out gpurun_out/f5_decode_n4.jsonl > gpurun_out/f5_decode_n4.log 2>&1; echo "decode n4 rc=$?"
export CUDA_VISIBLE_DEVICES=0,1
for tp in 1 2; do
  timeout 900 $R2 --master-port=$((32620 + tp)) tests/spmd_check.py --tp $tp > gpurun_out/f5_spmd_n2_tp$tp.log 2>&1; echo "spmd n2 tp$tp rc=$?"; grep -E "OK|FAIL" gpurun_out/f5_spmd_n2_tp$tp.log | tail -1
done
timeout 900 $R2 --master-port=32631 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/f5_b2.json 2> gpurun_out/f5_b2.err; echo "B n2 rc=$?"
timeout 1200 $R2 --master-port=32632 bench.py --gpus 2 --steps 10 --warmup 3 --config C > gpurun_out/f5_c2.json 2> gpurun_out/f5_c2.err; echo "C n2 rc=$?"
export CUDA_VISIBLE_DEVICES=0
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f5_b1.json 2> gpurun_out/f5_b1.err; echo "B n1 rc=$?"
timeout 1200 python bench.py --gpus 1 --steps 10 --warmup 3 --config C > gpurun_out/f5_c1.json 2> gpurun_out/f5_c1.err; echo "C n1 rc=$?"
unset CUDA_VISIBLE_DEVICES
python tools/summarize_line.py gpurun_out/f5_b1.json gpurun_out/f5_b2.json gpurun_out/f5_b4.json gpurun_out/f5_b4_tp2.json gpurun_out/f5_c1.json gpurun_out/f5_c2.json gpurun_out/f5_c4.json | cut -c1-200
python -c "
import json
print('decode n4', [(json.loads(l)['T_global'], round(json.loads(l)['fused_token_us'],1), round(json.loads(l)['nccl_us'],1)) for l in open('gpurun_out/f5_decode_n4.jsonl')])
"
