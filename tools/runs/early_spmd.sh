#!/bin/bash
# early-start GEMMs on every multi-GPU forward: parity (4 and 2 GPUs, one-device suite) and bench lines
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for tp in 1 2 4; do
  extra=""; [ $tp -ne 4 ] && extra="--bench-shape"
  timeout 900 $R4 --master-port=$((32200 + tp)) tests/spmd_check.py --tp $tp $extra > gpurun_out/es_spmd_n4_tp$tp.log 2>&1; echo "spmd n4 tp$tp rc=$?"; grep -E "bench shape|decode regime|OK|FAIL" gpurun_out/es_spmd_n4_tp$tp.log | tail -4
done
for tp in 1 2; do
  CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R2 --master-port=$((32210 + tp)) tests/spmd_check.py --tp $tp --bench-shape > gpurun_out/es_spmd_n2_tp$tp.log 2>&1; echo "spmd n2 tp$tp rc=$?"; grep -E "bench shape|OK|FAIL" gpurun_out/es_spmd_n2_tp$tp.log | tail -2
done
CUDA_VISIBLE_DEVICES=0 timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 900 $R4 --master-port=32221 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/es_b4.json 2> gpurun_out/es_b4.err; echo "B n4 rc=$?"
timeout 900 $R4 --master-port=32222 bench.py --gpus 4 --steps 20 --warmup 5 --tp 2 > gpurun_out/es_b4_tp2.json 2> gpurun_out/es_b4_tp2.err; echo "B n4 tp2 rc=$?"
timeout 1200 $R4 --master-port=32223 bench.py --gpus 4 --steps 10 --warmup 3 --config C > gpurun_out/es_c4.json 2> gpurun_out/es_c4.err; echo "C n4 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R2 --master-port=32224 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/es_b2.json 2> gpurun_out/es_b2.err; echo "B n2 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R2 --master-port=32225 bench.py --gpus 2 --steps 20 --warmup 5 --tp 2 > gpurun_out/es_b2_tp2.json 2> gpurun_out/es_b2_tp2.err; echo "B n2 tp2 rc=$?"
python tools/summarize_line.py gpurun_out/es_b4.json gpurun_out/es_b4_tp2.json gpurun_out/es_c4.json gpurun_out/es_b2.json gpurun_out/es_b2_tp2.json | cut -c1-250
