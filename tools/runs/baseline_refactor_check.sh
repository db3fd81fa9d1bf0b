#!/bin/bash
# 2-GPU check after moving the NCCL arm's group / split-size logic into
# layer.tp_ep_groups / layer.baseline_splits: SPMD parity (fused + NCCL arm)
# at TP1/TP2 and the default 2-GPU bench line (graph-captured NCCL arm).
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for tp in 1 2; do
  timeout 600 $R2 --master-port=$((33800 + tp)) tests/spmd_check.py --tp $tp > gpurun_out/brc_spmd_tp$tp.log 2>&1; echo "spmd tp$tp rc=$?"; grep -E "OK|FAIL" gpurun_out/brc_spmd_tp$tp.log | tail -1
done
timeout 600 $R2 --master-port=33811 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/brc_b2.json 2>gpurun_out/brc_b2.err; echo "b2 rc=$?"
python tools/summarize_line.py gpurun_out/brc_b2.json | cut -c1-200
