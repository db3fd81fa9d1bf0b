#!/bin/bash
# remote-first dispatch order for n >= 3: parity at 4 GPUs (EP4 and the 8-process one-GPU layouts) and the EP4 line
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
timeout 900 $R4 --master-port=33401 tests/spmd_check.py --tp 1 --bench-shape > gpurun_out/dc2_spmd.log 2>&1; echo "spmd n4 tp1 rc=$?"; grep -E "bench shape|decode regime|OK|FAIL" gpurun_out/dc2_spmd.log | tail -4
CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests/test_spmd_gpu.py -m gpu -x -q -k one_device 2>&1 | tail -1
for r in 1 2; do
  timeout 900 $R4 --master-port=$((33410 + r)) bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/dc2_b4.json 2> gpurun_out/dc2_b4.err
  python tools/summarize_line.py gpurun_out/dc2_b4.json | cut -c1-120
done
