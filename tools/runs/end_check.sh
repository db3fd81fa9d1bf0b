#!/bin/bash
# last check at HEAD: parity at 2 GPUs, the one-GPU suite, smoke, the default bench lines at 1 and 2 GPUs
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for tp in 1 2; do
  timeout 900 $R2 --master-port=$((33700 + tp)) tests/spmd_check.py --tp $tp > gpurun_out/ec_spmd_tp$tp.log 2>&1; echo "spmd tp$tp rc=$?"; grep -E "OK|FAIL" gpurun_out/ec_spmd_tp$tp.log | tail -1
done
CUDA_VISIBLE_DEVICES=0 timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/ec_b1.json 2>/dev/null; echo "b1 rc=$?"
timeout 900 $R2 --master-port=33711 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/ec_b2.json 2>/dev/null; echo "b2 rc=$?"
timeout 300 $R2 --master-port=33712 bench.py --gpus 2 --steps 5 --warmup 3 --impl reference > gpurun_out/ec_ref2.json 2>/dev/null; echo "ref2 rc=$?"
python tools/summarize_line.py gpurun_out/ec_b1.json gpurun_out/ec_b2.json | cut -c1-150
cut -c1-150 gpurun_out/ec_ref2.json
