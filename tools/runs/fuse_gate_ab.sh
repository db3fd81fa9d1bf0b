#!/bin/bash
# (experiment: the code it toggles was reverted after this A/B; the numbers are in DESIGN.md §5/§8)
# decode: softmax gate fused into k_route for groups of <= 16 tokens (one launch fewer)
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 900 $R2 --master-port=33201 tests/spmd_check.py --tp 1 > gpurun_out/fg_spmd.log 2>&1; echo "spmd rc=$?"; grep -E "decode regime|OK|FAIL" gpurun_out/fg_spmd.log | tail -3
for r in 1 2; do
for f in 0 1; do
  MX_FUSE_GATE=$f timeout 600 $R2 --master-port=$((33210 + 10*r + f)) tools/decode_sweep.py --tp 1 --iters 30 --out gpurun_out/fg_$f.jsonl > gpurun_out/fg_$f.log 2>&1
  python -c "
import json
print('r$r ep2 MX_FUSE_GATE=$f', [(json.loads(l)['T_global'], round(json.loads(l)['fused_token_us'],1)) for l in open('gpurun_out/fg_$f.jsonl')])
" || tail -3 gpurun_out/fg_$f.log
done
done
