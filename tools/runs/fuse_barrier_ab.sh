#!/bin/bash
# opt-in in-kernel barriers (MX_FUSE_BARRIER_T) with lean arrivals: parity and decode A/B at 2 GPUs
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
MX_FUSE_BARRIER_T=4096 timeout 900 $R2 --master-port=33101 tests/spmd_check.py --tp 1 > gpurun_out/fb_spmd_tp1.log 2>&1; echo "spmd tp1 rc=$?"; grep -E "decode regime|OK|FAIL" gpurun_out/fb_spmd_tp1.log | tail -3
MX_FUSE_BARRIER_T=4096 timeout 900 $R2 --master-port=33102 tests/spmd_check.py --tp 2 > gpurun_out/fb_spmd_tp2.log 2>&1; echo "spmd tp2 rc=$?"; grep -E "OK|FAIL" gpurun_out/fb_spmd_tp2.log | tail -1
for r in 1 2; do
for t in 0 1024; do
  MX_FUSE_BARRIER_T=$t timeout 600 $R2 --master-port=$((33110 + 10*r + (t>0))) tools/decode_sweep.py --tp 1 --iters 30 --out gpurun_out/fb_$t.jsonl > gpurun_out/fb_$t.log 2>&1
  python -c "
import json
print('r$r ep2 MX_FUSE_BARRIER_T=$t', [(json.loads(l)['T_global'], round(json.loads(l)['fused_token_us'],1)) for l in open('gpurun_out/fb_$t.jsonl')])
" || tail -3 gpurun_out/fb_$t.log
done
done
