#!/bin/bash
# decode weight prefetch A/B at 2 GPUs (EP2 and TP2), plus SPMD parity with it on
mkdir -p gpurun_out
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
timeout 600 $R2 --master-port=31201 tests/spmd_check.py --tp 1 > gpurun_out/pf_spmd_tp1.log 2>&1; echo "spmd tp1 rc=$?"; grep -E "OK|FAIL" gpurun_out/pf_spmd_tp1.log | tail -1
for mb in 0 64 128; do
  for tp in 1 2; do
    MX_PREFETCH_MB=$mb timeout 900 $R2 --master-port=$((31210 + tp + mb)) tools/decode_sweep.py --tp $tp --out gpurun_out/pf_decode_tp${tp}_mb$mb.jsonl > gpurun_out/pf_decode_tp${tp}_mb$mb.log 2>&1; echo "decode tp$tp mb$mb rc=$?"
    python -c "
import json
print('tp$tp mb$mb', [(json.loads(l)['T_global'], round(json.loads(l)['fused_token_us'],1)) for l in open('gpurun_out/pf_decode_tp${tp}_mb$mb.jsonl')])
"
  done
done
