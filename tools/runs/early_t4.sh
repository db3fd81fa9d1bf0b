#!/bin/bash
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
timeout 900 $R2 --master-port=32701 tests/spmd_check.py --tp 1 > gpurun_out/et_spmd.log 2>&1; echo "spmd rc=$?"; grep -E "decode regime|OK|FAIL" gpurun_out/et_spmd.log | tail -3
for r in 1 2; do
for e in 0 1; do
  MX_PDL_EARLY=$e timeout 600 $R2 --master-port=$((32710 + e + 10*r)) tools/decode_sweep.py --tp 1 --iters 30 --out gpurun_out/et_$e.jsonl > gpurun_out/et_$e.log 2>&1
  python -c "
import json
print('r$r ep2 MX_PDL_EARLY=$e', [(json.loads(l)['T_global'], round(json.loads(l)['fused_token_us'],1)) for l in open('gpurun_out/et_$e.jsonl')])
"
done
done
