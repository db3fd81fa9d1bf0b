# 4 GPUs: GPU tests, SPMD parity (tp2), decode sweep
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/dc_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/dc_tests.log
timeout 600 $R --master-port=29981 tests/spmd_check.py --tp 2 > gpurun_out/dc_spmd.log 2>&1; echo "spmd rc=$?"; grep -E "OK|FAIL" gpurun_out/dc_spmd.log | tail -2
timeout 900 $R --master-port=29982 tools/decode_sweep.py --iters 30 --out gpurun_out/decode_n4_b.jsonl > gpurun_out/dc.log 2>&1; echo "decode rc=$?"
python -c "
import json
for l in open('gpurun_out/decode_n4_b.jsonl'):
    d=json.loads(l); print(d['T_global'], round(d['fused_token_us'],1), round(d['nccl_us'],1), d['token_phases_us'].get('route'), d['token_phases_us'].get('barrier_counts'))
"
