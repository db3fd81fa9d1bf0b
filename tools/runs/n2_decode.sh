# decode sweep at 2 GPUs (TP2 and EP2), graph-captured NCCL baseline
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
timeout 900 $R --master-port=29771 tools/decode_sweep.py --iters 30 --tp 2 --out gpurun_out/decode_n2_tp2.jsonl > gpurun_out/dec2a.log 2>&1; echo "tp2 rc=$?"
timeout 900 $R --master-port=29772 tools/decode_sweep.py --iters 30 --tp 1 --out gpurun_out/decode_n2_ep2.jsonl > gpurun_out/dec2b.log 2>&1; echo "ep2 rc=$?"
for f in decode_n2_tp2 decode_n2_ep2; do echo "== $f"; python -c "
import json
for l in open('gpurun_out/$f.jsonl'):
    d=json.loads(l)
    print(d['T_global'], d['layout'], round(d['fused_token_us'],1), round(d['nccl_us'],1), round(d['speedup_token_vs_nccl'],2))
"; done
