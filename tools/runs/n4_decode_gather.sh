# decode at 4 GPUs: the default expand path vs the gathered GEMM1 (MX_GATHER=1)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
timeout 900 $R --master-port=29761 tools/decode_sweep.py --iters 30 > gpurun_out/dec_a.log 2>&1; echo "default rc=$?"
MX_GATHER=1 timeout 900 $R --master-port=29762 tools/decode_sweep.py --iters 30 > gpurun_out/dec_g.log 2>&1; echo "gather rc=$?"
for f in dec_a dec_g; do echo "== $f"; grep T_global gpurun_out/$f.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l[l.index('{'):])
    print(d['T_global'], round(d['fused_token_us'],1), round(d['nccl_us'],1), d['token_phases_us'].get('expand'), d['token_phases_us'].get('gemm1_swiglu'))
"; done
