#!/bin/bash
# comprehensive pass at HEAD on a 4-GPU box: SPMD parity (incl. bench shape), bench lines of configs
# B and C at 1/2/4 GPUs, decode sweeps, the 1-GPU driver sequence
mkdir -p gpurun_out
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for tp in 1 2 4; do
  extra=""; [ $tp -ne 4 ] && extra="--bench-shape"
  timeout 900 $R4 --master-port=$((31600 + tp)) tests/spmd_check.py --tp $tp $extra > gpurun_out/f3_spmd_n4_tp$tp.log 2>&1; echo "spmd n4 tp$tp rc=$?"; grep -E "bench shape|OK|FAIL" gpurun_out/f3_spmd_n4_tp$tp.log | tail -2
done
timeout 900 $R4 --master-port=31611 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/f3_b4.json 2> gpurun_out/f3_b4.err; echo "B n4 rc=$?"
timeout 900 $R4 --master-port=31612 bench.py --gpus 4 --steps 20 --warmup 5 --tp 2 > gpurun_out/f3_b4_tp2.json 2> gpurun_out/f3_b4_tp2.err; echo "B n4 tp2 rc=$?"
timeout 1200 $R4 --master-port=31613 bench.py --gpus 4 --steps 10 --warmup 3 --config C > gpurun_out/f3_c4.json 2> gpurun_out/f3_c4.err; echo "C n4 rc=$?"
timeout 300 $R4 --master-port=31614 bench.py --gpus 4 --steps 5 --warmup 3 --impl reference > gpurun_out/f3_ref4.json 2> gpurun_out/f3_ref4.err; echo "ref n4 rc=$?"
timeout 900 $R4 --master-port=31615 tools/decode_sweep.py --out gpurun_out/f3_decode_n4.jsonl > gpurun_out/f3_decode_n4.log 2>&1; echo "decode n4 rc=$?"
timeout 900 $R4 --master-port=31616 tools/decode_sweep.py --tp 1 --out gpurun_out/f3_decode_n4_ep4.jsonl > gpurun_out/f3_decode_n4_ep4.log 2>&1; echo "decode n4 ep4 rc=$?"
export CUDA_VISIBLE_DEVICES=0,1
timeout 900 $R2 --master-port=31621 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/f3_b2.json 2> gpurun_out/f3_b2.err; echo "B n2 rc=$?"
timeout 900 $R2 --master-port=31622 bench.py --gpus 2 --steps 20 --warmup 5 --tp 2 > gpurun_out/f3_b2_tp2.json 2> gpurun_out/f3_b2_tp2.err; echo "B n2 tp2 rc=$?"
timeout 1200 $R2 --master-port=31623 bench.py --gpus 2 --steps 10 --warmup 3 --config C > gpurun_out/f3_c2.json 2> gpurun_out/f3_c2.err; echo "C n2 rc=$?"
timeout 900 $R2 --master-port=31624 tools/decode_sweep.py --tp 1 --out gpurun_out/f3_decode_n2_ep2.jsonl > gpurun_out/f3_decode_n2_ep2.log 2>&1; echo "decode n2 ep2 rc=$?"
timeout 900 $R2 --master-port=31625 tools/decode_sweep.py --tp 2 --out gpurun_out/f3_decode_n2_tp2.jsonl > gpurun_out/f3_decode_n2_tp2.log 2>&1; echo "decode n2 tp2 rc=$?"
export CUDA_VISIBLE_DEVICES=0
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/f3_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/f3_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f3_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f3_b1.json 2> gpurun_out/f3_b1.err; echo "B n1 rc=$?"
timeout 1200 python bench.py --gpus 1 --steps 10 --warmup 3 --config C > gpurun_out/f3_c1.json 2> gpurun_out/f3_c1.err; echo "C n1 rc=$?"
timeout 300 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/f3_ref1.json 2> gpurun_out/f3_ref1.err; echo "ref n1 rc=$?"
unset CUDA_VISIBLE_DEVICES
python tools/summarize_line.py gpurun_out/f3_b1.json gpurun_out/f3_b2.json gpurun_out/f3_b2_tp2.json gpurun_out/f3_b4.json gpurun_out/f3_b4_tp2.json gpurun_out/f3_c1.json gpurun_out/f3_c2.json gpurun_out/f3_c4.json | cut -c1-330
for f in f3_decode_n4 f3_decode_n4_ep4 f3_decode_n2_ep2 f3_decode_n2_tp2; do
python -c "
import json
print('$f', [(json.loads(l)['T_global'], round(json.loads(l)['fused_token_us'],1), round(json.loads(l)['nccl_us'],1)) for l in open('gpurun_out/$f.jsonl')])
"
done
