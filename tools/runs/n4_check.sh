# 4-GPU box: SPMD parity on real NVLink, bench lines for config B (TP2xEP2, EP4) and config C (TP4)
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
for tp in 2 4 1; do
  timeout 600 $R --master-port=$((29700 + tp)) tests/spmd_check.py --tp $tp > gpurun_out/spmd_n4_tp$tp.log 2>&1; echo "spmd tp$tp rc=$?"; grep -E "OK|FAIL" gpurun_out/spmd_n4_tp$tp.log | tail -3
done
timeout 900 $R --master-port=29711 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/b4.json 2> gpurun_out/b4.err; echo "bench B tp2 rc=$?"
timeout 900 $R --master-port=29712 bench.py --gpus 4 --steps 20 --warmup 5 --tp 1 > gpurun_out/b4_ep4.json 2> gpurun_out/b4_ep4.err; echo "bench B ep4 rc=$?"
timeout 900 $R --master-port=29713 bench.py --gpus 4 --steps 20 --warmup 5 --tp auto --no-nccl > gpurun_out/b4_auto.json 2> gpurun_out/b4_auto.err; echo "bench B auto rc=$?"
timeout 1200 $R --master-port=29714 bench.py --gpus 4 --steps 10 --warmup 3 --config C > gpurun_out/c4.json 2> gpurun_out/c4.err; echo "bench C rc=$?"
timeout 300 $R --master-port=29715 bench.py --gpus 4 --steps 5 --warmup 2 --impl reference > gpurun_out/ref4.json 2> gpurun_out/ref4.err; echo "ref rc=$?"
for f in b4 b4_ep4 b4_auto c4; do python tools/summarize_line.py gpurun_out/$f.json; done
cat gpurun_out/ref4.json | cut -c1-300
