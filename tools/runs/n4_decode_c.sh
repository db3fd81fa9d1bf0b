# 4-GPU box: decode sweep (graph-captured NCCL baseline, token-wire phases) and config C
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
timeout 1200 $R --master-port=29741 tools/decode_sweep.py --iters 30 --out gpurun_out/decode_n4.jsonl > gpurun_out/decode_n4.log 2>&1; echo "decode rc=$?"
timeout 1200 $R --master-port=29742 bench.py --gpus 4 --steps 10 --warmup 3 --config C > gpurun_out/c4.json 2> gpurun_out/c4.err; echo "bench C rc=$?"
python tools/summarize_line.py gpurun_out/c4.json
grep -E "Error" gpurun_out/c4.err | head -5
cut -c1-400 gpurun_out/decode_n4.jsonl
