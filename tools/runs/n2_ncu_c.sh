# 2-GPU box: NVLink counters of one rank's communicator kernels, then config C at N=2
mkdir -p gpurun_out
bash tools/runs/nvlink_ncu.sh
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
timeout 1200 $R --master-port=29731 bench.py --gpus 2 --steps 10 --warmup 3 --config C > gpurun_out/c2.json 2> gpurun_out/c2.err; echo "bench C rc=$?"
python tools/summarize_line.py gpurun_out/c2.json
grep -E "Error|error" gpurun_out/c2.err | head -5
