# 2 GPUs, EP2: the overlapped forward's stream timeline, co-resident and full-grid side kernels
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
timeout 300 $R --master-port=29621 tools/overlap_timeline.py --tp 1 2>gpurun_out/tl.err | tail -1
MX_OVERLAP_CORES=0 timeout 300 $R --master-port=29622 tools/overlap_timeline.py --tp 1 2>>gpurun_out/tl.err | tail -1
tail -n 3 gpurun_out/tl.err
