# 2 GPUs: SPMD parity incl. the fused combine kernel, then bench lines with and without it
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for tp in 1 2; do
  timeout 600 $R --master-port=$((29880 + tp)) tests/spmd_check.py --tp $tp > gpurun_out/sfc_tp$tp.log 2>&1; echo "spmd tp$tp rc=$?"; grep -E "fused-combine|OK|FAIL" gpurun_out/sfc_tp$tp.log | tail -3
done
for v in 1 0; do
  MX_FUSED_COMBINE=$v timeout 600 $R --master-port=$((29890 + v)) bench.py --gpus 2 --steps 20 --warmup 5 --tp 1 --no-nccl > gpurun_out/bfc$v.json 2> gpurun_out/bfc$v.err; echo "bench fused=$v rc=$?"
  python tools/summarize_line.py gpurun_out/bfc$v.json | cut -c1-200
done
