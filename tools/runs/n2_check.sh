# 2-GPU box: SPMD parity on real NVLink (EP2 and TP2), then bench lines
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29611 tests/spmd_check.py --tp 1 > gpurun_out/spmd_n2_tp1.log 2>&1; echo "spmd tp1 rc=$?"; tail -3 gpurun_out/spmd_n2_tp1.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29612 tests/spmd_check.py --tp 2 > gpurun_out/spmd_n2_tp2.log 2>&1; echo "spmd tp2 rc=$?"; tail -3 gpurun_out/spmd_n2_tp2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29613 bench.py --gpus 2 --steps 20 --warmup 5 --tp 1 > gpurun_out/b2_ep2.json 2> gpurun_out/b2_ep2.err; echo "bench ep2 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29614 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/b2.json 2> gpurun_out/b2.err; echo "bench tp2 rc=$?"
for f in b2_ep2 b2; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/{f}.json").read())
except Exception as e:
    print(f, "no line", e); sys.exit(0)
print(f, round(d["value"] / 1e6, 3), "M tok/s", round(d["ms_per_step"], 4), "ms",
      "seq", d.get("sequential_ms_per_step"), "nccl", (d.get("nccl_baseline") or {}).get("ms_per_step"),
      "captured", (d.get("nccl_baseline") or {}).get("captured"), "comm", d.get("comm_us"),
      "probe", (d.get("nvlink_probe") or {}).get("gbs_per_gpu"), "clk", d.get("gemm_sm_mhz"))
PY
done
tail -5 gpurun_out/b2_ep2.err gpurun_out/b2.err
