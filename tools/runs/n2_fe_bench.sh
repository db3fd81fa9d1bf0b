# 2 GPUs, EP2: bench with / without the expand fused into GEMM1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
timeout 600 $R --master-port=29931 tests/spmd_check.py --tp 1 > gpurun_out/fe_spmd1.log 2>&1; echo "spmd rc=$?"; grep -E "OK|FAIL" gpurun_out/fe_spmd1.log | tail -2
for rep in 1 2; do
for v in 1 0; do
  MX_FUSED_EXPAND=$v timeout 600 $R --master-port=$((29940 + v + 2 * rep)) bench.py --gpus 2 --steps 20 --warmup 5 --tp 1 --no-nccl > gpurun_out/fe$v.json 2> gpurun_out/fe$v.err
  python - "$v" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/fe{sys.argv[1]}.json").read())
p = d["phases_us"]
print("fused_expand", sys.argv[1], "ms", round(d["ms_per_step"], 4), "expand", round(p.get("expand", 0), 1),
      "gemm1", round(p["gemm1_swiglu"], 1))
PY
done
done
