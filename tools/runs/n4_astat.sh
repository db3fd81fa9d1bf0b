# A-stationary short-K GEMM: parity, microbench, 4-GPU layer
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/as_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/as_tests.log
for v in 1 0; do
  echo "== MX_GEMM_ASTAT=$v"
  MX_GEMM_ASTAT=$v python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 2048 --K 384 --reps 5
  MX_GEMM_ASTAT=$v python tools/gemm_bench.py --G 32 --rows 512 --jitter 56 --N 2048 --K 384 --reps 5
  MX_GEMM_ASTAT=$v python tools/gemm_bench.py --G 64 --rows 8 --jitter 4 --N 2048 --K 384 --reps 5
done
for rep in 1 2; do
for v in 1 0; do
  MX_GEMM_ASTAT=$v timeout 600 $R --master-port=$((30010 + v + 2 * rep)) bench.py --gpus 4 --steps 20 --warmup 5 --no-nccl > gpurun_out/as$v.json 2> gpurun_out/as$v.err
  python - "$v" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/as{sys.argv[1]}.json").read())
p = d["phases_us"]
print("astat", sys.argv[1], "ms", round(d["ms_per_step"], 4), "gemm2", round(p["gemm2"], 1),
      "frac", round(d["rooflines"]["gemm2"]["frac"], 3))
PY
done
done
