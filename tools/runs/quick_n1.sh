# quick N=1 check: the layer's GPU parity subset + one bench line
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -m gpu -x -q -k "config_b or graph_replay or capacity or validation or low_precision or swiglu" > gpurun_out/quick_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/quick_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/qb1.json 2> gpurun_out/qb1.err; echo "B rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/qb1.json").read())
print(round(d["value"] / 1e6, 3), "M tok/s", round(d["ms_per_step"], 4), "ms")
print({k: round(v, 1) for k, v in d["phases_us"].items()})
PY
