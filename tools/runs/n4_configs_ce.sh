# 4 GPUs: config E (Zipf skew, layout selection) and config C (fp8) layout sweeps
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
timeout 1500 $R --master-port=29781 tools/config_sweep.py --config E --out gpurun_out/configE_n4.jsonl > gpurun_out/ce_e.log 2>&1; echo "E rc=$?"
timeout 1500 $R --master-port=29782 tools/config_sweep.py --config C --out gpurun_out/configC_n4.jsonl > gpurun_out/ce_c.log 2>&1; echo "C rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/configE_n4.jsonl"):
    d = json.loads(l)
    print("E s=%.1f" % d["zipf_s"], {k: round(v["ms_per_step"], 3) for k, v in d["layouts"].items()},
          "best", d["measured_best"], "fused_model", d["fused_model_pick"], "selector", d["selector_pick"])
for l in open("gpurun_out/configC_n4.jsonl"):
    d = json.loads(l)
    print("C", d["layout"], round(d["ms_per_step"], 3), round(d["tokens_per_s"] / 1e6, 2), "M tok/s")
PY
