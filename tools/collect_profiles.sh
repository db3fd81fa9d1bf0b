#!/usr/bin/env bash
# Copy a profile_round.sh pass (gpurun_out/<tag>_*) into profiles/r01_* and
# rebuild the ncu summaries / traffic.json / model-vs-measured comparison.
#   bash tools/collect_profiles.sh r01h
set -eu
TAG=$1
G=gpurun_out
P=profiles
python tools/ncu_summary.py --launches $G/${TAG}_n1_launches.csv \
  --full $G/${TAG}_gemm_n1.ncu-rep $G/${TAG}_misc_n1.ncu-rep \
  --title "Round 1 final ncu summary -- N=1, Qwen3-30B-A3B-shaped MoE layer, 8192 tokens (bench.py --steps 3 --warmup 3 --no-cpu)" \
  --out $P/r01_n1_ncu_summary.txt --traffic-key n1 > /dev/null
python - "$TAG" <<'PY'
import json, sys
sys.path.insert(0, 'tools')
from ncu_summary import full_table
tag = sys.argv[1]
tf = json.load(open('profiles/traffic.json'))
lines = ["# Round 1 final: per-rank grouped-GEMM shapes of the 2- and 4-GPU layouts (TP2 x EP(N/2)),",
         "# tools/gemm_bench.py --G <experts per host> --rows 512 --jitter 56 (same kernel and shape as in the layer),",
         "# ncu --set full --clock-control none, one launch each", ""]
for key, G in (("n4", 64), ("n2", 128)):
    tf.setdefault(key, {})
    for N, K, ph in ((768, 2048, "gemm1_swiglu"), (2048, 384, "gemm2")):
        rec = full_table(f'gpurun_out/{tag}_gemm_{key}_N{N}_K{K}.ncu-rep')[0]
        tf[key][ph] = rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]
        lines += [f"## {key} {ph}: G={G} N={N} K={K}", json.dumps(rec, indent=1)]
tf["source"] = ("ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch; "
                "n1: r01_n1_ncu_summary.txt, n2/n4: r01_gemm_shapes_ncu.txt")
json.dump(tf, open('profiles/traffic.json', 'w'), indent=1)
open('profiles/r01_gemm_shapes_ncu.txt', 'w').write("\n".join(lines) + "\n")
PY
for n in 1 2 4; do tail -1 $G/${TAG}_n${n}_bench.json > $P/r01_n${n}_bench.json; done
tail -1 $G/${TAG}_ref.json > $P/r01_reference_arm.json
cp $G/${TAG}_n1_launches.csv $P/r01_n1_launches.csv
for f in configC_n4.jsonl configE_n4.jsonl decode_n2.jsonl decode_n4.jsonl mt_n4_gantt.csv mt_n4_trace.csv mt_n4.json; do
  cp $G/${TAG}_$f $P/r01_$f
done
if [ -d /root/reference/pkg/src ]; then
  PYTHONPATH=/root/reference/pkg/src python tools/model_vs_measured.py --trace $P/r01_mt_n4_trace.csv \
    --links $P/b200_links_n4.csv --n 2 --m 2 --out $P/r01_model_vs_measured_n4.json > /dev/null
fi
echo collected $TAG
