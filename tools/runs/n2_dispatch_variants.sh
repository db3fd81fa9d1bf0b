# token-wire dispatch compiled for 2/3/4 resident CTAs per SM (2 GPUs, EP2 and TP2)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
L=paper_2601_08800_b200/lib
port=29850
for rep in 1 2; do
for lib in $L/libmixserve_b200.so $L/variants/libmx_db3.so $L/variants/libmx_db4.so; do
  for tp in 1; do
    port=$((port+1))
    MIXSERVE_B200_LIB=$lib timeout 600 $R --master-port=$port bench.py --gpus 2 --steps 20 --warmup 5 --tp $tp --no-nccl > gpurun_out/dv.json 2> gpurun_out/dv.err
    python - "$lib" "$tp" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/dv.json").read())
p = d["phases_us"]
print(sys.argv[1].split("/")[-1], "tp", sys.argv[2], "ms", round(d["ms_per_step"], 4),
      "dispatch", round(p["dispatch"], 1), "expand", round(p.get("expand", 0), 1),
      "pair", round(p.get("pair_reduce", 0), 1), "combine", round(p["combine"], 1))
PY
  done
done
done
