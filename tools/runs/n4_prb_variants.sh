# pre-reduction CTA width (16 / 24 / 32 warps) at 4 GPUs, TP2xEP2 and EP4
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
L=paper_2601_08800_b200/lib
port=29990
for rep in 1 2; do
for lib in $L/libmixserve_b200.so $L/variants/libmx_prb24.so $L/variants/libmx_prb32.so; do
  for tp in 2 1; do
    port=$((port+1))
    MIXSERVE_B200_LIB=$lib timeout 600 $R --master-port=$port bench.py --gpus 4 --steps 20 --warmup 5 --tp $tp --no-nccl > gpurun_out/pv.json 2> gpurun_out/pv.err
    python - "$lib" "$tp" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/pv.json").read())
p = d["phases_us"]
print(sys.argv[1].split("/")[-1][:22], "tp", sys.argv[2], "ms", round(d["ms_per_step"], 4),
      "pair", round(p.get("pair_reduce", 0), 1), "combine", round(p["combine"], 1))
PY
  done
done
done
