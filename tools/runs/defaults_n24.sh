# the bench's default invocation at 2 and 4 GPUs (config B: the layout model's pick)
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=$((30100 + N)) \
    bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/def_n$N.json 2> gpurun_out/def_n$N.err; echo "n$N rc=$?"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=$((30110 + N)) \
    bench.py --gpus $N --steps 5 --warmup 2 --impl reference > gpurun_out/def_ref$N.json 2> gpurun_out/def_ref$N.err; echo "ref n$N rc=$?"
done
python tools/summarize_line.py gpurun_out/def_n2.json gpurun_out/def_n4.json | cut -c1-330
python -c "
import json
for n in (2,4):
    d=json.loads(open(f'gpurun_out/def_n{n}.json').read()); print(n, d['config']['parallelism'], d['config']['layout_choice'])
    r=json.loads(open(f'gpurun_out/def_ref{n}.json').read()); print('  ref', r['config']['parallelism'], round(r['value'],1))
"
