# final 4-GPU pass at HEAD: SPMD parity and the bench lines of configs B and C
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
for tp in 1 2 4; do
  timeout 600 $R --master-port=$((29960 + tp)) tests/spmd_check.py --tp $tp > gpurun_out/final_spmd_n4_tp$tp.log 2>&1; echo "spmd tp$tp rc=$?"; grep -E "OK|FAIL" gpurun_out/final_spmd_n4_tp$tp.log | tail -2
done
timeout 900 $R --master-port=29971 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/final_b4.json 2> gpurun_out/final_b4.err; echo "bench B rc=$?"
timeout 1200 $R --master-port=29972 bench.py --gpus 4 --steps 10 --warmup 3 --config C > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err; echo "bench C rc=$?"
timeout 300 $R --master-port=29973 bench.py --gpus 4 --steps 5 --warmup 2 --impl reference > gpurun_out/final_ref4.json 2> gpurun_out/final_ref4.err; echo "ref rc=$?"
python tools/summarize_line.py gpurun_out/final_b4.json gpurun_out/final_c4.json | cut -c1-420
