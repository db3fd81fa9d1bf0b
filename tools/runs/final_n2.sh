# final 2-GPU pass at HEAD: SPMD parity and the bench lines of configs B (TP2, EP2) and C (default EP2)
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
for tp in 1 2; do
  timeout 600 $R --master-port=$((30060 + tp)) tests/spmd_check.py --tp $tp > gpurun_out/final_spmd_n2_tp$tp.log 2>&1; echo "spmd tp$tp rc=$?"; grep -E "OK|FAIL" gpurun_out/final_spmd_n2_tp$tp.log | tail -2
done
timeout 900 $R --master-port=30071 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/final_b2.json 2> gpurun_out/final_b2.err; echo "bench B rc=$?"
timeout 900 $R --master-port=30072 bench.py --gpus 2 --steps 20 --warmup 5 --tp 1 > gpurun_out/final_b2_ep2.json 2> gpurun_out/final_b2_ep2.err; echo "bench B ep2 rc=$?"
timeout 1200 $R --master-port=30073 bench.py --gpus 2 --steps 10 --warmup 3 --config C > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err; echo "bench C rc=$?"
python tools/summarize_line.py gpurun_out/final_b2.json gpurun_out/final_b2_ep2.json gpurun_out/final_c2.json | cut -c1-330
