# N=1 bench lines: config B (+ the reference arm) and config C
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b1.json 2> gpurun_out/b1.err; echo "B rc=$?"
timeout 300 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/ref1.json 2> gpurun_out/ref1.err; echo "ref rc=$?"
timeout 900 python bench.py --config C --steps 10 --warmup 3 --no-cpu > gpurun_out/c1.json 2> gpurun_out/c1.err; echo "C rc=$?"
tail -3 gpurun_out/*.err
