# the driver's round-end sequence on one GPU: GPU tests, smoke, bench; plus host-copy bandwidth
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/val_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/val_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/val_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/val_bench.json 2> gpurun_out/val_bench.err; echo "bench rc=$?"
python tools/summarize_line.py gpurun_out/val_bench.json
timeout 300 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/val_ref.json 2> gpurun_out/val_ref.err; echo "ref rc=$?"; cut -c1-200 gpurun_out/val_ref.json
timeout 120 python tools/h2d_bench.py
