# config C at N=1: the full-size parity test and a bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k "config_c" > gpurun_out/c1_test.log 2>&1; echo "test rc=$?"; tail -1 gpurun_out/c1_test.log
timeout 900 python bench.py --config C --steps 10 --warmup 3 --no-cpu > gpurun_out/c1b.json 2> gpurun_out/c1b.err; echo "bench rc=$?"
python tools/summarize_line.py gpurun_out/c1b.json
