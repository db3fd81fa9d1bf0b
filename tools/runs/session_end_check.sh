#!/bin/bash
# one-GPU check at HEAD: the pytest -m gpu suite, smoke, the default bench line
CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/se_gpu_tests.log 2>&1; tail -1 gpurun_out/se_gpu_tests.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/se_b1.json 2>gpurun_out/se_b1.err; echo "b1 rc=$?"
python tools/summarize_line.py gpurun_out/se_b1.json | cut -c1-200
