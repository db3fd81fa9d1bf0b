#!/bin/bash
bash tools/runs/gemm_trace.sh
bash tools/runs/gemm_ab_head.sh
timeout 900 python -m pytest tests -m gpu -x -q -k "gemm or fp8 or config or swiglu" 2>&1 | tail -2
