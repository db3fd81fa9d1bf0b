# one compute-sanitizer tool per call (B200_PROFILING.md), after a plain run
TOOL=${1:-racecheck}
mkdir -p gpurun_out
timeout 300 python tools/sanitize_layer.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 20 python tools/sanitize_layer.py > gpurun_out/san_$TOOL.log 2>&1
echo "rc=$?"; tail -8 gpurun_out/san_$TOOL.log
