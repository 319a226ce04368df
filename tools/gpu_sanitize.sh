# one compute-sanitizer tool per gpurun call (B200_PROFILING.md), after a clean plain run
TOOL=${1:-memcheck}
mkdir -p gpurun_out
timeout 300 python tools/sanitize_case.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 20 $EXTRA python tools/sanitize_case.py \
  > gpurun_out/sanitize_$TOOL.log 2>&1
echo "exit $?"; tail -6 gpurun_out/sanitize_$TOOL.log
