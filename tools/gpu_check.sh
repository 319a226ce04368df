# parity + per-config timings (+ optional bench) on the GPU box
set -o pipefail
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
timeout ${PT_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q ${PT_ARGS:-} 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_time.py ${QT_CFGS:-} > gpurun_out/quick.log 2>&1; cat gpurun_out/quick.log
if [ -n "$BENCH" ]; then timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log; fi
