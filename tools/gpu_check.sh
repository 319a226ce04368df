# parity + per-config timings (+ optional bench) on the GPU box
set -o pipefail
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_time.py ${QT_CFGS:-} > gpurun_out/quick.log 2>&1; cat gpurun_out/quick.log
if [ -n "$BENCH" ]; then timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log; fi
