# round-2 GPU check: all -m gpu tests, quick per-config timings, bench (c5), ncu pipe counts of the tile kernel
set -o pipefail
mkdir -p gpurun_out
timeout ${PT_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_time.py ${QT_CFGS:-} > gpurun_out/quick.log 2>&1; cat gpurun_out/quick.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 4000 gpurun_out/bench.log
if [ -n "$NCU" ]; then
  timeout 300 python tools/run_cfg.py c5 0 1 > gpurun_out/plain_c5.log 2>&1 && \
  timeout 900 python tools/ncu_pipes.py run c5 gpurun_out/ncu_pipes_c5.csv > gpurun_out/ncu_pipes.log 2>&1
  tail -2 gpurun_out/ncu_pipes.log
fi
