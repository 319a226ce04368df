# round-2 iteration: targeted tests first, then the whole -m gpu suite, timings, ncu pipe counts
set -o pipefail
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "${PT_K:-split_device}" 2>&1 | tail -15 > gpurun_out/pytest_k.log
tail -4 gpurun_out/pytest_k.log
if [ -n "$FULL" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
  tail -4 gpurun_out/pytest_gpu.log
fi
timeout 600 python tools/quick_time.py ${QT_CFGS:-} > gpurun_out/quick.log 2>&1; cat gpurun_out/quick.log
if [ -n "$BENCH" ]; then timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log; fi
if [ -n "$NCU" ]; then
  timeout 300 python tools/run_cfg.py c5 0 1 > gpurun_out/plain_c5.log 2>&1 && \
  timeout 900 python tools/ncu_pipes.py run c5 gpurun_out/ncu_pipes_c5.csv > gpurun_out/ncu_pipes.log 2>&1
  tail -2 gpurun_out/ncu_pipes.log
fi
if [ -n "$LAUNCH" ]; then bash tools/gpu_launches.sh > gpurun_out/launches.log 2>&1; tail -3 gpurun_out/launches.log; fi
