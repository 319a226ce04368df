set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_time.py > gpurun_out/quick.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu.log 2>&1
python tools/launches.py gpurun_out/launches.csv > gpurun_out/launches.txt
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/quick.log; cat gpurun_out/bench.log | tail -2; cat gpurun_out/launches.txt
