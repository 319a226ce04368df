set -o pipefail
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 200 gpurun_out/bench.log
timeout 600 python tools/quick_time.py > gpurun_out/quick.log 2>&1; cut -c1-120 gpurun_out/quick.log
bash tools/gpu_launches.sh c5 > /dev/null 2>&1; head -8 gpurun_out/launches_c5.txt
timeout 300 python tools/run_cfg.py c5 0 1 > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 python tools/ncu_pipes.py run c5 gpurun_out/ncu_pipes_c5.csv > gpurun_out/ncu_pipes.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
