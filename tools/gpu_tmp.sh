set -o pipefail
mkdir -p gpurun_out
AB="base rmk0 ko0 both0 base rmk0 ko0 both0" QT_CFGS="c5" bash tools/ab.sh run > gpurun_out/ab4.log 2>&1
grep "c5 mode\|==" gpurun_out/ab4.log | cut -c1-130
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_time.py > gpurun_out/quick.log 2>&1; cat gpurun_out/quick.log | cut -c1-200
