# scratch script for one-off gpurun calls (dev tool): full GPU tests, bench, smoke
set -o pipefail
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 300 gpurun_out/bench.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
