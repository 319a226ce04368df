set -o pipefail
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/run_cfg.py c5 0 1 > gpurun_out/plain_c5.log 2>&1 || { echo plain run failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local_tile -s 2 -c 1 -o gpurun_out/ncu_tile -f python tools/run_cfg.py c5 0 1 > gpurun_out/ncu_tile.log 2>&1
tail -1 gpurun_out/ncu_tile.log
ls -la gpurun_out/ncu_tile.ncu-rep
