# iteration check on the GPU box: selected gpu tests, quick timings, optional ncu tile capture
set -o pipefail
mkdir -p gpurun_out
timeout ${PT_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${PT_ARGS:-} 2>&1 | tail -15 > gpurun_out/pytest_iter.log
tail -3 gpurun_out/pytest_iter.log
timeout 600 python tools/quick_time.py ${QT_CFGS:-c1 c2 c3 c4 c5} > gpurun_out/quick.log 2>&1; cat gpurun_out/quick.log
if [ -n "$NCUTILE" ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_local_tile -s 2 -c 1 \
    -o gpurun_out/ncu_tile_c5 -f python tools/run_cfg.py c5 0 1 > gpurun_out/ncu_tile_c5.log 2>&1
  tail -2 gpurun_out/ncu_tile_c5.log
fi
if [ -n "$NCUK" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCUK" -c 1 \
    -o gpurun_out/ncu_k -f python tools/run_cfg.py c5 0 1 > gpurun_out/ncu_k.log 2>&1
  tail -2 gpurun_out/ncu_k.log
fi
