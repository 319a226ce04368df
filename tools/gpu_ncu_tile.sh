# ncu --set full capture of one big-cluster K7 launch (function 1) on the given config
CFG=${1:-c5}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_local_tile -s 2 -c 1 \
  -o gpurun_out/ncu_tile_$CFG -f python tools/run_cfg.py $CFG 0 1 > gpurun_out/ncu_tile_$CFG.log 2>&1
tail -3 gpurun_out/ncu_tile_$CFG.log
