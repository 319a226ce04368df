# ncu --set full (with source) of the big-cluster and mixed-slice K7 launches of hash function 1
CFG=${1:-c5}
mkdir -p gpurun_out
timeout 300 python tools/run_cfg.py $CFG 0 1 > gpurun_out/plain_$CFG.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_local_tile -s 2 -c 2 \
  -o gpurun_out/ncu_tile_$CFG -f python tools/run_cfg.py $CFG 0 1 > gpurun_out/ncu_tile_$CFG.log 2>&1
tail -3 gpurun_out/ncu_tile_$CFG.log
