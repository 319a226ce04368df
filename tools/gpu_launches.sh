# ncu launch list (gpu__time_duration per kernel) of one c2_build on a config; summary by kernel
CFG=${1:-c5}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv \
  python tools/run_cfg.py $CFG 0 1 > gpurun_out/ncu_launch_$CFG.log 2>&1
python tools/launches.py gpurun_out/launches_$CFG.csv 25 > gpurun_out/launches_$CFG.txt; cat gpurun_out/launches_$CFG.txt
python tools/launches.py gpurun_out/launches_$CFG.csv --seq >> gpurun_out/launches_$CFG.txt; tail -30 gpurun_out/launches_$CFG.txt
