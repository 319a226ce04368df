set -o pipefail
mkdir -p gpurun_out
AB="rank1 rank2 rank1 rank2" QT_CFGS="c5" bash tools/ab.sh run > gpurun_out/ab3.log 2>&1
grep "c5 mode\|==" gpurun_out/ab3.log | cut -c1-120
bash tools/gpu_launches.sh c5 > /dev/null 2>&1; head -4 gpurun_out/launches_c5.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "build or merge or surv or light or c5 or c4 or random" 2>&1 | tail -3
