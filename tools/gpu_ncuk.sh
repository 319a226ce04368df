# ncu --set full of selected kernels of one c5 build: NCU_SPECS="k_sl_fill_rows:0:fill k_sketch_w:0:sketch"
set -o pipefail
mkdir -p gpurun_out
timeout 300 python tools/run_cfg.py ${CFG:-c5} 0 1 > gpurun_out/plain.log 2>&1 || { echo plain run failed; exit 1; }
for spec in $NCU_SPECS; do
  IFS=: read -r kn skip tag <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kn -s $skip -c 1 \
    -o gpurun_out/ncu_$tag -f python tools/run_cfg.py ${CFG:-c5} 0 1 > gpurun_out/ncu_$tag.log 2>&1
  tail -1 gpurun_out/ncu_$tag.log
done
