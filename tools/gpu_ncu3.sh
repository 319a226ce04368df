# ncu --set full captures of the three biggest Step-2 kernels of one c5 build (run after a plain run exits 0)
set -o pipefail
mkdir -p gpurun_out
timeout 300 python tools/run_cfg.py c5 0 1 > gpurun_out/plain_c5.log 2>&1 || { echo plain run failed; exit 1; }
for spec in "k_local_tile:2:tile" "k_row_topk:0:rowtopk" "k_surv_merge:1:survmerge" ${NCU_EXTRA:-}; do
  IFS=: read -r kn skip tag <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kn -s $skip -c 1 \
    -o gpurun_out/ncu_$tag -f python tools/run_cfg.py c5 0 1 > gpurun_out/ncu_$tag.log 2>&1
  tail -1 gpurun_out/ncu_$tag.log
done
