# A/B of runtime options: OPTS_LIST="9=256 9=512 9=1024" QT_CFGS="c4 c5" bash tools/gpu_opts.sh
mkdir -p gpurun_out
for o in $OPTS_LIST; do
  echo "== $o"
  QT_OPTS=$o timeout 600 python tools/quick_time.py ${QT_CFGS:-c4 c5} 2>&1 | tail -3
done
