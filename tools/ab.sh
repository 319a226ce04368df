# A/B timing of variant builds of the same sources (dev tool).
# usage (here):  tools/ab.sh build NAME -DX=1 ...   -> paper_2010_11497_b200/lib/variants/NAME.so
#        (GPU):  AB="base rm epi" QT_CFGS="c4 c5" bash tools/ab.sh run
set -e
if [ "$1" = build ]; then
  name=$2; shift 2
  mkdir -p paper_2010_11497_b200/lib/variants
  python -m paper_2010_11497_b200.build --out paper_2010_11497_b200/lib/variants/$name.so "$@" >/dev/null
  echo built $name
  exit 0
fi
mkdir -p gpurun_out
for v in $AB; do
  echo "== $v"
  C2_LIB=$PWD/paper_2010_11497_b200/lib/variants/$v.so timeout 600 python tools/quick_time.py ${QT_CFGS:-c4 c5} 2>&1 | tee gpurun_out/ab_$v.log
done
