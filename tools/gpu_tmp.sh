mkdir -p gpurun_out
echo "== base"; timeout 600 python tools/kstats.py c5 2>&1 | tail -9 | head -5
echo "== nocf"; C2_LIB=$PWD/paper_2010_11497_b200/lib/variants/nocf.so timeout 600 python tools/kstats.py c5 2>&1 | tail -9 | head -5
