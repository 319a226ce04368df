AB="main hp3 hp4 main hp3 hp4" QT_CFGS="c4 c5" bash tools/ab.sh run > gpurun_out/ab9.log 2>&1
grep "c5 mode\|c4 mode=0\|==" gpurun_out/ab9.log | cut -c1-130
C2_LIB=$PWD/paper_2010_11497_b200/lib/variants/hp3.so timeout 900 python -m pytest tests -m gpu -x -q -k "c5 or c4 or random" 2>&1 | tail -3
