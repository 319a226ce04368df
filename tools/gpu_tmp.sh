C2_LIB=$PWD/paper_2010_11497_b200/lib/variants/ksurv.so timeout 600 python tools/kstats.py c5 2>&1 | tail -4
