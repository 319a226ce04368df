AB="old main hs2n hs4n old main hs2n" QT_CFGS="c4 c5" bash tools/ab.sh run > gpurun_out/ab7.log 2>&1
grep "c5 mode\|c4 mode=0\|==" gpurun_out/ab7.log | cut -c1-130
