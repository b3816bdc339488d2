OUT=gpurun_out; mkdir -p $OUT
for r in 4 2 1; do echo "== RPW $r"; CCQ_GEMV_RPW=$r timeout 300 python tools/gemv_scaling.py 2.06 4096 1; done > $OUT/rpw.txt 2>&1
for r in 4 2; do echo "== 2.75 RPW $r"; CCQ_GEMV_RPW=$r timeout 300 python tools/gemv_scaling.py 2.75 4096 1; done >> $OUT/rpw.txt 2>&1
echo done
