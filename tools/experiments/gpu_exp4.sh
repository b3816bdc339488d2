OUT=gpurun_out; mkdir -p $OUT
for w in 16 12 8; do echo "== warps $w"; CCQ_GEMV_WARPS=$w timeout 300 python tools/gemv_scaling.py 2.06 4096 1; done > $OUT/warps.txt 2>&1
for w in 16 8; do echo "== 2.75 warps $w"; CCQ_GEMV_WARPS=$w timeout 300 python tools/gemv_scaling.py 2.75 4096 1; done >> $OUT/warps.txt 2>&1
