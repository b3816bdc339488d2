OUT=gpurun_out; mkdir -p $OUT
timeout 300 python tools/trace_mma.py 2.06 4096 14336 1 > $OUT/trace_mma_206.txt 2>&1
timeout 300 python tools/trace_mma.py 2.06 4096 14336 8 > $OUT/trace_mma_206_m8.txt 2>&1
timeout 600 python tools/gemv_scaling.py 2.06 4096 1,8 > $OUT/scaling_mma2_206.txt 2>&1
echo done
