#!/bin/bash
# Which pipe binds the tcgen05 GEMM at DeepSeek-like token-tile widths:
# dense 7168 -> 32768 (= 16 experts x 2048 rows... x 16) at M = 128/160/192/256,
# normal / no decode math / no MMAs (trace build, tools/trace_gemm.py).
OUT=gpurun_out; mkdir -p $OUT
for fam in 2.06 2.75; do
FAM=$fam DIN=7168 DOUT=32768 timeout 600 python tools/trace_gemm.py 128,160,192,256 0,1,2,3 > $OUT/gemm_bound_$fam.txt 2>&1
done
DIN=8192 DOUT=28672 timeout 600 python tools/trace_gemm.py 256,512 0,1,2,3 > $OUT/gemm_bound_dense.txt 2>&1
echo done
