set -u
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/disp.txt
for f in 2.75 2.5 2.06; do for k in auto gemm; do timeout 600 python tools/time_matmul.py --family $f --shapes 4096x14336,14336x4096,4096x4096,8192x28672 --M 2,4,6,8 --kernel $k >> $OUT/disp.txt 2>&1; done; done
