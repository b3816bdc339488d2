set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemv or baseline or randomized or experts or config" > $OUT/pytest_xh2.log 2>&1; echo "rc=$?" >> $OUT/pytest_xh2.log
: > $OUT/xh2.txt
for v in 0 1; do for f in 2.75 2.5; do CCQ_X_HALF=$v timeout 600 python tools/time_matmul.py --family $f --shapes 4096x14336,4096x4096 --M 1 >> $OUT/xh2.txt 2>&1; done; done
