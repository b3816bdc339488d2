set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemv or baseline or randomized or config0 or experts" > $OUT/pytest_sup.log 2>&1; echo "rc=$?" >> $OUT/pytest_sup.log
: > $OUT/sup.txt
for f in 2.06 2.75 2.5; do timeout 600 python tools/time_matmul.py --family $f --shapes 4096x14336,4096x4096,14336x4096 --M 1 >> $OUT/sup.txt 2>&1; done
echo done
