set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemv or baseline or randomized or experts or config0" > $OUT/pytest_skip.log 2>&1; echo "rc=$?" >> $OUT/pytest_skip.log
for f in 2.06 2.75 2.5; do timeout 600 python tools/time_matmul.py --family $f --shapes 4096x14336,14336x4096,4096x4096,8192x28672 --M 1 >> $OUT/skip_t.txt 2>&1; done
timeout 300 python tools/trace_gemv.py 2.06 4096 14336 > $OUT/trace_gemv_r02b.txt 2>&1
echo done
