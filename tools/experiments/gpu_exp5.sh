OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gemv" > $OUT/pytest_gemv.log 2>&1; tail -1 $OUT/pytest_gemv.log
for f in 2.06 2.75 2.5; do timeout 300 python tools/pdl_check.py $f; done > $OUT/pro.txt 2>&1
