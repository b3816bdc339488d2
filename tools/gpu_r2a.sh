set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemv or baseline or randomized or config4_shape or activation" > $OUT/pytest_hmma_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_hmma_all.log
CCQ_HMMA_FAMS=7 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemv or randomized or config4_shape" > $OUT/pytest_hmma_all7.log 2>&1; echo "rc=$?" >> $OUT/pytest_hmma_all7.log
timeout 600 python tools/time_matmul.py --family 2.06 --shapes 4096x14336,14336x4096,4096x4096 --M 1,2,4,8 > $OUT/hm_fix.txt 2>&1
