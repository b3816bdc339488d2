set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemv or randomized" > $OUT/pytest_hw.log 2>&1; echo "rc=$?" >> $OUT/pytest_hw.log
timeout 600 python tools/time_matmul.py --family 2.06 --shapes 4096x14336,14336x4096,4096x4096 --M 2,4,8 > $OUT/hw_new.txt 2>&1
