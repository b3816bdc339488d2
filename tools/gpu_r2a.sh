set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "moe" > $OUT/pytest_moe.log 2>&1; echo "rc=$?" >> $OUT/pytest_moe.log
