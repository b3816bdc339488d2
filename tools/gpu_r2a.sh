set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 2400 python -m pytest tests/test_sanitizer.py -m gpu -x -q > $OUT/pytest_sanitizer.log 2>&1; echo "rc=$?" >> $OUT/pytest_sanitizer.log
