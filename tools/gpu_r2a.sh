set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config0 or moe_configs_full" --durations=5 > $OUT/pytest_new.log 2>&1; echo "rc=$?" >> $OUT/pytest_new.log
