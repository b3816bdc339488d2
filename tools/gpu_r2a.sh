set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parallel.py -m gpu -x -q > $OUT/pytest_par.log 2>&1; echo "rc=$?" >> $OUT/pytest_par.log
timeout 900 python bench.py --steps 10 --no-cpu-baseline --no-gemm --sharded > $OUT/bench_sharded.json 2> $OUT/bench_sharded.err
