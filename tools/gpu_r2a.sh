set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemv or baseline or randomized or widening or config0 or acceptance" > $OUT/pytest_w64.log 2>&1; echo "rc=$?" >> $OUT/pytest_w64.log
for v in 0 1; do CCQ_W64=$v timeout 600 python tools/time_matmul.py --family 2.06 --shapes 4096x14336,14336x4096,4096x4096,8192x28672 --M 1 > $OUT/w64_$v.txt 2>&1; done
timeout 300 python bench.py --no-cpu-baseline --no-gemm > $OUT/bench_w64.json 2> $OUT/bench_w64.err
