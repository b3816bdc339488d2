set -u
OUT=gpurun_out
mkdir -p $OUT
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-gemm > $OUT/bench_e2e_$i.json 2> $OUT/bench_e2e.err; done
echo done
