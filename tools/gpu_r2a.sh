set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemm or prefill or experts or moe or randomized" > $OUT/pytest_bn.log 2>&1; echo "rc=$?" >> $OUT/pytest_bn.log
: > $OUT/bn.txt
for m in deepseek ernie; do timeout 300 python tools/gemm_knobs.py moe $m >> $OUT/bn.txt 2>&1; done
for M in 160 192 256; do timeout 300 python tools/gemm_knobs.py dense 2.06 4096 14336 $M >> $OUT/bn.txt 2>&1; done
for bn in 128 256; do CCQ_GROUPED_BN=$bn timeout 300 python tools/gemm_knobs.py moe deepseek >> $OUT/bn.txt 2>&1; done
