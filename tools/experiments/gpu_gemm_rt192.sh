#!/bin/bash
# RT=2 at 192-column tiles (SA = 2) and the grouped token-tile width with RT=2.
OUT=gpurun_out; mkdir -p $OUT
CCQ_GEMM_BN=192 CCQ_GEMM_RT=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemm_tcgen05 or prefill or gemm_bf16" > $OUT/rt192_pytest.log 2>&1; echo "rc=$?" >> $OUT/rt192_pytest.log
CCQ_GROUPED_BN=192 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "experts or moe" > $OUT/rt192g_pytest.log 2>&1; echo "rc=$?" >> $OUT/rt192g_pytest.log
R=$OUT/rt192_timing.jsonl; : > $R
for bn in 0 128 160 192 256; do
  for mdl in ernie deepseek; do CCQ_GROUPED_BN=$bn timeout 300 python tools/gemm_knobs.py moe $mdl >> $R 2>>$OUT/rt192_err.log; done
done
CCQ_GEMM_BN=192 CCQ_GEMM_RT=2 timeout 200 python tools/gemm_knobs.py dense 2.06 8192 28672 4096 >> $R 2>>$OUT/rt192_err.log
CCQ_GEMM_BN=192 timeout 200 python tools/gemm_knobs.py dense 2.06 8192 28672 4096 >> $R 2>>$OUT/rt192_err.log
for M in 192 384; do
  timeout 120 python tools/gemm_knobs.py dense 2.06 7168 32768 $M >> $R 2>>$OUT/rt192_err.log
  CCQ_GEMM_RT=1 timeout 120 python tools/gemm_knobs.py dense 2.06 7168 32768 $M >> $R 2>>$OUT/rt192_err.log
done
echo done
