#!/bin/bash
# Decode warp groups per GEMM CTA (CCQ_GEMM_PAR): parity of the GEMM paths
# under each variant, then timings (dense DeepSeek-shaped, configs[1] M=64..256,
# configs[4] prefill, ERNIE/DeepSeek grouped prefill).
OUT=gpurun_out; mkdir -p $OUT
for par in 4 6; do
  CCQ_GEMM_PAR=$par timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
    -k "gemm or prefill or experts or moe or sweep or k_heavy" > $OUT/par_pytest_$par.log 2>&1
  echo "rc=$?" >> $OUT/par_pytest_$par.log
done
R=$OUT/par_timing.jsonl; : > $R
for par in 3 4 5 6; do
  for fam in 2.06 2.75; do
    [ $fam = 2.75 ] && [ $par = 5 ] && continue
    for M in 128 160 192 256; do CCQ_GEMM_PAR=$par timeout 120 python tools/gemm_knobs.py dense $fam 4096 14336 $M >> $R 2>>$OUT/par_err.log; done
    CCQ_GEMM_PAR=$par timeout 200 python tools/gemm_knobs.py dense $fam 8192 28672 4096 >> $R 2>>$OUT/par_err.log
  done
  for mdl in deepseek ernie; do CCQ_GEMM_PAR=$par timeout 300 python tools/gemm_knobs.py moe $mdl >> $R 2>>$OUT/par_err.log; done
done
echo done
