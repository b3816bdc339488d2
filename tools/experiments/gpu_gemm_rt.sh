#!/bin/bash
# Two row tiles per GEMM CTA (CCQ_GEMM_RT=2): parity, then timings.
OUT=gpurun_out; mkdir -p $OUT
R=$OUT/rt_timing.jsonl; : > $R
for par in 2 3; do
  CCQ_GEMM_RT=2 CCQ_GEMM_PAR=$par timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
    -k "gemm or prefill or experts or moe or k_heavy" > $OUT/rt_pytest_$par.log 2>&1
  echo "rc=$?" >> $OUT/rt_pytest_$par.log
  grep -q "rc=0" $OUT/rt_pytest_$par.log || { echo "parity failed for par=$par"; exit 1; }
done
for cfg in "1 0" "2 2" "2 3"; do
  set -- $cfg; rt=$1; par=$2
  ENVS="CCQ_GEMM_RT=$rt"; [ $par != 0 ] && ENVS="$ENVS CCQ_GEMM_PAR=$par"
  env $ENVS timeout 300 python tools/gemm_knobs.py moe deepseek >> $R 2>>$OUT/rt_err.log
  for M in 128 160; do
    env $ENVS timeout 120 python tools/gemm_knobs.py dense 2.06 7168 32768 $M >> $R 2>>$OUT/rt_err.log
    env $ENVS timeout 120 python tools/gemm_knobs.py dense 2.06 4096 14336 $M >> $R 2>>$OUT/rt_err.log
  done
  env $ENVS CCQ_GEMM_BN=160 timeout 200 python tools/gemm_knobs.py dense 2.06 8192 28672 4096 >> $R 2>>$OUT/rt_err.log
done
timeout 200 python tools/gemm_knobs.py dense 2.06 8192 28672 4096 >> $R 2>>$OUT/rt_err.log
echo done
