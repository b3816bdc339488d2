#!/bin/bash
# Decode warp groups (PAR) at small batches (BN = 64 tiles): configs[1] shapes at M = 4..64 on the GEMM.
OUT=gpurun_out; mkdir -p $OUT
CCQ_GEMM_PAR=6 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemm or k_heavy or sweep" > $OUT/ps_pytest_6.log 2>&1; echo "rc=$?" >> $OUT/ps_pytest_6.log
R=$OUT/ps_timing.jsonl; : > $R
for par in 3 4 5 6; do
  for shp in "4096 14336" "14336 4096" "4096 4096"; do
    for M in 4 8 16 32 64; do
      CCQ_GEMM_PAR=$par KNOB_KERNEL=gemm timeout 120 python tools/gemm_knobs.py dense 2.06 $shp $M >> $R 2>>$OUT/ps_err.log
    done
  done
done
for shp in "4096 14336" "14336 4096" "4096 4096"; do for M in 4 8; do timeout 120 python tools/gemm_knobs.py dense 2.06 $shp $M >> $R 2>>$OUT/ps_err.log; done; done
echo done
