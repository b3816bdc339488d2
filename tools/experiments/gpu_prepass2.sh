#!/bin/bash
# Shared-memory staged pre-pass for 2.75 / 2.5 (16-bit x): GEMM parity + prefill timings.
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemm or prefill or experts or moe or k_heavy or two_row or sweep" > $OUT/pp2_pytest.log 2>&1; echo "rc=$?" >> $OUT/pp2_pytest.log
R=$OUT/pp2_timing.jsonl; : > $R
for fam in 2.75 2.5; do
  timeout 200 python tools/gemm_knobs.py dense $fam 8192 28672 4096 >> $R 2>>$OUT/pp2_err.log
  timeout 120 python tools/gemm_knobs.py dense $fam 4096 14336 256 >> $R 2>>$OUT/pp2_err.log
done
echo done
