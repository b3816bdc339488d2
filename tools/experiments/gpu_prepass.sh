#!/bin/bash
# Single-pass activation pre-pass (2.06, 16-bit x): GEMM parity + MoE/prefill timings.
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemm or prefill or experts or moe or k_heavy or two_row" > $OUT/pp_pytest.log 2>&1; echo "rc=$?" >> $OUT/pp_pytest.log
R=$OUT/pp_timing.jsonl; : > $R
for mdl in deepseek ernie; do timeout 300 python tools/gemm_knobs.py moe $mdl >> $R 2>>$OUT/pp_err.log; done
timeout 200 python tools/gemm_knobs.py dense 2.06 8192 28672 4096 >> $R 2>>$OUT/pp_err.log
timeout 120 python tools/gemm_knobs.py dense 2.06 4096 14336 64 >> $R 2>>$OUT/pp_err.log
echo done
