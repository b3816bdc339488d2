#!/bin/bash
# RT=2 for 2.75 at 160-column tiles: parity (forced) and timing vs RT=1.
OUT=gpurun_out; mkdir -p $OUT
CCQ_GEMM_BN=160 CCQ_GEMM_RT=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemm_tcgen05 or gemm_bf16 or prefill" > $OUT/rt275_pytest.log 2>&1; echo "rc=$?" >> $OUT/rt275_pytest.log
CCQ_GROUPED_BN=160 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "experts" > $OUT/rt275g_pytest.log 2>&1; echo "rc=$?" >> $OUT/rt275g_pytest.log
R=$OUT/rt275_timing.jsonl; : > $R
for M in 150 160; do
  for rt in 1 2; do CCQ_GEMM_RT=$rt timeout 120 python tools/gemm_knobs.py dense 2.75 7168 32768 $M >> $R 2>>$OUT/rt275_err.log; done
done
for rt in 1 2; do CCQ_GEMM_RT=$rt CCQ_GEMM_BN=160 timeout 200 python tools/gemm_knobs.py dense 2.75 8192 28672 4096 >> $R 2>>$OUT/rt275_err.log; done
echo done
