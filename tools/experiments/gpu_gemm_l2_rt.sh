#!/bin/bash
# L2 -> SM crossbar traffic of the DeepSeek grouped prefill with 256-row CTAs (RT=2, default) vs RT=1.
OUT=gpurun_out; mkdir -p $OUT
M="--metrics lts__t_bytes.sum.per_second,l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second"
timeout 300 ncu $M --clock-control none -k regex:gemm_ccq -s 2 -c 1 python tools/gemm_knobs.py moe deepseek > $OUT/l2rt_deepseek_rt2.txt 2>&1
CCQ_GEMM_RT=1 timeout 300 ncu $M --clock-control none -k regex:gemm_ccq -s 2 -c 1 python tools/gemm_knobs.py moe deepseek > $OUT/l2rt_deepseek_rt1.txt 2>&1
echo done
