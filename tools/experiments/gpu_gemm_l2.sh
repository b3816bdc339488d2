#!/bin/bash
# Is the tcgen05 GEMM bound by L2 -> SM traffic of the activation operand?
# SpeedOfLight + memory workload sections for configs[4] prefill and the
# DeepSeek grouped prefill.
OUT=gpurun_out; mkdir -p $OUT
M="--metrics lts__t_bytes.sum.per_second,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second"
timeout 300 ncu $M --section SpeedOfLight --clock-control none -k regex:gemm_ccq -s 4 -c 1 \
  python tools/prof_kernel.py --family 2.06 --din 8192 --dout 28672 --M 4096 --kernel gemm --copies 2 --reps 3 > $OUT/l2_prefill.txt 2>&1
timeout 300 ncu $M --section SpeedOfLight --clock-control none -k regex:gemm_ccq -s 2 -c 1 \
  python tools/gemm_knobs.py moe deepseek > $OUT/l2_deepseek.txt 2>&1
timeout 300 ncu $M --section SpeedOfLight --clock-control none -k regex:gemm_ccq -s 4 -c 1 \
  python tools/prof_kernel.py --family 2.06 --din 4096 --dout 14336 --M 160 --kernel gemm --copies 2 --reps 3 > $OUT/l2_m160.txt 2>&1
echo done
