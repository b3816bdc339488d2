#!/bin/bash
# Experiment batch: micro-benchmarks, per-warp GEMV trace, GEMV row scaling.
OUT=gpurun_out; mkdir -p $OUT
( tools/micro/pipe_rate; tools/micro/hmma_rate ) > $OUT/micro.txt 2>&1
make -s -C paper_2507_07145_b200/csrc trace > $OUT/trace_build.log 2>&1
timeout 300 python tools/trace_gemv.py 2.06 > $OUT/trace_gemv.txt 2>&1
timeout 600 python tools/gemv_scaling.py 2.06 4096 1,4,16 > $OUT/scaling_206.txt 2>&1
timeout 600 python tools/gemv_scaling.py 2.75 4096 1 > $OUT/scaling_275.txt 2>&1
echo done
