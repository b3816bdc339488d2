set -u
OUT=gpurun_out
mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pr2 tools/micro/pipe_rate2.cu > $OUT/micro_build.log 2>&1
/tmp/pr2 > $OUT/micro_pipe_rate2.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/dr3 tools/micro/decode_rate3.cu >> $OUT/micro_build.log 2>&1
timeout 300 ncu --section WarpStateStats --section ComputeWorkloadAnalysis --section SchedulerStats --section InstructionStats --clock-control none --csv --page raw -c 12 /tmp/dr3 > $OUT/ncu_micro3.csv 2> $OUT/ncu_micro3.err
echo done
