set -u
OUT=gpurun_out
mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/dr2 tools/micro/decode_rate2.cu > $OUT/micro_build.log 2>&1
/tmp/dr2 > $OUT/micro_decode_rate2c.txt 2>&1
timeout 300 ncu --section WarpStateStats --section ComputeWorkloadAnalysis --section SchedulerStats --clock-control none --csv --page raw /tmp/dr2 > $OUT/ncu_micro_c.csv 2> $OUT/ncu_micro_c.err
echo done
