set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_hmma -s 8 -c 1 \
    -o $OUT/prof_hmma -f python tools/prof_kernel.py --family 2.06 --din 4096 --dout 57344 --M 1 > $OUT/ncu_hmma.log 2>&1
echo done
