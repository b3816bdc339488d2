OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_pipe or bf16_device" > $OUT/pytest_mma.log 2>&1; echo "rc=$?" >> $OUT/pytest_mma.log
timeout 600 python tools/gemv_scaling.py 2.06 4096 1,4,8,16 > $OUT/scaling_mma_206.txt 2>&1
timeout 600 python tools/gemv_scaling.py 2.75 4096 1,8 > $OUT/scaling_mma_275.txt 2>&1
timeout 600 python tools/gemv_scaling.py 2.5 4096 1,8 > $OUT/scaling_mma_25.txt 2>&1
echo done
