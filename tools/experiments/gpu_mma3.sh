OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_pipe or bf16_device" > $OUT/pytest_mma.log 2>&1
CCQ_FORCE_MMA=1 timeout 300 python tools/gemv_scaling.py 2.06 4096 1,8 > $OUT/scaling_mma3_206.txt 2>&1
CCQ_FORCE_MMA=1 timeout 300 python tools/gemv_scaling.py 2.75 4096 1 > $OUT/scaling_mma3_275.txt 2>&1
CCQ_FORCE_MMA=1 timeout 300 python tools/trace_mma.py 2.06 4096 14336 1 > $OUT/trace_mma_206.txt 2>&1
CCQ_FORCE_MMA=1 timeout 300 python tools/trace_mma.py 2.06 4096 14336 8 > $OUT/trace_mma_206_m8.txt 2>&1
CCQ_FORCE_MMA=1 timeout 300 python tools/trace_mma.py 2.75 4096 14336 1 > $OUT/trace_mma_275.txt 2>&1
echo done
