OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_pipe or bf16_device or gemv" > $OUT/pytest_mma.log 2>&1
CCQ_FORCE_MMA=1 timeout 300 python tools/gemv_scaling.py 2.06 4096 1,2,4,8,16 > $OUT/scaling_rec_206.txt 2>&1
CCQ_FORCE_MMA=1 timeout 300 python tools/gemv_scaling.py 2.06 14336 1,4 > $OUT/scaling_rec_206_k14336.txt 2>&1
echo done
