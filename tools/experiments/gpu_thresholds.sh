for f in 2.06 2.75 2.5; do
  for k in auto gemm; do
    python tools/time_matmul.py --family $f --shapes 4096x14336,14336x4096 --M 2,3,4,6,8,12,16 --kernel $k
  done
done > gpurun_out/thr_matmul.txt 2>&1
python tools/time_moe.py > gpurun_out/thr_moe_default.txt 2>&1
CCQ_NO_GROUPED_GEMV=1 python tools/time_moe.py > gpurun_out/thr_moe_nogemv.txt 2>&1
