for k in auto gemv gemm; do python tools/time_matmul.py --family 2.06 --shapes 4096x4096,4096x14336,14336x4096,8192x28672 --M 3,4,6,7,8 --kernel $k; done > gpurun_out/thr2.txt 2>&1
timeout 600 python -m pytest tests -x -q -m gpu -k "matmul or gemm or gemv" > gpurun_out/t_thr2.txt 2>&1
