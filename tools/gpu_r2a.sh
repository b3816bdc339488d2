set -u
OUT=gpurun_out
mkdir -p $OUT
L=paper_2507_07145_b200
g++ -std=c++20 -O2 -I include -I /usr/local/cuda/include tools/ccq_gpu_bench.cpp -o /tmp/ccq_gpu_bench $L/libccq_b200.so -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/$L -Wl,-rpath,/usr/local/cuda/lib64 > $OUT/gb_build.log 2>&1
/tmp/ccq_gpu_bench --shapes 4096x4096,4096x14336,14336x4096 --m 1,4,16 --bpw 2.06 --iters 50 > $OUT/ccq_gpu_bench.csv 2>&1
timeout 900 python -m pytest tests/test_cpp_api.py tests/test_gpu_bench_cli.py tests/test_acceptance.py tests/test_gpu_parity.py -m gpu -x -q -k "host or cpp or bench or acceptance or gemv_f32 or single_vector or output" > $OUT/pytest_host.log 2>&1; echo "rc=$?" >> $OUT/pytest_host.log
