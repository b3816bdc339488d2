OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "experts" > $OUT/pytest_exp.log 2>&1; tail -1 $OUT/pytest_exp.log
for bn in 0 64 128 256; do echo "== BN $bn"; CCQ_GROUPED_BN=$bn timeout 800 python tools/time_moe.py | grep -E '"batch": (256|4096)' | cut -c1-200; done > $OUT/moe_bn.txt 2>&1
