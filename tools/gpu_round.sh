#!/bin/bash
# One GPU session: parity tests, smoke, bench (+sweep), ncu launch list and
# full captures of the GEMV and GEMM kernels.  Run under gpurun from the repo root:
#   gpurun --timeout 1800 -- 'bash tools/gpu_round.sh'
# Everything lands in gpurun_out/ (scratch); summaries worth keeping are copied
# into profiles/ by hand.
set -u
OUT=gpurun_out
mkdir -p $OUT
STAGES=${STAGES:-"info test smoke bench sweep launches ncu_gemv ncu_gemm ncu_mma ncu_hmma ncu_decode"}
has() { [[ " $STAGES " == *" $1 "* ]]; }

has info && { nvidia-smi > $OUT/nvidia-smi.txt 2>&1; nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1; }
has test && timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
has smoke && timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
has bench && timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
has sweep && timeout 1500 python bench.py --sweep --no-cpu-baseline --steps 20 > $OUT/bench_sweep.json 2> $OUT/bench_sweep.err
has launches && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-gemm > $OUT/launches_bench.log 2>&1
has ncu_gemv && timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_stream -s 8 -c 3 \
    -o $OUT/prof_gemv -f python tools/prof_kernel.py --family 2.06 --din 4096 --dout 14336 --M 1 > $OUT/ncu_gemv.log 2>&1
has ncu_gemm && timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ccq -s 4 -c 2 \
    -o $OUT/prof_gemm -f python tools/prof_kernel.py --family 2.06 --din 8192 --dout 28672 --M 4096 --kernel gemm --copies 2 --reps 3 > $OUT/ncu_gemm.log 2>&1
has ncu_mma && timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_rec206 -s 4 -c 1 \
    -o $OUT/prof_mma_m4 -f python tools/prof_kernel.py --family 2.06 --din 4096 --dout 14336 --M 4 > $OUT/ncu_mma.log 2>&1
has ncu_hmma && timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_hmma -s 4 -c 1 \
    -o $OUT/prof_hmma_m4 -f python tools/prof_kernel.py --family 2.06 --din 4096 --dout 14336 --M 4 > $OUT/ncu_hmma.log 2>&1
has ncu_decode && timeout 600 ncu --set full --clock-control none -k regex:decode_rec -s 4 -c 1 \
    -o $OUT/prof_decode -f python tools/prof_kernel.py --family 2.06 --din 4096 --dout 14336 --decode > $OUT/ncu_decode.log 2>&1
echo done
