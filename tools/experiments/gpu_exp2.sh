OUT=gpurun_out; mkdir -p $OUT
for lib in libccq_b200_trace.so libccq_b200_exp1.so libccq_b200_exp2.so; do echo "== $lib"; CCQ_FORCE_MMA=1 CCQ_TRACE_LIB=$lib timeout 300 python tools/trace_mma.py 2.06 4096 14336 1; done > $OUT/trace_exp.txt 2>&1
echo done
