set -u
OUT=gpurun_out
mkdir -p $OUT
F=$OUT/raster2.txt; : > $F
for r in -1 0 -1 0; do
  for f in 2.06 2.75; do CCQ_GEMM_RASTER=$r timeout 300 python tools/gemm_knobs.py dense $f 8192 28672 4096 >> $F 2>&1; done
  CCQ_GEMM_RASTER=$r timeout 300 python tools/gemm_knobs.py moe ernie >> $F 2>&1
done
