set -u
OUT=gpurun_out
mkdir -p $OUT
s=$(date +%s.%N); timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; e=$(date +%s.%N); echo "bench wall $(echo "$e - $s" | bc) s" >> $OUT/bench.err
