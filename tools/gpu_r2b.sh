set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "decode or loader or acceptance or zero_scale or empty or config0" > $OUT/pytest_dec.log 2>&1; echo "rc=$?" >> $OUT/pytest_dec.log
timeout 300 python tools/time_decode.py > $OUT/decode_time.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:decode_rec -s 4 -c 1 -o $OUT/prof_decode -f python tools/prof_kernel.py --family 2.06 --din 4096 --dout 14336 --decode > $OUT/ncu_decode.log 2>&1
echo done
