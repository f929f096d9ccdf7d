OUT=gpurun_out; mkdir -p $OUT; T=${1:-cf6}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_free_functions.py -m gpu -q -x > $OUT/pytest_$T.log 2>&1; echo "pytest_exit=$?" >> $OUT/pytest_$T.log
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_$T.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c2d_$T.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ib_fused|fluid_ghost" -s 4 -c 2 \
     -o $OUT/prof_c4_$T python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_c4_$T.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ib_fused" -s 3 -c 1 \
     -o $OUT/prof_c2ib_$T python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
gzip -f $OUT/*.ncu-rep
