OUT=gpurun_out; mkdir -p $OUT; T=${1:-ss}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_full_configs.py -m gpu -q -x > $OUT/pytest_$T.log 2>&1; echo "pytest_exit=$?" >> $OUT/pytest_$T.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c2d_$T.json 2>&1
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_$T.json 2>&1
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_$T.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fluid_ghost" -s 2 -c 1 \
     -o $OUT/prof_c4fl_$T python bench.py --config c4 --steps 1 --warmup 2 --no-cpu-baseline > /dev/null 2>&1
gzip -f $OUT/*.ncu-rep
