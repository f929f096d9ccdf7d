OUT=gpurun_out; mkdir -p $OUT; T=${1:-bp}
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x > $OUT/pytest_var_$T.log 2>&1; echo "pytest_exit=$?" >> $OUT/pytest_var_$T.log
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4_$T.json 2>&1
LBMG_IB_BAND=0 timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4_noband_$T.json 2>&1
LBMG_IB_BAND=1 timeout 600 python bench.py --config c5 --steps 40 --warmup 5 --no-cpu-baseline > $OUT/bench_c5_band_$T.json 2>&1
LBMG_IB_BAND=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_band_$T.json 2>&1
