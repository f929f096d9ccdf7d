OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $OUT/pytest_cf2.log 2>&1; echo "pytest_exit=$?" >> $OUT/pytest_cf2.log
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_cf2.json 2>&1
LBMG_FILL_PLAN=0 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_cf2_noplan.json 2>&1
LBMG_IB_NOSCATTER=2 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > $OUT/bench_c2_cf2_noflag.json 2>&1
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_cf2.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 150 --csv --log-file $OUT/launches_c2_cf2.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
